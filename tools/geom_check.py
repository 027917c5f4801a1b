"""MTTKRP error (tcgen05 vs the fp64 engine) at the iterates of the
kernel-geometry test fit (tests/test_gpu_parity.py), for the configured CTA
grouping (NTF_TC_CG with a diagnostic build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa
import numpy as np, torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200.engine import mttkrp_device
from oracle import ntf_oracle as O
E = P.solver._engine_code
rng = np.random.default_rng(8)
dims, R = (512, 400, 300), 20
x = (O.reconstruct([rng.random((d, R)) for d in dims]) + 0.1 * rng.standard_normal(dims)).astype(np.float32)
for n in (1, 2, 3):
    cfg = P.SolverConfig(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=n, max_restarts=0, inner_sweeps=2)
    res = P.fit(P.DenseTensor(x), R, None, cfg, engine="cuda_core")
    f = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in res.state.factors]
    xd = torch.from_numpy(x).cuda()
    for mode in (1, 2, 3):
        a = mttkrp_device(xd, f, mode, E("tcgen05"))
        b = mttkrp_device(xd.double(), f, mode, E("cuda_core"))
        err = a - b
        print(f"iter {n} mode {mode} CG={os.environ.get('NTF_TC_CG','auto')}: rel {float(torch.linalg.norm(err)/torch.linalg.norm(b)):.2e} "
              f"max row rel {float((torch.linalg.norm(err,dim=1)/torch.linalg.norm(b,dim=1)).max()):.2e}", flush=True)
got = P.fit(P.DenseTensor(x), R, None, P.SolverConfig(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=3, max_restarts=0, inner_sweeps=2))
print("fit rfe", got.rfe)
