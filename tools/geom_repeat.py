"""Repeat the kernel-geometry test fit (tests/test_gpu_parity.py) and the
MTTKRP of its final state a few times in one process: run-to-run identical?"""
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
cfg = P.SolverConfig(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=3, max_restarts=0, inner_sweeps=2)
res = P.fit(P.DenseTensor(x), R, None, cfg, engine="cuda_core")
f = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in res.state.factors]
xd = torch.from_numpy(x).cuda()
for mode in (1, 2, 3):
    outs = [mttkrp_device(xd, f, mode, E("tcgen05")) for _ in range(6)]
    b = mttkrp_device(xd.double(), f, mode, E("cuda_core"))
    print(f"mode {mode}: identical {all(torch.equal(outs[0], o) for o in outs)}; rel "
          + " ".join(f"{float(torch.linalg.norm(o - b) / torch.linalg.norm(b)):.2e}" for o in outs), flush=True)
for k in range(4):
    got = P.fit(P.DenseTensor(x), R, None, cfg)
    print("fit rfe", got.rfe, flush=True)
    P.solver.release_plan_cache()
