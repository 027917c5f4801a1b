"""Error of the tensor-core MTTKRP against the fp64 engine (exact arithmetic
on the upcast tensor) at a BASELINE config's tensor and a mid-fit iterate:
per mode the relative Frobenius error, the largest row-relative error and the
mean signed error (bias) relative to the output.

  python tools/mttkrp_error.py c4 [outer iterations before sampling]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa: F401,E402
import numpy as np
import torch

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import mttkrp_device

name = sys.argv[1]
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = synth.CONFIGS[name]
dseed, fseed = synth.seeds()
x = synth.generate_box(synth.SynthSpec.of(w), dtype="float32")
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)
res = P.fit(P.DenseTensor(x), w.rank, None, cfg, engine="cuda_core")
f = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in res.state.factors]
x64 = x.double()
for mode in (1, 2, 3):
    tc = mttkrp_device(x, f, mode, P.solver._engine_code("tcgen05"))
    ref = mttkrp_device(x64, f, mode, P.solver._engine_code("cuda_core"))
    err = tc - ref
    fro = float(torch.linalg.norm(err) / torch.linalg.norm(ref))
    rowrel = float((torch.linalg.norm(err, dim=1) / torch.linalg.norm(ref, dim=1).clamp_min(1e-300)).max())
    bias = float((err * torch.sign(ref)).sum() / ref.abs().sum())
    colrel = (torch.linalg.norm(err, dim=0) / torch.linalg.norm(ref, dim=0)).cpu().numpy()
    print(f"{name} after {outer} outer, mode {mode}: rel fro {fro:.2e}, max row rel {rowrel:.2e}, "
          f"bias {bias:.2e}, worst column rel {colrel.max():.2e}", flush=True)

if os.environ.get("DETAIL"):
    fl = {1: (1, 2), 2: (0, 2), 3: (0, 1)}  # (F_hi, F_lo) factor indices per mode
    for mode in (1, 2):
        tc = mttkrp_device(x, f, mode, P.solver._engine_code("tcgen05"))
        ref = mttkrp_device(x64, f, mode, P.solver._engine_code("cuda_core"))
        err = (tc - ref)
        hi, lo = f[fl[mode][0]], f[fl[mode][1]]
        for r in range(w.rank):
            nr = float(torch.linalg.norm(ref[:, r]))
            if nr == 0:
                print(f"mode {mode} col {r}: zero column (hi max {float(hi[:, r].abs().max()):.3e} lo max {float(lo[:, r].abs().max()):.3e})")
                continue
            e = float(torch.linalg.norm(err[:, r])) / nr
            b = float((err[:, r] * torch.sign(ref[:, r])).sum() / ref[:, r].abs().sum())
            lc = lo[:, r].abs()
            print(f"mode {mode} col {r}: rel {e:.2e} bias {b:+.2e} | lo max {float(lc.max()):.3e} "
                  f"mean/max {float(lc.mean() / lc.max().clamp_min(1e-300)):.2e} zeros {int((lc == 0).sum())}"
                  f" neg {int((lo[:, r] < 0).sum())} | hi max {float(hi[:, r].abs().max()):.3e} "
                  f"hi neg {int((hi[:, r] < 0).sum())}", flush=True)
