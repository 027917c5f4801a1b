"""Per-iteration comparison of a fp32 golden fit (tests/golden/fp32_NAME.npz,
the reference's own trajectory) with the device fit, per engine: penalty
sequence, primal/dual residuals, final RFE."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth

name = sys.argv[1]
engines = sys.argv[2:] or ["tcgen05", "cuda_core"]
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", f"fp32_{name}.npz"))
dims = tuple(int(d) for d in g["dims"])
R = int(g["rank"])
spec = synth.SynthSpec.make(dims, R, float(g["snr_db"]), int(g["data_seed"]), float(g["zero_frac"]))
x = synth.generate_box(spec, dtype="float32")
cfg = P.SolverConfig(seed=int(g["fit_seed"]), eps_abs=0.0, eps_rel=0.0, n_max=int(g["outer"]), max_restarts=0,
                     inner_sweeps=int(g["inner"]), rho_init=float(g["rho0"]))
want = float(g["fit_rfe"])
for eng in engines:
    res = P.fit(P.DenseTensor(x), R, None, cfg, engine=eng)
    rho = np.array(res.rho_history)
    prim = np.array([r.primal for r in res.residual_history])
    dual = np.array([r.dual for r in res.residual_history])
    first = next((i for i in range(len(rho)) if not np.array_equal(rho[i], g["fit_rho"][i])), None)
    dp = np.max(np.abs(prim - g["fit_primal"]) / np.abs(g["fit_primal"]), axis=1)
    print(f"{name} {eng}: rfe {res.rfe:.12f} ref {want:.12f} rel {abs(res.rfe - want) / want:.3e}; "
          f"first rho difference at iteration {first}", flush=True)
    print("  primal rel diff per iteration:", " ".join(f"{v:.1e}" for v in dp), flush=True)
    if first is not None:
        print("  rho ours", rho[first], "ref", g["fit_rho"][first], flush=True)
    P.solver.release_plan_cache()
