"""How sensitive is a BASELINE fp32 config's final RFE to rounding-level
perturbations of the input, in the REFERENCE itself?  Runs cpadmm.fit on the
generator's tensor and on copies with i.i.d. relative perturbations of each
element (build container only: imports the reference from /root/reference).

  python tools/sensitivity.py c4 1e-15 1e-12 1e-9
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpadmm  # noqa: E402
from cpadmm import solver, tensors  # noqa: E402

from oracle import ntf_oracle as O  # noqa: E402

name = sys.argv[1]
eps = [float(v) for v in sys.argv[2:]] or [1e-15, 1e-12, 1e-9]
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                         f"fp32_{name}.npz"))
dims = tuple(int(d) for d in g["dims"])
R = int(g["rank"])
x, _, _ = O.generate(dims, R, float(g["snr_db"]), int(g["data_seed"]), float(g["zero_frac"]), dtype=np.float32)
x64 = x.astype(np.float64)
del x
cfg = solver.SolverConfig(seed=int(g["fit_seed"]), eps_abs=0.0, eps_rel=0.0, n_max=int(g["outer"]),
                          max_restarts=0, inner_sweeps=int(g["inner"]), rho_init=float(g["rho0"]))
base = float(g["fit_rfe"])
rng = np.random.default_rng(5)
for e in eps:
    t0 = time.time()
    xp = x64 * (1.0 + e * rng.standard_normal(x64.shape))
    res = cpadmm.fit(tensors.DenseTensor(xp), R, None, cfg)
    print(f"{name} input perturbation {e:.0e}: rfe {res.rfe:.12f} vs unperturbed {base:.12f} "
          f"rel {abs(res.rfe - base) / base:.3e} ({time.time() - t0:.0f}s)", flush=True)
