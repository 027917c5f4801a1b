"""Diagnostic: per-iteration deviation of the c1 fit from the reference fixture."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import load_golden, rel
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from oracle import ntf_oracle as O

g = load_golden("c1.npz")
w = synth.CONFIGS["c1"]
dseed, fseed = synth.seeds()
x, _ = synth.generate(w.dims, w.rank, w.snr_db, dseed)
rng = np.random.default_rng(0)
f = [rng.random((d, 10)) for d in x.shape]
t = O.OracleTensor(x)
for mode in (1, 2, 3):
    print("mttkrp mode", mode, rel(P.mttkrp_factors(x, f, mode), O.mttkrp(t, f, mode)))
for inner in (1, 10):
    cfg = dict(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=12, max_restarts=0, inner_sweeps=inner,
               rho_init=1.0, track_factors=True)
    a = P.fit(x, 10, None, P.SolverConfig(**cfg))
    b = O.fit(x, 10, O.Config(**cfg))
    for it in range(12):
        print(inner, it, [f"{rel(a.factor_history[it][m], b.factor_history[it][m]):.2e}" for m in range(3)],
              a.rho_history[it], b.rho_history[it])
