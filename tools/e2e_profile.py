"""cProfile of the public fit() call (c2) as bench.py's e2e leg runs it."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth

w = synth.CONFIGS["c2"]
dseed, fseed = synth.seeds()
xh = torch.empty(w.dims, dtype=torch.float32, pin_memory=True)
synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=np.float32, out=xh.numpy())
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)
P.fit(P.DenseTensor(xh), w.rank, None, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(2):
    P.fit(P.DenseTensor(xh), w.rank, None, cfg)
torch.cuda.synchronize()
pr.disable()
print("per fit s", (time.perf_counter() - t0) / 2)
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
