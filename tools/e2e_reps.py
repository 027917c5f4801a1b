"""Wall time of repeated public fit() calls (c2, bench e2e leg) to expose outliers."""
import os, sys, time
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
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.fit(P.DenseTensor(xh), w.rank, None, cfg)
    torch.cuda.synchronize()
    print(f"fit {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
