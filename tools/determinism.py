"""Run the same fit several times in one process (fresh plan each time) and
report whether the final RFE and residual histories are bitwise equal.

  python tools/determinism.py c4 [reps] [engine]
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa: F401,E402
import numpy as np
import torch

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = sys.argv[3] if len(sys.argv) > 3 else "auto"
outer = int(os.environ.get("OUTER", "0"))
w = synth.CONFIGS[name]
dseed, fseed = synth.seeds()
x = synth.generate_box(synth.SynthSpec.of(w), dtype=w.dtype)
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=outer or w.outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)
seen = []
for r in range(reps):
    res = P.fit(P.DenseTensor(x), w.rank, None, cfg, engine=eng)
    h = hashlib.sha256(np.array([v for rr in res.residual_history for v in rr.primal + rr.dual]).tobytes()).hexdigest()[:16]
    print(f"{name} rep {r}: rfe {res.rfe!r} residual-history {h}", flush=True)
    seen.append((res.rfe, h))
    P.solver.release_plan_cache()
    torch.cuda.empty_cache()
print(f"{name}: {'DETERMINISTIC' if len(set(seen)) == 1 else 'NOT deterministic'}", flush=True)
