"""Run a few eager outer iterations of a BASELINE config (ncu target)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa: F401,E402  (NTF_VARIANT_LIB)
import numpy as np
import torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--engine", default="auto")
a = ap.parse_args()
w = synth.CONFIGS[a.config]
dt = torch.float32 if w.dtype == "float32" else torch.float64
x = torch.rand(w.dims, dtype=dt, device="cuda")
cfg = P.SolverConfig(seed=1, eps_abs=0, eps_rel=0, n_max=a.iters + 2, max_restarts=0,
                     inner_sweeps=w.inner)
prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=a.iters + 2,
                     engine=P.solver._engine_code(a.engine))
st = P.init_state(w.dims, w.rank, cfg)
prob.load_state(st.factors, st.aux, st.duals, st.rho)
prob.run(a.iters, use_graph=a.graph)
torch.cuda.synchronize()
print("iterations", prob.check_status())
