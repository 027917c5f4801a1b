"""Find where the tcgen05 plan path goes wrong at a BASELINE size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem, mttkrp_device
from oracle import ntf_oracle as O

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = synth.CONFIGS[cfgname]
dims = tuple(int(d) for d in (sys.argv[2].split(",") if len(sys.argv) > 2 else w.dims))
R = w.rank
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.random(dims, dtype=np.float32)).cuda()
cfg = P.SolverConfig(seed=1, eps_abs=0, eps_rel=0, n_max=4, max_restarts=0, inner_sweeps=2)
for eng in ("cuda_core", "tcgen05"):
    prob = DeviceProblem(x, dims, R, cfg, history_capacity=4, engine=P.solver._engine_code(eng))
    st = P.init_state(dims, R, cfg)
    st.factors[0] = rng.random((dims[0], R))
    prob.load_state(st.factors, st.aux, st.duals, st.rho)
    for mode in (1, 2, 3):
        prob.mode_update(mode, False)
        prob.stream.synchronize()
        f = prob.factors[mode - 1].cpu().numpy()
        g = prob.grams[mode - 1].cpu().numpy()
        print(eng, "mode", mode, "finite", np.isfinite(f).all(), "norm", np.linalg.norm(f), "gram", np.linalg.norm(g),
              "status", prob.counters.cpu().numpy().tolist(), flush=True)
    prob.close()
