import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem, mttkrp_device

w = synth.CONFIGS["c2"]
dseed, fseed = synth.seeds()
xh, _ = synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=np.float32)
x = torch.from_numpy(xh).cuda()
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0, eps_rel=0, n_max=8, max_restarts=0, inner_sweeps=2, rho_init=rho0)
st = P.init_state(w.dims, w.rank, cfg)
for eng in ("cuda_core", "tcgen05"):
    prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=8, engine=P.solver._engine_code(eng))
    prob.load_state(st.factors, st.aux, st.duals, st.rho)
    for sw in range(2):
        for mode in (1, 2, 3):
            prob.mode_update(mode, sw == 1)
            prob.stream.synchronize()
            fm = prob.factors[mode - 1].cpu().numpy()
            print(eng, sw, mode, np.isfinite(fm).all(), np.linalg.norm(fm), np.abs(fm).max(axis=0)[:4], prob.counters.cpu().numpy().tolist(), flush=True)
    prob.close()
