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
print("xmax", np.abs(xh).max(), "xmin", xh.min())
x = torch.from_numpy(xh).cuda()
cfg = P.SolverConfig(seed=fseed, eps_abs=0, eps_rel=0, n_max=8, max_restarts=0, inner_sweeps=2, rho_init=1.0)
st = P.init_state(w.dims, w.rank, cfg)
f = [torch.from_numpy(v).cuda() for v in st.factors]
for mode in (1, 2, 3):
    a = mttkrp_device(x, f, mode, 1).cpu().numpy()
    b = mttkrp_device(x, f, mode, 2).cpu().numpy()
    print("standalone mode", mode, np.isfinite(b).all(), np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-300), np.linalg.norm(a))
for eng in ("cuda_core", "tcgen05"):
    prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=8, engine=P.solver._engine_code(eng))
    prob.load_state(st.factors, st.aux, st.duals, st.rho)
    for mode in (1, 2, 3):
        prob.mode_update(mode, False)
        prob.stream.synchronize()
        fm = prob.factors[mode - 1].cpu().numpy()
        print(eng, mode, np.isfinite(fm).all(), np.linalg.norm(fm), prob.counters.cpu().numpy().tolist(), flush=True)
    prob.close()
