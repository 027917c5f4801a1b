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
cfg = P.SolverConfig(seed=fseed, eps_abs=0, eps_rel=0, n_max=8, max_restarts=0, inner_sweeps=10, rho_init=rho0)
st = P.init_state(w.dims, w.rank, cfg)
probs = {e: DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=8, engine=P.solver._engine_code(e)) for e in ("cuda_core", "tcgen05")}
for p in probs.values():
    p.load_state(st.factors, st.aux, st.duals, st.rho)
for sw in range(10):
    for mode in (1, 2, 3):
        out = {}
        for e, p in probs.items():
            p.mode_update(mode, sw == 9)
            p.stream.synchronize()
            out[e] = (p.factors[mode - 1].cpu().numpy(), p.grams[mode - 1].cpu().numpy(), p.counters.cpu().numpy().tolist())
        a, b = out["cuda_core"], out["tcgen05"]
        print(sw, mode, "rel", np.linalg.norm(a[0] - b[0]) / np.linalg.norm(a[0]), "gram rel", np.linalg.norm(a[1] - b[1]) / np.linalg.norm(a[1]), a[2], b[2], "colmin", np.abs(b[0]).max(axis=0).min(), flush=True)
        # resync TC state to CC state to isolate single-step errors
        tp = probs["tcgen05"]
        tp.factors[mode - 1].copy_(probs["cuda_core"].factors[mode - 1])
        tp.grams[mode - 1].copy_(probs["cuda_core"].grams[mode - 1])
