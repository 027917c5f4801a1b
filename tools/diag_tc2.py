"""Replicate bench.py's plan usage with each engine / graph / timing combination."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dseed, fseed = synth.seeds()
xh, _ = synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=np.float32)
x = torch.from_numpy(xh).cuda()
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
for eng in ("cuda_core", "tcgen05"):
    for graph in (False, True):
        for timing in (False, True):
            cfg = P.SolverConfig(seed=fseed, eps_abs=0, eps_rel=0, n_max=8, max_restarts=0,
                                 inner_sweeps=w.inner, rho_init=rho0)
            prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=8, engine=P.solver._engine_code(eng))
            st = P.init_state(w.dims, w.rank, cfg)
            prob.load_state(st.factors, st.aux, st.duals, st.rho)
            if timing:
                prob.set_timing(True)
            msg = []
            for it in range(3):
                prob.run(1, use_graph=graph)
                c = prob.counters_host()
                msg.append(f"{c.tolist()}")
            r, rh = prob.histories(3)
            print(eng, "graph" if graph else "eager", "timing" if timing else "", msg, r[:, 0].tolist(), flush=True)
            prob.close()
