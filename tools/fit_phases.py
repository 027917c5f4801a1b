"""Wall-clock phases of one fit() from pinned host memory at a BASELINE config
(what bench.py's e2e leg times as a whole): upload, norm, plan creation (block
images), state upload, iterations, read-back, final RFE, teardown.

  python tools/fit_phases.py c5 [calls]
"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem, device_tensor, order3_view, sq_error
from paper_1409_2383_b200.solver import init_state

name = sys.argv[1]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = synth.CONFIGS[name]
dseed, fseed = synth.seeds()
xd = synth.generate_box(synth.SynthSpec.of(w), dtype="float32")
host = torch.empty(xd.shape, dtype=xd.dtype, pin_memory=True)
host.copy_(xd)
del xd
torch.cuda.synchronize()
torch.cuda.empty_cache()
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)


def tick(label, t0, out):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out.append((label, t1 - t0))
    return t1


for c in range(calls):
    ph = []
    t0 = time.perf_counter()
    t = P.DenseTensor(host)
    x = device_tensor(t)
    t1 = tick("H2D", t0, ph)
    x_norm = math.sqrt(float(sq_error(order3_view(x)[0])[0].item()))
    t1 = tick("norm", t1, ph)
    prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=cfg.n_max)
    t1 = tick("plan", t1, ph)
    st = init_state(w.dims, w.rank, cfg, 0)
    t1 = tick("init_state(host)", t1, ph)
    prob.load_state(st.factors, st.aux, st.duals, st.rho)
    t1 = tick("load_state", t1, ph)
    prob.run(cfg.n_max)
    prob.check_status()
    t1 = tick("iterations", t1, ph)
    prob.histories(cfg.n_max)
    state = prob.read_state()
    t1 = tick("read-back", t1, ph)
    _, err = prob.final_sq_error(state[1])
    t1 = tick("final RFE", t1, ph)
    prob.close()
    del prob, x, t
    t1 = tick("teardown", t1, ph)
    total = t1 - t0
    print(f"{name} call {c}: total {total * 1e3:.1f} ms | " +
          " | ".join(f"{k} {v * 1e3:.1f}" for k, v in ph), flush=True)
t0 = time.perf_counter()
res = P.fit(P.DenseTensor(host), w.rank, None, cfg)
torch.cuda.synchronize()
print(f"{name} fit(): {(time.perf_counter() - t0) * 1e3:.1f} ms, rfe {res.rfe:.12f}")
