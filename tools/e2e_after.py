"""Does a previous solver plan in the process slow a later fit()? (bench e2e)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem

w = synth.CONFIGS["c2"]
dseed, fseed = synth.seeds()
xh = torch.empty(w.dims, dtype=torch.float32, pin_memory=True)
synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=np.float32, out=xh.numpy())
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)

def timed_fits(tag, n=3):
    P.fit(P.DenseTensor(xh), w.rank, None, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        P.fit(P.DenseTensor(xh), w.rank, None, cfg)
    torch.cuda.synchronize()
    print(tag, "ms/fit", (time.perf_counter() - t0) / n * 1e3, flush=True)

timed_fits("fresh")
mode = sys.argv[1] if len(sys.argv) > 1 else "timing"
x = xh.to("cuda")
cap = 520
cfg2 = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=cap, max_restarts=0,
                      inner_sweeps=w.inner, rho_init=rho0)
prob = DeviceProblem(x, w.dims, w.rank, cfg2, history_capacity=cap)
st = P.init_state(w.dims, w.rank, cfg2)
prob.load_state(st.factors, st.aux, st.duals, st.rho)
for i in range(405):
    if mode == "timing":
        prob.set_timing(i == 404 or i == 3)
    prob.step()
prob.stream.synchronize()
timed_fits("with live plan")
prob.close()
timed_fits("after close")
del prob, x
torch.cuda.empty_cache()
timed_fits("after free")
