"""Phase timing of one public fit() call (c2) to explain the e2e number."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth, solver
from paper_1409_2383_b200.engine import DeviceProblem, device_tensor, sq_error

w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dseed, fseed = synth.seeds()
xh = torch.empty(w.dims, dtype=torch.float32, pin_memory=True)
synth.generate(w.dims, w.rank, w.snr_db, dseed, w.zero_frac, dtype=np.float32, out=xh.numpy())
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)
t = P.DenseTensor(xh)
for rep in range(int(os.environ.get("REPS", "3"))):
    T = {}
    def mark(k, t0):
        torch.cuda.synchronize(); T[k] = time.perf_counter() - t0; return time.perf_counter()
    t0 = time.perf_counter()
    x = device_tensor(P.tensors.as_dense(t), None); t0 = mark("h2d", t0)
    xn = float(sq_error(x)[0].item()) ** 0.5; t0 = mark("norm", t0)
    prob = DeviceProblem(x, t.dims, w.rank, cfg, history_capacity=cfg.n_max); t0 = mark("plan", t0)
    st = P.init_state(t.dims, w.rank, cfg); prob.load_state(st.factors, st.aux, st.duals, st.rho); t0 = mark("load", t0)
    prob.run(1); t0 = mark("run1(capture)", t0)
    prob.run(w.outer - 1); t0 = mark(f"run{w.outer-1}", t0)
    done, stopped = prob.check_status(); r, rh = prob.histories(done); t0 = mark("hist", t0)
    f, a, y, rho = prob.read_state(); t0 = mark("read", t0)
    _, e = prob.final_sq_error(a); t0 = mark("rfe", t0)
    prob.close(); t0 = mark("close", t0)
    print({k: round(v * 1e3, 2) for k, v in T.items()}, flush=True)
