"""Cancellation probe for the tensor-core MTTKRP (DESIGN 6b).

Runs a BASELINE fp32 config outer iteration by outer iteration, printing per
iteration the cancellation index of the working factors

    kappa = max over modes n and columns r of  prod_{m != n} sum_i |F_m[i,r]| / |sum_i F_m[i,r]|

and emulates the engine gate: an iteration whose entering kappa exceeds the
threshold runs on the exact fp64 CUDA-core engine, the others on tcgen05.

  python tools/cancel_probe.py c4 [threshold|inf|0] [golden-name]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import _native as N
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem
from paper_1409_2383_b200.solver import init_state

name = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else float("inf")
gname = sys.argv[3] if len(sys.argv) > 3 else name
w = synth.CONFIGS[name]
dseed, fseed = synth.seeds()
x = synth.generate_box(synth.SynthSpec.of(w), dtype="float32")
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)
want = None
gp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                  f"fp32_{gname}.npz")
if os.path.exists(gp):
    g = np.load(gp)
    want = float(g["fit_rfe"])
    assert float(g["rho0"]) == rho0, (float(g["rho0"]), rho0)

probs = {"tc": DeviceProblem(x, w.dims, w.rank, cfg, 1, engine=N.ENGINE_TCGEN05)}
if thr != float("inf"):
    probs["cc"] = DeviceProblem(x, w.dims, w.rank, cfg, 1, engine=N.ENGINE_CUDA_CORE)


def kappa(factors):
    q = []
    for f in factors:
        s = np.abs(f.sum(axis=0))
        a = np.abs(f).sum(axis=0)
        # (columns decayed to denormals count as dead: s / max(a, 1e-300) once reported ~1e9 for them)
        q.append(np.where(a > 1e-290, s / np.maximum(a, 1e-290), 1.0))
    worst = 1.0
    for n in range(len(factors)):
        prod = np.ones_like(q[0])
        for m in range(len(factors)):
            if m != n:
                prod = prod * q[m]
        worst = max(worst, float(1.0 / max(prod.min(), 1e-300)))
    nu = max(float((np.maximum(-f, 0).max(axis=0) / np.maximum(np.abs(f).max(axis=0), 1e-300)).max())
             for f in factors)
    eta = max(float((np.minimum(f, 0) ** 2).sum() / max((f ** 2).sum(), 1e-300)) for f in factors)
    etac = max(float(((np.minimum(f, 0) ** 2).sum(axis=0) / np.maximum((f ** 2).sum(axis=0), 1e-300)).max())
               for f in factors)
    return worst, nu, eta, etac


st = init_state(w.dims, w.rank, cfg, 0)
state = (st.factors, st.aux, st.duals, st.rho)
cur = None
used = {"tc": 0, "cc": 0}
x_norm = float(torch.linalg.norm(x.double()))
for it in range(w.outer):
    k, nu, eta, etac = kappa(state[0])
    eng = "cc" if k > thr else "tc"
    if eng != cur:
        probs[eng].load_state(*state)
        cur = eng
    probs[eng].run(1)
    probs[eng].check_status()
    state = probs[eng].read_state()
    used[eng] += 1
    print(f"{name} it {it:3d}: entering kappa {k:9.3f} negmax {nu:6.3f} eta {eta:.2e} eta_col {etac:.2e} engine {eng} rho {state[3][0]:.4g}", flush=True)
k, nu, eta, etac = kappa(state[0])
_, err_sq = probs[cur].final_sq_error([torch.from_numpy(a).cuda() for a in state[1]])
rfe = float(np.sqrt(err_sq)) / x_norm
msg = f"{name} thr {thr}: final kappa {k:.3f}; iterations tc {used['tc']} cc {used['cc']}; rfe {rfe:.12f}"
if want is not None:
    msg += f" reference {want:.12f} rel {abs(rfe - want) / want:.2e}"
print(msg, flush=True)
