"""Per-mode-update emulation of the MTTKRP engine gate (DESIGN 6b): before
every mode update the companions' negative-part ratio

    nu = max over companions m and columns r of  max_i(-F_m[i,r])+ / max_i |F_m[i,r]|

decides between the tensor-core engine (nu <= threshold) and the exact fp64
CUDA-core engine.  Two plans on the same tensor are kept in lockstep.

  python tools/cancel_probe_mode.py c4 0.05 [golden-name]
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
thr = float(sys.argv[2])
gname = sys.argv[3] if len(sys.argv) > 3 else name
w = synth.CONFIGS[name]
dseed, fseed = synth.seeds()
x = synth.generate_box(synth.SynthSpec.of(w), dtype="float32")
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                         f"fp32_{gname}.npz"))
want = float(g["fit_rfe"])
probs = {"tc": DeviceProblem(x, w.dims, w.rank, cfg, 1, engine=N.ENGINE_TCGEN05),
         "cc": DeviceProblem(x.double() if os.environ.get("EXACT", "1") == "1" else x, w.dims, w.rank, cfg, 1,
                             engine=N.ENGINE_CUDA_CORE)}
st = init_state(w.dims, w.rank, cfg, 0)
for p in probs.values():
    p.load_state(st.factors, st.aux, st.duals, st.rho)
    p.stream.synchronize()


def mirror(src, dst):
    src.stream.synchronize()
    with torch.cuda.stream(dst.stream):
        for a, b in zip(src.factors + src.aux + src.duals + src.grams, dst.factors + dst.aux + dst.duals + dst.grams):
            b.copy_(a)
        dst.colmax.copy_(src.colmax)
        dst.rho.copy_(src.rho)
        dst.norm_acc.copy_(src.norm_acc)
        dst.counters.copy_(src.counters)
    # the CUDA-core plan does not maintain the column maxima (tensor-core W scales)
    for m in range(3):
        N.check(dst.lib.ntf_colmax(dst.factors[m].data_ptr(), dst.dims[m], dst.R,
                                   dst.colmax.data_ptr() + m * dst.R * 8, dst._sh))
    dst.stream.synchronize()


def nu_of(f):
    neg = (-f).clamp_min(0).amax(dim=0)
    mx = f.abs().amax(dim=0).clamp_min(1e-300)
    return float((neg / mx).max())


used = {"tc": 0, "cc": 0}
cur = "tc"
for it in range(w.outer):
    for sw in range(w.inner):
        for mode in (1, 2, 3):
            nu = max(nu_of(probs[cur].factors[m]) for m in range(3) if m != mode - 1)
            eng = "cc" if nu > thr else "tc"
            if eng == "tc" or it < 1:
                nus = [nu_of(probs[cur].factors[m]) for m in range(3)]
                print(f"  it {it} sweep {sw} mode {mode}: nu per factor {nus} -> {eng}", flush=True)
            if eng != cur:
                mirror(probs[cur], probs[eng])
                cur = eng
            probs[cur].mode_update(mode, sw == w.inner - 1)
            probs[cur].stream.synchronize()
            used[cur] += 1
    probs[cur].finalize()
    probs[cur].check_status()
    print(f"{name} it {it}: mode updates so far tc {used['tc']} cc {used['cc']}", flush=True)
aux = probs[cur].aux
x_norm = float(torch.linalg.norm(x.double()))
_, err_sq = probs[cur].final_sq_error(aux)
rfe = float(np.sqrt(err_sq)) / x_norm
print(f"{name} per-mode gate nu > {thr}: mode updates tc {used['tc']} cc {used['cc']}; rfe {rfe:.12f} "
      f"reference {want:.12f} rel {abs(rfe - want) / want:.2e}", flush=True)
