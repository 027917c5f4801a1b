"""Per-CTA timeline of one tcgen05 MTTKRP launch (diagnostic build only:
NTF_VARIANT_LIB=<NTF_DIAG variant> NTF_TC_DEBUG=256): globaltimer stamps at
kernel entry, after the prologue, at the end of each role's loop and at the
TMEM release, relative to the first CTA's entry.

  NTF_VARIANT_LIB=paper_1409_2383_b200/var_diag.so NTF_TC_DEBUG=256 python tools/tc_timeline.py c2 [mode]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa: F401,E402
import numpy as np
import torch

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import _native, synth
from paper_1409_2383_b200.engine import DeviceProblem

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = synth.CONFIGS[name]
x = torch.rand(w.dims, dtype=torch.float32, device="cuda")
cfg = P.SolverConfig(seed=1, eps_abs=0, eps_rel=0, n_max=4, max_restarts=0, inner_sweeps=w.inner)
prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=4)
st = P.init_state(w.dims, w.rank, cfg)
prob.load_state(st.factors, st.aux, st.duals, st.rho)
if os.environ.get("NTF_TIMELINE_GRAPH"):  # graph replays (PDL chain): the stamps are the last launch's, mode 3
    prob.run(4)
    mode = 3
else:
    for rep in range(3):
        for m in (1, 2, 3):
            prob.mode_update(m, False)
    prob.mode_update(mode, False)
torch.cuda.synchronize()
lib = _native.load()
n = 160
buf = (ctypes.c_ulonglong * (8 * n))()
lib.ntf_debug_tc_times.restype = ctypes.c_int
got = lib.ntf_debug_tc_times(buf, n)
t = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8)[:got].astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = lambda c: (t[:, c] - t0) / 1e3  # us
units = t[:, 7] & 0xFFFF
kb = t[:, 7] >> 32
print(f"{name} mode {mode}: {len(t)} CTAs, units/CTA {units.min()}..{units.max()}, KiB/CTA {kb.min()}..{kb.max()}")
for label, c in (("entry", 0), ("prologue done", 1), ("producer done", 2), ("issuer 1 done", 3), ("W loader done", 4),
                 ("issuer 3 done", 5), ("TMEM released", 6)):
    v = rel(c)
    v = v[t[:, c] > 0]
    if len(v):
        print(f"  {label:16s} min {v.min():7.2f}  median {np.median(v):7.2f}  max {v.max():7.2f} us")
print(f"  prologue (ready - entry): median {np.median((t[:, 1] - t[:, 0]) / 1e3):.2f} us; "
      f"tail (release - last issuer): median {np.median((t[:, 6] - np.maximum(t[:, 3], t[:, 5])) / 1e3):.2f} us")
if os.environ.get("NTF_TIMELINE_ROWS"):
    order = np.argsort(t[:, 6])
    print("  cta  smid  entry   ready  prod_end  mma_end  release  units   KiB   GB/s")
    for i in list(order[:8]) + list(order[-16:]):
        smid = (t[i, 7] >> 16) & 0xFFFF
        dur = (t[i, 6] - t[i, 0]) / 1e3
        print(f"  {i:4d} {smid:4d} {rel(0)[i]:7.2f} {rel(1)[i]:7.2f} {rel(2)[i]:8.2f} {max(rel(3)[i], rel(5)[i]):8.2f} "
              f"{rel(6)[i]:8.2f} {units[i]:5d} {kb[i]:6d} {kb[i] * 1024 / dur / 1e3:6.1f}")
