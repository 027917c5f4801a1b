"""Per-CTA globaltimer breakdown of the tcgen05 MTTKRP (NTF_TC_DEBUG=256).

  NTF_TC_DEBUG=256 python tools/tc_times.py c2 [modes]

For each mode: launch skew (entry spread), prologue (ready - entry), each
role's loop end and the CTA exit, relative to the earliest CTA entry (us)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1409_2383_b200 import synth, _native
from paper_1409_2383_b200.engine import mttkrp_device

assert int(os.environ.get("NTF_TC_DEBUG", "0")) & 256
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "custom":  # tc_times.py custom I J K R [modes]
    I, J, K, R = (int(v) for v in sys.argv[2:6])
    w = synth.Workload("custom", (I, J, K), R, "float32", 20.0, 1, 1)
    modes = sys.argv[6] if len(sys.argv) > 6 else "123"
else:
    modes = sys.argv[2] if len(sys.argv) > 2 else "123"
    w = synth.CONFIGS[cfg]
x = torch.rand(w.dims, dtype=torch.float32, device="cuda")
f = [torch.rand((d, w.rank), dtype=torch.float64, device="cuda") for d in w.dims]
lib = _native.load()
fn = lib.ntf_debug_tc_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1024, 8), dtype=np.uint64)
seen = 0
for mode in map(int, modes):
    for rep in range(3):
        mttkrp_device(x, f, mode)
        torch.cuda.synchronize()
        fn(buf.ctypes.data, 1024)
        ts = buf.astype(np.int64)
        ok = ts[:, 0] > seen
        seen = int(ts[:, [0, 6]].max())
    t = ts[ok]
    t0 = t[:, 0].min()
    rel = (t[:, :7] - t0) / 1e3
    units = t[:, 7]
    q = lambda v: f"{np.median(v):6.1f}/{v.max():6.1f}"
    print(f"{cfg} mode {mode}: ctas {len(t)} units {units.min()}-{units.max()} | entry {q(rel[:,0])} "
          f"ready {q(rel[:,1])} | loop end (med/max) X {q(rel[:,2])} MMA {q(rel[:,3])} "
          f"Fhi {q(rel[:,4])} MMA2 {q(rel[:,5])} | exit {q(rel[:,6])} us", flush=True)
