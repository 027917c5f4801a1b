"""Per-SM stream rate of the tcgen05 MTTKRP (NTF_TC_DEBUG=256): is the
X-loop spread a fixed property of the SM (GPC/die placement) or run noise?

  NTF_TC_DEBUG=256 python tools/tc_smid.py c2 [reps]
Prints, per mode, the correlation across repetitions of each SM's rate
(KiB streamed / X-loop duration), and the rate spread; writes the raw table
to gpurun_out/tc_smid_<cfg>.npy ([mode, rep, cta, (smid, kib, ready, xend)])."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1409_2383_b200 import synth, _native
from paper_1409_2383_b200.engine import mttkrp_device

assert int(os.environ.get("NTF_TC_DEBUG", "0")) & 256
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = synth.CONFIGS[cfg]
x = torch.rand(w.dims, dtype=torch.float32, device="cuda")
f = [torch.rand((d, w.rank), dtype=torch.float64, device="cuda") for d in w.dims]
fn = _native.load().ntf_debug_tc_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1024, 8), dtype=np.uint64)
seen = 0
out = []
for mode in (1, 2, 3):
    rows = []
    for rep in range(reps + 1):
        mttkrp_device(x, f, mode)
        torch.cuda.synchronize()
        fn(buf.ctypes.data, 1024)
        ts = buf.astype(np.int64)
        ok = ts[:, 0] > seen
        seen = int(ts[:, [0, 6]].max())
        t = ts[ok]
        if rep == 0:
            continue  # warm-up
        t0 = t[:, 0].min()
        smid = (t[:, 7] >> 16) & 0xFFFF
        kib = t[:, 7] >> 32
        rows.append(np.stack([smid, kib, t[:, 1] - t0, t[:, 2] - t0], 1))
    n = min(len(r) for r in rows)
    rows = np.stack([r[:n] for r in rows])
    out.append(rows)
    rate = {}  # smid -> [rates]
    for r in rows:
        for sm, kb, rd, xe in r:
            rate.setdefault(int(sm), []).append(kb / max(xe - rd, 1) * 1.024)  # GB/s per SM
    sms = sorted(k for k, v in rate.items() if len(v) >= 2)
    a = np.array([[rate[s][0], rate[s][1]] for s in sms])
    m = np.array([np.mean(rate[s]) for s in sms])
    print(f"{cfg} mode {mode}: SMs {len(sms)} rate GB/s per SM med {np.median(m):.1f} "
          f"min {m.min():.1f} max {m.max():.1f}; corr(rep0, rep1) {np.corrcoef(a[:, 0], a[:, 1])[0, 1]:.2f}; "
          f"slowest SMs {[sms[i] for i in np.argsort(m)[:8]]}", flush=True)
    # per-CTA: is xend explained by bytes?
    r = rows[0]
    print(f"   xend spread {np.percentile(r[:,3],50)/1e3:.1f}/{r[:,3].max()/1e3:.1f} us; "
          f"corr(kib, xend) {np.corrcoef(r[:,1], r[:,3])[0,1]:.2f}", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
acc = {}
for rows in out:
    for r in rows:
        for sm, kb, rd, xe in r:
            acc.setdefault(int(sm), []).append(kb * 1024 / max(xe - rd, 1))
med = float(np.median([np.mean(v) for v in acc.values()]))
with open(f"gpurun_out/smw_{cfg}.txt", "w") as fh:
    for s_ in range(nsm):
        fh.write(f"{(np.mean(acc[s_]) if s_ in acc else med) / med:.4f}\n")
print(f"wrote gpurun_out/smw_{cfg}.txt ({len(acc)} SMs measured of {nsm})")
np.save(f"gpurun_out/tc_smid_{cfg}.npy", np.array([np.asarray(o, dtype=np.int64) for o in out] + [None], dtype=object)[:-1], allow_pickle=True)
