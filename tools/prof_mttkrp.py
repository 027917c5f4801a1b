"""Time the dense MTTKRP alone (each mode) at a BASELINE config; ncu target."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa: F401,E402  (NTF_VARIANT_LIB)
import numpy as np
import torch
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import mttkrp_device
from paper_1409_2383_b200.solver import _engine_code

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--engine", default="auto")
ap.add_argument("--modes", default="123")
a = ap.parse_args()
w = synth.CONFIGS[a.config]
dt = torch.float32 if w.dtype == "float32" else torch.float64
x = torch.rand(w.dims, dtype=dt, device="cuda")
f = [torch.rand((d, w.rank), dtype=torch.float64, device="cuda") for d in w.dims]
eng = _engine_code(a.engine)
s = torch.cuda.current_stream()
for mode in map(int, a.modes):
    for _ in range(2):
        mttkrp_device(x, f, mode, eng)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        mttkrp_device(x, f, mode, eng)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    b = x.numel() * x.element_size() + 8 * w.rank * sum(w.dims)
    print(f"{a.config} mode {mode}: {ms*1e3:.1f} us/call (incl. reduce+alloc)  {b/ms/1e6:.0f} GB/s")
