"""Bring-up check of the tcgen05 MTTKRP engine against the fp64 oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1409_2383_b200 as P
from oracle import ntf_oracle as O

def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

rng = np.random.default_rng(3)
for dims, R in [((40, 48, 64), 8), ((130, 96, 200), 20), ((64, 64, 64), 32), ((300, 17, 72), 50), ((128, 128, 128), 16)]:
    x = rng.random(dims, dtype=np.float32) - np.float32(0.1)
    f = [rng.random((d, R)) for d in dims]
    t = O.OracleTensor(x.astype(np.float64))
    out = []
    for mode in (1, 2, 3):
        want = O.mttkrp(t, f, mode)
        try:
            got = P.mttkrp_factors(P.DenseTensor(x), f, mode, engine="tcgen05")
            cc = P.mttkrp_factors(P.DenseTensor(x), f, mode, engine="cuda_core")
            out.append(f"m{mode}: tc {rel(got, want):.2e} cc {rel(cc, want):.2e}")
        except Exception as e:
            out.append(f"m{mode}: ERR {type(e).__name__}: {str(e)[:120]}")
    print(dims, R, " | ".join(out), flush=True)
