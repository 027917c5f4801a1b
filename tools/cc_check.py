import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200.engine import mttkrp_device
E = P.solver._engine_code
for dims, R in [((100, 100, 100), 50), ((200, 180, 160), 20), ((300, 300, 300), 50), ((1000, 1000, 1000), 50), ((400,400,400),100)]:
    torch.manual_seed(0)
    x = torch.rand(dims, dtype=torch.float32, device="cuda")
    f = [torch.rand((d, R), dtype=torch.float64, device="cuda") for d in dims]
    x64 = x.double()
    for mode in (1, 2, 3):
        a = mttkrp_device(x, f, mode, E("cuda_core"))
        b = mttkrp_device(x64, f, mode, E("cuda_core"))
        c = mttkrp_device(x, f, mode, E("tcgen05"))
        print(dims, R, mode, "cc32 vs cc64", float(torch.linalg.norm(a - b) / torch.linalg.norm(b)),
              "tc vs cc64", float(torch.linalg.norm(c - b) / torch.linalg.norm(b)), flush=True)
