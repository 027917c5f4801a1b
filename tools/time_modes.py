"""Per-kernel MTTKRP / row-update times of one sweep set (no finalize, so
debug variants with garbage math cannot trip the stop flag)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa: F401,E402  (NTF_VARIANT_LIB)
import numpy as np
import torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
eng = sys.argv[2] if len(sys.argv) > 2 else "auto"
if cfgname == "custom":  # time_modes.py custom ENGINE I J K R INNER [DTYPE]
    I, J, K, R, inner = (int(v) for v in sys.argv[3:8])
    dtype = sys.argv[8] if len(sys.argv) > 8 else "float32"
    w = synth.Workload("custom", (I, J, K), R, dtype, 20.0, inner, 1)
else:
    w = synth.CONFIGS[cfgname]
dt = torch.float32 if w.dtype == "float32" else torch.float64
x = torch.rand(w.dims, dtype=dt, device="cuda")
cfg = P.SolverConfig(seed=1, eps_abs=0, eps_rel=0, n_max=4, max_restarts=0, inner_sweeps=w.inner)
prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=4, engine=P.solver._engine_code(eng))
st = P.init_state(w.dims, w.rank, cfg)
prob.load_state(st.factors, st.aux, st.duals, st.rho)
prob.set_timing(True)
for rep in range(2):
    for sw in range(w.inner):
        for mode in (1, 2, 3):
            prob.mode_update(mode, sw == w.inner - 1)
kt = prob.kernel_times()
mt = kt[:, 0].reshape(w.inner, 3).mean(axis=0)
ut = kt[:, 1].reshape(w.inner, 3).mean(axis=0)
sx = x.element_size()
gbs = [(sx * x.numel() + 8 * w.rank * sum(w.dims)) / (t * 1e-3) / 1e9 for t in mt]
print(cfgname, eng, os.environ.get("NTF_TC_DEBUG", "0"), "mttkrp_us", np.round(mt * 1e3, 1).tolist(),
      "GB/s", np.round(gbs).tolist(), "update_us", np.round(ut * 1e3, 1).tolist(), flush=True)
