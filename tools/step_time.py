"""ms per outer iteration (graph replay, no instrumentation) of a BASELINE
config, optionally with a diagnostic variant library (NTF_VARIANT_LIB).

  python tools/step_time.py c2 [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _variant  # noqa: F401,E402
import torch

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = synth.CONFIGS[name]
dseed, fseed = synth.seeds()
x = synth.generate_box(synth.SynthSpec.of(w), dtype=w.dtype)
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=steps + 10, max_restarts=0,
                     inner_sweeps=w.inner, rho_init=rho0)
prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=steps + 10)
st = P.init_state(w.dims, w.rank, cfg)
prob.load_state(st.factors, st.aux, st.duals, st.rho)
for _ in range(5):
    prob.step()
prob.stream.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(prob.stream)
prob.run(steps)
e1.record(prob.stream)
torch.cuda.synchronize()
plain = e0.elapsed_time(e1) / steps
prob.set_timing(True)
prob.run(1)
e0.record(prob.stream)
prob.run(1)
e1.record(prob.stream)
torch.cuda.synchronize()
kt = prob.kernel_times()
prob.set_timing(False)
print(f"{name} {os.environ.get('NTF_TC_CG', 'default')}: {plain:.4f} ms/step; instrumented step "
      f"{e0.elapsed_time(e1):.4f} ms, mttkrp {kt[:, 0].mean() * 1e3:.2f} us, row update {kt[:, 1].mean() * 1e3:.2f} us "
      f"(x{len(kt)})", flush=True)
