import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200.engine import DeviceProblem, device_tensor
from oracle import ntf_oracle as O
from conftest import load_golden
g = load_golden("small_fits.npz")
x = g["bigrho_x"]
R = 5
cfg = P.SolverConfig(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=15, max_restarts=0, rho_init=300.0, inner_sweeps=4)
t = P.DenseTensor(x)
xd = device_tensor(t)
prob = DeviceProblem(xd, t.dims, R, cfg, history_capacity=4)
st = P.init_state(t.dims, R, cfg)
prob.load_state(st.factors, st.aux, st.duals, st.rho)
prob.mode_update(1, False)
prob.stream.synchronize()
got = prob.factors[0].cpu().numpy()
want = O.factor_update(O.OracleTensor(x), st.factors, st.aux[0], st.duals[0], 300.0, 1)
print("got", got[:2]); print("want", want[:2]); print("status", prob.counters.cpu().numpy())
print("colmax", prob.colmax.cpu().numpy()); print("gram0", prob.grams[0].cpu().numpy()[:2])
for sw in range(4):
    for mode in (1, 2, 3):
        prob.mode_update(mode, sw == 3)
        prob.stream.synchronize()
        print(sw, mode, np.abs(prob.factors[mode-1].cpu().numpy()).max(), prob.counters.cpu().numpy(), np.abs(prob.aux[mode-1].cpu().numpy()).max(), prob.norm_acc.cpu().numpy()[5*(mode-1):5*mode])
