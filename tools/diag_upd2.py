import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_1409_2383_b200 as P
from paper_1409_2383_b200.engine import DeviceProblem, device_tensor
from oracle import ntf_oracle as O
from conftest import load_golden
g = load_golden("small_fits.npz")
x = g["bigrho_x"]; R = 5
cfg = P.SolverConfig(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=15, max_restarts=0, rho_init=300.0, inner_sweeps=4)
t = P.DenseTensor(x); xd = device_tensor(t)
prob = DeviceProblem(xd, t.dims, R, cfg, history_capacity=4)
st = P.init_state(t.dims, R, cfg)
prob.load_state(st.factors, st.aux, st.duals, st.rho)
f = [a.copy() for a in st.factors]
ot = O.OracleTensor(x)
for sw in range(2):
    for mode in (1, 2, 3):
        prob.mode_update(mode, False); prob.stream.synchronize()
        f[mode-1] = O.factor_update(ot, f, st.aux[mode-1], st.duals[mode-1], 300.0, mode)
        got = prob.factors[mode-1].cpu().numpy()
        G = prob.grams[mode-1].cpu().numpy()
        print(sw, mode, np.linalg.norm(got - f[mode-1]) / np.linalg.norm(f[mode-1]), "gram", np.linalg.norm(G - f[mode-1].T @ f[mode-1]) / np.linalg.norm(f[mode-1].T @ f[mode-1]))
