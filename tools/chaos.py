"""Sensitivity of a BASELINE config's fit to tiny perturbations of the
initial factors, per engine: the spread of the final RFE says how far apart
two correct implementations (different but equally exact summation orders)
can land, i.e. what a final-RFE tolerance can resolve.

  python tools/chaos.py c5 [cuda_core tcgen05]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.engine import DeviceProblem, sq_error

name = sys.argv[1]
engines = sys.argv[2:] or ["cuda_core", "tcgen05"]
w = synth.CONFIGS[name]
dseed, fseed = synth.seeds()
x = synth.generate_box(synth.SynthSpec.of(w), dtype=w.dtype)
rho0 = synth.initial_rho_trace(w.dims, w.rank, fseed)
xn = math.sqrt(float(sq_error(x)[0].item()))
for rho_init in (rho0, 1.0):
    cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=w.outer, max_restarts=0,
                         inner_sweeps=w.inner, rho_init=rho_init)
    for eng in engines:
        prob = DeviceProblem(x, w.dims, w.rank, cfg, history_capacity=w.outer,
                             engine=P.solver._engine_code(eng))
        out = []
        for eps in (0.0, 1e-15, 1e-12, 1e-9):
            st = P.init_state(w.dims, w.rank, cfg)
            rng = np.random.default_rng(3)
            f = [a * (1.0 + eps * rng.standard_normal(a.shape)) for a in st.factors]
            prob.load_state(f, st.aux, st.duals, st.rho)
            prob.run(w.outer)
            prob.check_status()
            _, _, aux_unused, _ = None, None, None, None
            fac, aux, duals, rho = prob.read_state()
            err = float(sq_error(x, aux)[1].item())
            out.append(math.sqrt(err) / xn)
        base = out[0]
        print(f"{name} rho0={rho_init:.6g} {eng}: rfe {base:.12f}; perturbed initial factors "
              + " ".join(f"{e:.0e}->{abs(v - base) / base:.2e}" for e, v in zip((1e-15, 1e-12, 1e-9), out[1:])),
              flush=True)
        prob.close()
        del prob
        torch.cuda.empty_cache()
