"""Per-iteration GPU vs oracle deviation for a constraints fixture case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1409_2383_b200 as P
from oracle import ntf_oracle as O
from conftest import CONSTRAINT_CASES, load_golden, rel

name = sys.argv[1] if len(sys.argv) > 1 else "cardall"
g = load_golden("constraints.npz")
specs = [str(s) for s in g[f"{name}_specs"]]
x = g[f"{name}_x"]
R = int(g[f"{name}_rank"])
kw = dict(CONSTRAINT_CASES[name])
for n_max in range(1, kw["n_max"] + 1):
    kw2 = dict(kw, n_max=n_max)
    got = P.fit(x, R, [P.ConstraintSpec.parse(s) for s in specs], P.SolverConfig(**kw2))
    want = O.fit(x, R, O.Config(**kw2), specs)
    fa = [rel(got.factor_history[-1][m], want.factor_history[-1][m]) for m in range(3)]
    aa = [rel(got.model.factors[m], want.factors[m]) for m in range(3)]
    rho_g = got.state.rho if hasattr(got, "state") and got.state is not None else None
    print(n_max, "F", ["%.1e" % v for v in fa], "aux", ["%.1e" % v for v in aa],
          "rho", rho_g, want.state.rho, "prim", got.residual_history[-1].primal, want.residual_history[-1][0])
