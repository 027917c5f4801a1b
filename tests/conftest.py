"""Shared test configuration: the ``gpu`` marker and fixture loaders."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_algebra():
    return load_golden("algebra.npz")


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("small_fits.npz")


@pytest.fixture(scope="session")
def golden_constraints():
    return load_golden("constraints.npz")


@pytest.fixture(scope="session")
def golden_c1():
    return load_golden("c1.npz")


# cases of tests/golden/make_golden.py (kept in sync by test_golden_cases_listed)
SMALL_CASES = {
    "noiseless12": dict(seed=0, eps_abs=0.0, eps_rel=0.0, n_max=20, max_restarts=0, track_factors=True),
    "sweeps3": dict(seed=4, eps_abs=0.0, eps_rel=0.0, n_max=12, max_restarts=0, inner_sweeps=3,
                    track_factors=True, track_rfe=True),
    "converge": dict(seed=1),
    "restarts": dict(seed=0, n_max=3, max_restarts=2, track_factors=True),
    "noadapt": dict(seed=8, eps_abs=0.0, eps_rel=0.0, n_max=10, max_restarts=0, adapt=False,
                    inner_sweeps=2, track_factors=True),
    "ragged": dict(seed=2, eps_abs=0.0, eps_rel=0.0, n_max=8, max_restarts=0, track_factors=True),
    "bigrho": dict(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=15, max_restarts=0, rho_init=300.0,
                   inner_sweeps=4, track_factors=True),
}
# cases of make_golden.constraint_fits (specs are stored in the fixture)
CONSTRAINT_CASES = {
    "rowstoch": dict(seed=5, eps_abs=0.0, eps_rel=0.0, n_max=12, max_restarts=0, track_factors=True),
    "card": dict(seed=6, eps_abs=0.0, eps_rel=0.0, n_max=12, max_restarts=0, track_factors=True),
    "mixed": dict(seed=7, eps_abs=0.0, eps_rel=0.0, n_max=10, max_restarts=0, inner_sweeps=2,
                  track_factors=True),
    "cardall": dict(seed=8, eps_abs=0.0, eps_rel=0.0, n_max=8, max_restarts=0, track_factors=True),
}
# cases of make_golden.sparse_fits (COO tensors)
SPARSE_CASES = {
    "sp1": dict(seed=1, eps_abs=0.0, eps_rel=0.0, n_max=10, max_restarts=0, track_factors=True),
    "sp2": dict(seed=2, eps_abs=0.0, eps_rel=0.0, n_max=8, max_restarts=0, inner_sweeps=2,
                track_factors=True, track_rfe=True),
    "sp3": dict(seed=3),
}
# cases of make_golden.order4_fits (order-4 dense tensors)
ORDER4_CASES = {
    "o4a": dict(seed=1, eps_abs=0.0, eps_rel=0.0, n_max=10, max_restarts=0, track_factors=True),
    "o4b": dict(seed=2, eps_abs=0.0, eps_rel=0.0, n_max=8, max_restarts=0, inner_sweeps=2,
                track_factors=True, track_rfe=True),
    "o4c": dict(seed=3),
}
MESH2_CFG = dict(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=20, max_restarts=0, track_factors=True,
                 inner_sweeps=2)


def rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b)) / max(float(np.linalg.norm(b)), 1e-300)
