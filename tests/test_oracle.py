"""Pin the CPU oracle (oracle/ntf_oracle.py) before trusting it.

Two independent anchors: (1) the reference test-suite's literal golden values
(pkg/tests/test_tensors.py, test_solver.py), restated here as numbers, and
(2) fixtures produced by running the reference package itself
(tests/golden/make_golden.py).  CPU only.
"""

import hashlib

import numpy as np
import pytest

from conftest import CONSTRAINT_CASES, MESH2_CFG, SMALL_CASES, SPARSE_CASES, rel
from oracle import ntf_oracle as O


# ---- literal goldens of the reference test-suite -------------------------

def test_kr_column_vectors():  # test_tensors.py:95-98
    c = np.array([[1.0], [2.0]])
    b = np.array([[3.0], [4.0]])
    assert O.khatri_rao([c, b]).ravel().tolist() == [3.0, 4.0, 6.0, 8.0]


def test_kr_identity_rows():  # test_tensors.py:100-102
    eye = np.eye(2)
    assert O.khatri_rao([eye, eye]).tolist() == [[1, 0], [0, 0], [0, 0], [0, 1]]


def test_mttkrp_ones_sum_rows():  # test_tensors.py:143-146
    t = O.OracleTensor(np.einsum("i,j,k->ijk", [1.0, 2.0], np.ones(2), np.ones(2)))
    f = [np.ones((2, 1))] * 3
    assert O.mttkrp(t, f, 1).tolist() == [[4.0], [8.0]]


def test_unfold_linear_index_map():  # test_tensors.py:66-72
    vals = np.fromfunction(lambda i, j, k: i + 2 * j + 4 * k, (2, 2, 2))
    assert O.unfold(vals, 1)[0].tolist() == [0.0, 2.0, 4.0, 6.0]


def test_scalar_update_and_hand_trajectory():  # test_solver.py:82-84, 222-235
    t = O.OracleTensor(np.full((1, 1, 1), 2.0))
    ones = [np.ones((1, 1)) for _ in range(3)]
    zeros = [np.zeros((1, 1)) for _ in range(3)]
    assert O.factor_update(t, ones, zeros[0], zeros[0], 1.0, 1)[0, 0] == pytest.approx(1.0)
    st = O.State([f.copy() for f in ones], zeros, [z.copy() for z in zeros], [1.0] * 3)
    cfg = O.Config()
    st, (p, d) = O.iterate(st, t, cfg)
    assert [f[0, 0] for f in st.factors] == pytest.approx([1.0, 1.0, 1.0])
    assert p == (0.0, 0.0, 0.0) and d == pytest.approx((1.0, 1.0, 1.0))
    assert st.rho == [1.0, 1.0, 1.0]
    st, _ = O.iterate(st, t, cfg)
    assert st.factors[0][0, 0] == pytest.approx(1.5)


def test_adapt_branches():  # test_solver.py:203-217
    cfg = O.Config()
    assert O.adapt([1.0], (10.0,), (1.0,), cfg) == [4.0]
    assert O.adapt([1.0], (1.0,), (10.0,), cfg) == [0.5]
    assert O.adapt([1.0], (1.0,), (1.0,), cfg) == [1.0]
    assert O.adapt([1.0], (0.0,), (10.0,), cfg) == [1.0]


def test_stop_boundary_inclusive():  # test_solver.py:181-193
    z = np.zeros((4, 3))
    st = O.State([z] * 3, [z] * 3, [z] * 3, [1.0] * 3)
    cfg = O.Config()
    thr = np.sqrt(12) * cfg.eps_abs
    assert O.stop_test((thr, 0, 0), (0, 0, 0), st, cfg)
    assert not O.stop_test((0, 0, 0), (0, thr * 1.000001, 0), st, cfg)


def test_uniform_extents():  # blocks.py:48-61
    assert O.uniform_extents(10, 3) == (4, 3, 3)
    assert O.uniform_extents(7, 7) == (1,) * 7
    with pytest.raises(ValueError):
        O.uniform_extents(3, 4)


# ---- fixtures produced by the reference itself ----------------------------

def test_algebra_matches_reference(golden_algebra):
    g = golden_algebra
    for case in range(3):
        x = g[f"c{case}_x"]
        fac = [g[f"c{case}_f{m}"] for m in range(3)]
        t = O.OracleTensor(x)
        for mode in (1, 2, 3):
            assert np.array_equal(O.unfold(x, mode), g[f"c{case}_unfold{mode}"])
            assert rel(O.mttkrp(t, fac, mode), g[f"c{case}_mttkrp{mode}"]) <= 1e-15
            assert rel(O.companion_gram(fac, mode), g[f"c{case}_gram{mode}"]) <= 1e-15
        assert np.array_equal(O.khatri_rao([fac[2], fac[1]]), g[f"c{case}_kr"])
        assert rel(O.reconstruct(fac), g[f"c{case}_recon"]) <= 1e-15


@pytest.mark.parametrize("name", sorted(SMALL_CASES))
def test_small_fit_trajectories_match_reference(golden_small, name):
    g = golden_small
    cfg = O.Config(**SMALL_CASES[name])
    res = O.fit(g[f"{name}_x"], int(g[f"{name}_rank"]), cfg)
    assert res.iterations == int(g[f"{name}_iterations"])
    assert res.restarts == int(g[f"{name}_restarts"])
    assert res.converged == bool(g[f"{name}_converged"])
    assert np.array_equal(np.array([p for p, _ in res.residual_history]), g[f"{name}_primal"])
    assert np.array_equal(np.array([d for _, d in res.residual_history]), g[f"{name}_dual"])
    assert np.array_equal(np.array(res.rho_history), g[f"{name}_rho"])
    assert res.rfe == float(g[f"{name}_rfe"])
    for m in range(3):
        assert np.array_equal(res.factors[m], g[f"{name}_aux{m}"])
    if f"{name}_hist_idx" in g:
        for n, it in enumerate(g[f"{name}_hist_idx"]):
            for m in range(3):
                assert np.array_equal(res.factor_history[it][m], g[f"{name}_hist{m}"][n])
    if f"{name}_rfe_hist" in g:
        assert np.allclose(res.rfe_history, g[f"{name}_rfe_hist"], rtol=1e-13, atol=0)


def test_mesh2_fixture_is_centralized_to_rounding(golden_small):
    """The reference's plan=2 mesh run equals the centralized oracle to 1e-12
    (mesh.py:341-343) — the bar our sharded path is held to."""
    g = golden_small
    res = O.fit(g["mesh2_x"], 3, O.Config(**MESH2_CFG))
    for n, it in enumerate(g["mesh2_hist_idx"]):
        for m in range(3):
            assert rel(g[f"mesh2_hist{m}"][n], res.factor_history[it][m]) <= 1e-12


def test_c1_generator_and_trajectory(golden_c1):
    g = golden_c1
    dseed, fseed = O.derive_seed(0, O.DATA_SALT, 0), O.derive_seed(0, O.FIT_SALT, 0)
    assert dseed == int(g["data_seed"]) and fseed == int(g["fit_seed"])
    x, _, sigma = O.generate((100, 100, 100), 10, 20.0, dseed)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(g["x_sha256"])
    assert sigma == float(g["sigma"])
    cfg = O.Config(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=50, max_restarts=0,
                   inner_sweeps=10, rho_init=float(g["rho1_rho0"]), track_factors=True)
    res = O.fit(x, 10, cfg)
    for n, it in enumerate(g["rho1_hist_idx"]):
        for m in range(3):
            assert np.array_equal(res.factor_history[it][m], g[f"rho1_hist{m}"][n])
    assert res.rfe == float(g["rho1_rfe"])


@pytest.mark.parametrize("k", range(4))
def test_constraint_projections_match_reference(golden_constraints, k):
    """constraints.py:72-111 goldens: simplex rows (an already-feasible row
    unchanged, ties) and the global top-c cardinality keep (stable ties)."""
    g = golden_constraints
    m = g[f"proj{k}_m"]
    assert np.array_equal(O.project(m, "row_stochastic"), g[f"proj{k}_simplex"])
    for c in (1, 4, 9, 40):
        assert np.array_equal(O.project(m, f"nonneg_card:{c}"), g[f"proj{k}_card{c}"])


@pytest.mark.parametrize("name", sorted(CONSTRAINT_CASES))
def test_constraint_fit_trajectories_match_reference(golden_constraints, name):
    """Fits with row-stochastic / cardinality modes (solver.py:182-193 equality
    constrained solve) reproduce the reference bit for bit."""
    g = golden_constraints
    specs = [str(s) for s in g[f"{name}_specs"]]
    res = O.fit(g[f"{name}_x"], int(g[f"{name}_rank"]), O.Config(**CONSTRAINT_CASES[name]), specs)
    assert np.array_equal(np.array([p for p, _ in res.residual_history]), g[f"{name}_primal"])
    assert np.array_equal(np.array([d for _, d in res.residual_history]), g[f"{name}_dual"])
    assert res.rfe == float(g[f"{name}_rfe"])
    for m in range(3):
        assert np.array_equal(res.factors[m], g[f"{name}_aux{m}"])
    for n, it in enumerate(g[f"{name}_hist_idx"]):
        for m in range(3):
            assert np.array_equal(res.factor_history[it][m], g[f"{name}_hist{m}"][n])


def test_sparse_mttkrp_and_fits_match_reference():
    """COO tensors (tensors.py:84-132, 263-273, 291-301): per-entry MTTKRP
    accumulated in entry order, Gram-identity RFE, fits bit for bit."""
    from conftest import load_golden

    g = load_golden("sparse.npz")
    for k in range(3):
        t = O.OracleSparse(g[f"m{k}_dims"], g[f"m{k}_idx"], g[f"m{k}_vals"])
        f = [g[f"m{k}_f{m}"] for m in range(3)]
        for m in range(3):
            assert np.array_equal(O.mttkrp(t, f, m + 1), g[f"m{k}_mttkrp{m + 1}"])
    for name, kw in SPARSE_CASES.items():
        t = O.OracleSparse(g[f"{name}_dims"], g[f"{name}_idx"], g[f"{name}_vals"])
        specs = [str(s) for s in g[f"{name}_specs"]]
        res = O.fit(t, int(g[f"{name}_rank"]), O.Config(**kw), specs)
        assert res.iterations == int(g[f"{name}_iterations"])
        assert res.rfe == float(g[f"{name}_rfe"])
        assert np.array_equal(np.array([p for p, _ in res.residual_history]), g[f"{name}_primal"])
        for m in range(3):
            assert np.array_equal(res.factors[m], g[f"{name}_aux{m}"])


def test_order4_mttkrp_and_fits_match_reference():
    """Order-4 dense tensors (unfold / khatri_rao for N = 4, four-mode
    solver): the oracle reproduces the reference bit for bit."""
    from conftest import ORDER4_CASES, load_golden

    g = load_golden("order4.npz")
    for k in range(2):
        t = O.OracleTensor(g[f"m{k}_x"])
        f = [g[f"m{k}_f{m}"] for m in range(4)]
        for m in range(4):
            assert np.array_equal(O.mttkrp(t, f, m + 1), g[f"m{k}_mttkrp{m + 1}"])
    for name, kw in ORDER4_CASES.items():
        specs = [str(s) for s in g[f"{name}_specs"]]
        res = O.fit(g[f"{name}_x"], int(g[f"{name}_rank"]), O.Config(**kw), specs)
        assert res.iterations == int(g[f"{name}_iterations"])
        assert res.rfe == float(g[f"{name}_rfe"])
        for m in range(4):
            assert np.array_equal(res.factors[m], g[f"{name}_aux{m}"])


def test_sparse_order4_matches_reference():
    from conftest import load_golden

    g = load_golden("order4.npz")
    for k in range(2):
        t = O.OracleSparse(g[f"s{k}_dims"], g[f"s{k}_idx"], g[f"s{k}_vals"])
        f = [g[f"s{k}_f{m}"] for m in range(4)]
        for m in range(4):
            assert np.array_equal(O.mttkrp(t, f, m + 1), g[f"s{k}_mttkrp{m + 1}"])
    t = O.OracleSparse(g["sp4_dims"], g["sp4_idx"], g["sp4_vals"])
    res = O.fit(t, 2, O.Config(seed=4, eps_abs=0.0, eps_rel=0.0, n_max=8, max_restarts=0,
                               track_factors=True))
    assert res.rfe == float(g["sp4_rfe"])
    for m in range(4):
        assert np.array_equal(res.factors[m], g[f"sp4_aux{m}"])
