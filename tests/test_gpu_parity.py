"""Parity of the B200 path against the CPU oracle and the reference fixtures.

All tests here need a CUDA device and call the product through the C ABI
(libntf_b200.so).  Tolerances: fp64 <= 1e-12 for the MTTKRP (test_tensors.py
bar) and <= 1e-9 per-iteration working-factor difference for fits (north
star); fp32 tensors: final RFE within 1e-4 relative of the oracle, and the
fp32 MTTKRP within 1e-6 relative of the fp64 oracle.
"""

import numpy as np
import pytest

from conftest import MESH2_CFG, SMALL_CASES, rel
from oracle import ntf_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1409_2383_b200 as P  # noqa: E402
from paper_1409_2383_b200 import _native  # noqa: E402
from paper_1409_2383_b200 import synth  # noqa: E402


def _factors(rng, dims, R):
    return [rng.random((d, R)) for d in dims]


@pytest.mark.parametrize("dims,R", [((3, 4, 5), 2), ((7, 2, 6), 3), ((1, 5, 3), 1), ((33, 17, 65), 7),
                                    ((40, 50, 60), 20), ((9, 130, 11), 33), ((64, 64, 64), 128),
                                    ((129, 3, 257), 10)])
@pytest.mark.parametrize("engine", ["auto", "cuda_core"])
def test_mttkrp_fp64_matches_oracle(dims, R, engine):
    rng = np.random.default_rng(11)
    x = rng.random(dims)
    f = _factors(rng, dims, R)
    t = O.OracleTensor(x)
    for mode in (1, 2, 3):
        got = P.mttkrp_factors(P.DenseTensor(x), f, mode, engine=engine)
        assert rel(got, O.mttkrp(t, f, mode)) <= 1e-12


@pytest.mark.parametrize("dims,R", [
    ((130, 40, 64), 5),     # K a multiple of the chunk, one 8-column block, ragged second m-tile
    ((70, 33, 31), 12),     # odd K < chunk: every chunk straddles F_hi rows, scalar copies
    ((20, 200, 36), 17),    # odd R: 8-byte factor-row copies
    ((96, 50, 48), 24), ((150, 30, 40), 40), ((64, 70, 34), 48), ((200, 24, 66), 56),
    ((40, 90, 100), 64),    # block counts 3..8 of the 128-row kernels
    ((90, 40, 44), 72), ((48, 64, 80), 100),  # 64-row kernels (9 and 13 blocks)
    ((300, 6, 4), 128),     # 16 blocks over tiny extents (the stage ring shrinks)
    ((4, 6, 1000), 20),     # two rows, long contraction
])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fp64_engine_geometries(dims, R, dtype):
    """The fp64-arithmetic engine (DMMA fragments, DESIGN 4b) over its tile
    geometries: every 8-column block count class, vector and scalar copies,
    chunks that straddle F_hi rows, ragged m-tiles, fp32 and fp64 tensors —
    all at the fp64 bar (fp32 values are exact in fp64)."""
    rng = np.random.default_rng(sum(dims) + R)
    x = (rng.random(dims) - 0.3).astype(dtype)
    f = [rng.random((d, R)) - 0.4 for d in dims]
    t = O.OracleTensor(x.astype(np.float64))
    for mode in (1, 2, 3):
        got = P.mttkrp_factors(P.DenseTensor(x), f, mode, engine="cuda_core")
        want = O.mttkrp(t, f, mode)
        # mixed signs: the bar is relative to |X_(n)| |KR| (the sums cancel)
        kr = O.khatri_rao([f[m - 1] for m in O.companion_modes(mode, 3)])
        scale = np.linalg.norm(np.abs(t.unfolding(mode)) @ np.abs(kr))
        assert np.linalg.norm(got - want) <= 1e-12 * scale, (mode, dims, R)


@pytest.mark.parametrize("dims,R,dtype", [((300, 200, 150), 50, np.float64), ((257, 130, 96), 100, np.float32),
                                          ((1000, 40, 30), 20, np.float64)])
def test_fp64_engine_bitwise_repeatable(dims, R, dtype):
    """The producer / DMMA-warp pipeline (named barriers, cp.async ring) and
    the cluster reduction have no float atomics and a fixed order: 25 launches
    per mode give bit-identical results (a race in the stage hand-over would
    show up here), and they match the oracle."""
    rng = np.random.default_rng(8)
    x = rng.random(dims).astype(dtype)
    f = _factors(rng, dims, R)
    t = P.DenseTensor(x)
    ot = O.OracleTensor(x.astype(np.float64))
    for mode in (1, 2, 3):
        first = P.mttkrp_factors(t, f, mode, engine="cuda_core")
        assert rel(first, O.mttkrp(ot, f, mode)) <= 1e-12
        for _ in range(24):
            again = P.mttkrp_factors(t, f, mode, engine="cuda_core")
            assert np.array_equal(first, again), mode


def test_mttkrp_golden_ones():  # reference test_tensors.py:143-146
    x = np.einsum("i,j,k->ijk", [1.0, 2.0], np.ones(2), np.ones(2))
    got = P.mttkrp_factors(P.DenseTensor(x), [np.ones((2, 1))] * 3, 1)
    assert got.tolist() == [[4.0], [8.0]]


def test_mttkrp_reference_fixture(golden_algebra):
    g = golden_algebra
    for case in range(3):
        x = g[f"c{case}_x"]
        fac = [g[f"c{case}_f{m}"] for m in range(3)]
        for mode in (1, 2, 3):
            got = P.mttkrp_factors(P.DenseTensor(x), fac, mode)
            assert rel(got, g[f"c{case}_mttkrp{mode}"]) <= 1e-12


@pytest.mark.parametrize("dims,R", [((50, 60, 70), 20), ((128, 64, 100), 32), ((31, 45, 29), 50),
                                    ((100, 100, 100), 100)])
def test_mttkrp_fp32_accuracy(dims, R):
    """fp32 tensor, fp64 factors: error must be at the iid-rounding level
    (recipe of SURVEY 8(d)), far below the 1e-7 structured-rounding level."""
    rng = np.random.default_rng(5)
    x32 = rng.random(dims).astype(np.float32)
    f = _factors(rng, dims, R)
    t = O.OracleTensor(x32.astype(np.float64))
    for mode in (1, 2, 3):
        got = P.mttkrp_factors(P.DenseTensor(x32), f, mode)
        assert rel(got, O.mttkrp(t, f, mode)) <= 2e-8


@pytest.mark.parametrize("dims,R", [((96, 80, 72), 1), ((130, 40, 64), 7), ((260, 200, 136), 20),
                                    ((70, 300, 48), 33), ((129, 129, 200), 50), ((64, 64, 64), 64),
                                    ((150, 90, 112), 100), ((40, 50, 64), 128),
                                    ((1, 3, 37), 5), ((200, 7, 1), 16), ((3, 500, 9), 128),
                                    ((129, 1, 65), 31)])
def test_mttkrp_tcgen05_accuracy(dims, R):
    """Tensor-core engine (fp32 X, exact fixed-point slicing) against the fp64
    oracle on the same fp32 values, every mode, all accumulator widths
    (N = 16..128: single and split first MMA, 4/8/16 epilogue warps), equal
    and ragged m-tiles, extents of 1 and l extents that are not a multiple of
    the 64-wide l block (the block image has no stride requirement)."""
    rng = np.random.default_rng(11)
    x32 = rng.random(dims).astype(np.float32)
    f = _factors(rng, dims, R)
    x64 = x32.astype(np.float64)
    t = O.OracleTensor(x64)
    t_abs, t_one = O.OracleTensor(np.abs(x64)), O.OracleTensor(np.ones(dims))
    f_abs = [np.abs(a) for a in f]
    for mode in (1, 2, 3):
        got = P.mttkrp_factors(P.DenseTensor(x32), f, mode, engine="tcgen05")
        want = O.mttkrp(t, f, mode)
        # worst case, every contraction length: the 22-bit split of X moves each
        # element by <= 2^-22 max|X| (mttkrp_tc.cu image_split_kernel); the
        # 33-bit factor slices and the double-float epilogue stay below 1e-9
        bound = 2.0**-22 * np.abs(x64).max() * O.mttkrp(t_one, f_abs, mode) \
            + 1e-9 * O.mttkrp(t_abs, f_abs, mode)
        assert np.all(np.abs(got - want) <= bound), (mode, float(np.max(np.abs(got - want) / bound)))
        # long contractions: the per-element errors are independent and average
        # out to the i.i.d.-rounding level of SURVEY 7.3 #2
        if x32.size // dims[mode - 1] >= 2000:
            assert rel(got, want) <= 5e-9, (mode, rel(got, want))


@pytest.mark.parametrize("engine,tol", [("cuda_core", 1e-9), ("tcgen05", 5e-9)])
def test_mttkrp_mode_consistency_c2_full_size(engine, tol):
    """Size-independent property at BASELINE c2 size: for every column r,
    sum_i M1[i,r] A[i,r] = sum_j M2[j,r] B[j,r] = sum_k M3[k,r] C[k,r].
    (tcgen05: the i.i.d. 2^-22 KR-slice quantisation differs per mode.)"""
    w = synth.CONFIGS["c2"]
    rng = np.random.default_rng(1)
    x = rng.random(w.dims, dtype=np.float32)
    f = _factors(rng, w.dims, w.rank)
    t = P.DenseTensor(x)
    v = [np.sum(P.mttkrp_factors(t, f, m, engine=engine) * f[m - 1], axis=0) for m in (1, 2, 3)]
    assert rel(v[1], v[0]) <= tol and rel(v[2], v[0]) <= tol


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_mttkrp_mode_consistency_large_configs(name):
    """The same property at the other BASELINE configs' full sizes (c3 1000^3
    R=50, c4 5000x500x200 R=32, c5 2000^3 R=100: 4, 2 and 32 GB fp32
    tensors), i.e. the tcgen05 engine's N = 64, 32 and 112 instances with
    many m-tiles, on a device-resident tensor."""
    w = synth.CONFIGS[name]
    need = 4 * int(np.prod(w.dims)) * 2 + (1 << 30)  # tensor + one mode's block image
    free, _ = torch.cuda.mem_get_info()
    if free < need:  # pragma: no cover
        pytest.skip(f"{name} needs {need >> 30} GiB")
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(w.dims, dtype=torch.float32, device="cuda", generator=g)
    rng = np.random.default_rng(4)
    f = _factors(rng, w.dims, w.rank)
    t = P.DenseTensor(x)
    v = []
    for m in (1, 2, 3):
        got = P.mttkrp_factors(t, f, m)
        got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
        v.append(np.sum(got * f[m - 1], axis=0))
        torch.cuda.empty_cache()
    assert rel(v[1], v[0]) <= 5e-9 and rel(v[2], v[0]) <= 5e-9, (rel(v[1], v[0]), rel(v[2], v[0]))
    del x, t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("R", [88, 97, 100, 104, 105, 128])
def test_mttkrp_pair_kernel_packed_ranges(R):
    """CTA-pair kernel with merged accumulator sets (N = 96, 112, 128; tensors
    of 2^28 elements and more: R = 88 and 128 are the N = 96 / 128 instances
    with 16 epilogue warps).  At N = 112: for
    R <= 104 the T0 / T1 slice ranges and ACC0 are packed to 104 columns (the
    first MMA of a K step runs at N' = 208 instead of 224, the epilogue drains
    52 columns per thread as 6 x 8 + 4); R = 105 is the unpacked instance.
    Every mode, every element, against the fp64-arithmetic engine on the same
    fp32 values, on a ragged shape (m-tiles of 96..128 rows, last l block
    partly filled)."""
    dims = (768, 650, 600)
    g = torch.Generator(device="cuda").manual_seed(R)
    x = torch.rand(dims, dtype=torch.float32, device="cuda", generator=g)
    rng = np.random.default_rng(R)
    f = _factors(rng, dims, R)
    t = P.DenseTensor(x)
    for m in (1, 2, 3):
        got = np.asarray(P.mttkrp_factors(t, f, m, engine="tcgen05"))
        want = np.asarray(P.mttkrp_factors(t, f, m, engine="cuda_core"))
        assert got.shape == (dims[m - 1], R)
        assert rel(got, want) <= 5e-9, (m, rel(got, want))
        assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-7, m
    del x, t
    torch.cuda.empty_cache()


def test_norm_and_rfe_kernel():
    rng = np.random.default_rng(2)
    dims = (13, 9, 21)
    f = _factors(rng, dims, 4)
    x = O.reconstruct(f) + 0.01 * rng.standard_normal(dims)
    t = P.DenseTensor(x)
    assert t.norm() == pytest.approx(np.linalg.norm(x), rel=1e-14)
    from paper_1409_2383_b200.engine import device_tensor, sq_error

    out = sq_error(device_tensor(t), f).cpu().numpy()
    assert out[1] == pytest.approx(np.linalg.norm(x - O.reconstruct(f)) ** 2, rel=1e-12)


@pytest.mark.parametrize("dims,R,dtype", [((5, 24, 33), 3, np.float64), ((3, 40, 300), 10, np.float32),
                                          ((2, 65, 257), 21, np.float64), ((4, 32, 64), 100, np.float32),
                                          ((1, 100, 7), 256, np.float64)])
def test_rfe_kernel_wide_tensors(dims, R, dtype):
    """Tensors at least 24 wide in mode 2 take the DMMA reconstruction
    kernel: ragged j and k tiles, ranks that are not multiples of 4, fp32 and
    fp64 tensors, against the explicit reconstruction (tensors.py:276-290)."""
    rng = np.random.default_rng(R)
    f = [rng.random((d, R)) - 0.2 for d in dims]
    x = (O.reconstruct(f) + 0.05 * rng.standard_normal(dims)).astype(dtype)
    from paper_1409_2383_b200.engine import device_tensor, sq_error

    out = sq_error(device_tensor(P.DenseTensor(x)), f).cpu().numpy()
    x64 = x.astype(np.float64)
    assert out[0] == pytest.approx(np.sum(x64 ** 2), rel=1e-12)
    assert out[1] == pytest.approx(np.sum((x64 - O.reconstruct(f)) ** 2), rel=1e-11)


def _cmp_fit(res, g, name, tol=1e-9):
    assert res.iterations == int(g[f"{name}_iterations"])
    assert res.restarts == int(g[f"{name}_restarts"])
    assert res.converged == bool(g[f"{name}_converged"])
    # residual norms: relative 1e-8, with an absolute floor at 1e-9 of the
    # history's scale (late dual residuals sit at the rounding level, ~1e-12)
    for key, got in (("primal", [r.primal for r in res.residual_history]),
                     ("dual", [r.dual for r in res.residual_history])):
        want = g[f"{name}_{key}"]
        got = np.array(got)
        assert np.all(np.abs(got - want) <= 1e-8 * np.abs(want) + 1e-9 * np.max(np.abs(want))), key
    assert np.array_equal(np.array(res.rho_history), g[f"{name}_rho"])
    assert res.rfe == pytest.approx(float(g[f"{name}_rfe"]), rel=1e-9)
    worst = 0.0
    if f"{name}_hist_idx" in g:
        for n, it in enumerate(g[f"{name}_hist_idx"]):
            for m in range(3):
                worst = max(worst, rel(res.factor_history[it][m], g[f"{name}_hist{m}"][n]))
    for m in range(3):
        worst = max(worst, rel(res.model.factors[m], g[f"{name}_aux{m}"]))
    assert worst <= tol, worst
    return worst


@pytest.mark.parametrize("name", sorted(SMALL_CASES))
def test_small_fits_match_reference(golden_small, name):
    g = golden_small
    res = P.fit(g[f"{name}_x"], int(g[f"{name}_rank"]), None, P.SolverConfig(**SMALL_CASES[name]))
    _cmp_fit(res, g, name)
    if f"{name}_rfe_hist" in g:
        assert np.allclose(res.rfe_history, g[f"{name}_rfe_hist"], rtol=1e-9, atol=1e-12)


def test_reference_densetensor_accepted(golden_small):
    """A foreign DenseTensor-like object (.values/.dims) is accepted as is."""
    g = golden_small

    class Foreign:
        def __init__(self, v):
            self.values = v
            self.dims = v.shape

    res = P.fit(Foreign(g["noiseless12_x"]), 3, None, P.SolverConfig(**SMALL_CASES["noiseless12"]))
    _cmp_fit(res, g, "noiseless12")


def _c1_inputs(g, tag):
    w = synth.CONFIGS["c1"]
    dseed, fseed = synth.seeds()
    x, _ = synth.generate(w.dims, w.rank, w.snr_db, dseed)
    cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=50, max_restarts=0,
                         inner_sweeps=10, rho_init=float(g[f"{tag}_rho0"]), track_factors=True)
    return x, cfg


@pytest.mark.parametrize("tag", ["rho1", "rhotr"])
def test_c1_per_iteration_parity_replayed_penalties(golden_c1, tag):
    """BASELINE config 1 (100^3, R=10, fp64, 10 inner x 50 outer) under the
    reference's own penalty sequence: max per-iteration working-factor
    relative difference <= 1e-9 over all 50 iterations."""
    g = golden_c1
    x, cfg = _c1_inputs(g, tag)
    res = P.fit(x, 10, None, cfg, rho_schedule=g[f"{tag}_rho"])
    worst = _cmp_fit(res, g, tag, tol=1e-9)
    print(f"c1 {tag} (replayed rho): max per-iteration factor rel diff {worst:.3e}")


def _degenerate(p, d, mu=8.0, floor=1e-13):
    """A penalty decision (solver.py:286-291) decided by rounding noise: the
    primal residual at the rounding floor (the p > 0 guard) or a ratio test
    within 1e-9 of its threshold."""
    return (p < floor or abs(p - mu * d) <= 1e-9 * max(p, mu * d)
            or abs(d - mu * p) <= 1e-9 * max(d, mu * p))


@pytest.mark.parametrize("tag", ["rho1", "rhotr"])
def test_c1_free_running_parity(golden_c1, tag):
    """Free-running c1 fit: identical penalty decisions and <= 1e-9 factor
    parity for every iteration up to the first decision the reference itself
    takes on rounding noise; final RFE within 1e-6 relative."""
    g = golden_c1
    x, cfg = _c1_inputs(g, tag)
    res = P.fit(x, 10, None, cfg)
    prim, dual = g[f"{tag}_primal"], g[f"{tag}_dual"]
    first = len(prim)
    for it in range(len(prim)):
        if any(_degenerate(prim[it][m], dual[it][m]) for m in range(3)):
            first = it
            break
    rho = np.array(res.rho_history)
    assert np.array_equal(rho[:first], g[f"{tag}_rho"][:first])
    idx = g[f"{tag}_hist_idx"]
    worst = 0.0
    for n, it in enumerate(idx):
        if it > first:
            break
        for m in range(3):
            worst = max(worst, rel(res.factor_history[it][m], g[f"{tag}_hist{m}"][n]))
    assert worst <= 1e-9
    assert abs(res.rfe - float(g[f"{tag}_rfe"])) <= 1e-6 * float(g[f"{tag}_rfe"])
    print(f"c1 {tag} free-running: first noise-level decision at iteration {first}, "
          f"max factor diff before it {worst:.2e}, rfe {res.rfe:.12f} vs {float(g[f'{tag}_rfe']):.12f}")


def test_fp32_final_rfe_parity():
    """fp32 tensor (200^3, R=20, 20 dB, 10 inner x 20 outer): final RFE within
    1e-4 relative of the oracle on the identical (upcast) values."""
    dseed, fseed = synth.seeds()
    x, _ = synth.generate((200, 200, 200), 20, 20.0, dseed, dtype=np.float32)
    cfg = P.SolverConfig(seed=fseed, eps_abs=0.0, eps_rel=0.0, n_max=20, max_restarts=0,
                         inner_sweeps=10)
    got = P.fit(P.DenseTensor(x), 20, None, cfg)
    want = O.fit(x.astype(np.float64), 20, O.Config(**vars(cfg)))
    d = abs(got.rfe - want.rfe) / want.rfe
    print(f"fp32 200^3 R=20: rfe gpu {got.rfe:.10f} oracle {want.rfe:.10f} rel {d:.2e}")
    assert d <= 1e-4


def test_fp32_fit_modes_with_different_kernel_geometry():
    """A plan whose three tcgen05 MTTKRPs need different shared-memory sizes
    (m-tiles of 128, 104 and 112 rows; l extents of 1, 2 and 5 blocks share
    one kernel instance): the fit runs and matches the oracle's final RFE."""
    rng = np.random.default_rng(8)
    dims, R = (512, 400, 300), 20
    x = (O.reconstruct([rng.random((d, R)) for d in dims])
         + 0.1 * rng.standard_normal(dims)).astype(np.float32)
    cfg = P.SolverConfig(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=3, max_restarts=0, inner_sweeps=2)
    got = P.fit(P.DenseTensor(x), R, None, cfg)
    want = O.fit(x.astype(np.float64), R, O.Config(**vars(cfg)))
    assert abs(got.rfe - want.rfe) <= 1e-4 * want.rfe, (got.rfe, want.rfe)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_interleaved_plans_with_different_ranks(dtype):
    """Two live plans whose kernels need different shared memory (R = 3 and
    R = 100 share the row-update, ridge and MTTKRP kernel instances): running
    them interleaved gives bitwise the results each gives alone."""
    from paper_1409_2383_b200.engine import DeviceProblem

    rng = np.random.default_rng(12)
    dims = (40, 30, 24)
    x = torch.from_numpy(rng.random(dims).astype(dtype)).cuda()
    cfg = P.SolverConfig(seed=4, eps_abs=0.0, eps_rel=0.0, n_max=4, max_restarts=0, inner_sweeps=2)

    def make(R):
        prob = DeviceProblem(x, dims, R, cfg, history_capacity=4)
        st = P.init_state(dims, R, cfg)
        prob.load_state(st.factors, st.aux, st.duals, st.rho)
        return prob

    def state(prob):
        torch.cuda.synchronize()
        return [np.array(f, copy=True) for f in prob.read_state()[0]]

    alone = {}
    for R in (3, 100):
        prob = make(R)
        prob.run(2)
        alone[R] = state(prob)
        prob.close()
    b = make(100)
    a = make(3)  # prepared last, with the smaller shared-memory needs
    b.run(1)
    a.run(1)
    b.run(1)
    a.run(1)
    for R, prob in ((3, a), (100, b)):
        for got, want in zip(state(prob), alone[R]):
            assert np.array_equal(got, want), R
        prob.close()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_plan_cache_reuse_is_bitwise_fresh(dtype, monkeypatch):
    """Back-to-back fits of one geometry reuse the plan (its tensor buffer
    is refilled, block images re-split, state reloaded): bitwise the results
    of fresh plans, the caller's device tensor untouched, and a config change
    builds a new plan."""
    rng = np.random.default_rng(21)
    dims, R = (36, 28, 20), 4
    xs = [rng.random(dims).astype(dtype) for _ in range(3)]
    cfg = P.SolverConfig(seed=5, eps_abs=0.0, eps_rel=0.0, n_max=6, max_restarts=0, inner_sweeps=3)
    cfg2 = P.SolverConfig(seed=5, eps_abs=0.0, eps_rel=0.0, n_max=6, max_restarts=0, inner_sweeps=2)
    xd = torch.from_numpy(xs[0]).cuda()
    keep = xd.clone()
    P.release_plan_cache()
    cached = [P.fit(P.DenseTensor(xd), R, None, cfg), P.fit(xs[1], R, None, cfg),
              P.fit(xs[2], R, None, cfg2), P.fit(xs[1], R, None, cfg)]
    assert torch.equal(xd, keep)
    monkeypatch.setenv("NTF_B200_PLAN_CACHE", "0")
    fresh = [P.fit(xs[0], R, None, cfg), P.fit(xs[1], R, None, cfg),
             P.fit(xs[2], R, None, cfg2), P.fit(xs[1], R, None, cfg)]
    for a, b in zip(cached, fresh):
        for m in range(3):
            assert np.array_equal(a.model.factors[m], b.model.factors[m])
        assert a.residual_history == b.residual_history and a.rfe == b.rfe
    P.release_plan_cache()


def test_iterate_matches_oracle(golden_small):
    g = golden_small
    x = g["sweeps3_x"]
    cfg = P.SolverConfig(seed=4, inner_sweeps=3)
    st = P.init_state(x.shape, 2, cfg)
    ost = O.init_state(x.shape, 2, O.Config(seed=4, inner_sweeps=3))
    t = P.DenseTensor(x)
    ot = O.OracleTensor(x)
    for _ in range(4):
        st, res = P.iterate(st, t, None, cfg)
        ost, (p, d) = O.iterate(ost, ot, O.Config(seed=4, inner_sweeps=3))
        for m in range(3):
            assert rel(st.factors[m], ost.factors[m]) <= 1e-12
            assert rel(st.aux[m], ost.aux[m]) <= 1e-12
            assert rel(st.duals[m], ost.duals[m]) <= 1e-11
        assert np.allclose(res.primal, p, rtol=1e-9) and np.allclose(res.dual, d, rtol=1e-9)
        assert st.rho == ost.rho


def test_errors_match_reference():
    with pytest.raises(ValueError):
        P.fit(np.zeros((2, 2, 2)), 1)
    with pytest.raises(ValueError):
        P.fit(np.ones((2, 2, 2)), 0)
    x = np.ones((3, 3, 3))
    x[1, 1, 1] = np.nan
    with pytest.raises(ValueError):
        P.fit(x, 1, None, P.SolverConfig(n_max=2, max_restarts=0))
    with pytest.raises(ValueError, match="exceeds factor size"):  # solver.py:359-363
        P.fit(np.ones((3, 3, 3)), 1, P.ConstraintSpec.nonneg_card(4))


def test_deterministic_and_graph_equals_eager(golden_small):
    g = golden_small
    x = g["bigrho_x"]
    cfg = P.SolverConfig(**{**SMALL_CASES["bigrho"], "track_factors": False})
    a = P.fit(x, 5, None, cfg)
    b = P.fit(x, 5, None, cfg)
    for m in range(3):
        assert np.array_equal(a.model.factors[m], b.model.factors[m])
    assert a.residual_history == b.residual_history
    c = P.fit(x, 5, None, P.SolverConfig(**SMALL_CASES["bigrho"]))  # per-iteration host path
    for m in range(3):
        assert np.array_equal(a.model.factors[m], c.model.factors[m])


def test_distributed_fit_single_rank_is_fit(golden_small):
    g = golden_small
    res = P.distributed_fit(g["mesh2_x"], 3, None, P.SolverConfig(**MESH2_CFG), plan=1)
    want = O.fit(g["mesh2_x"], 3, O.Config(**MESH2_CFG))
    for it in range(len(want.factor_history)):
        for m in range(3):
            assert rel(res.factor_history[it][m], want.factor_history[it][m]) <= 1e-9


def test_library_is_the_one_loaded():
    lib = _native.load()
    assert lib.ntf_abi_version() == 2
    import os

    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libntf_b200.so" in maps


def test_sharded_engine_one_rank_nccl_graph(golden_small, tmp_path, monkeypatch):
    """The sharded engine (slab images, row all-gathers, norm gather, the
    graph-captured outer iteration) on a one-rank NCCL group: per-iteration
    factors within 1e-9 of the oracle, and the captured iteration bitwise equal
    to the eager one (NTF_B200_SHARDED_GRAPH=0)."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        g = golden_small
        kw = dict(MESH2_CFG)
        kw["n_max"] = max(int(kw.get("n_max", 0)), 8)
        want = O.fit(g["mesh2_x"], 3, O.Config(**kw))
        import warnings

        with warnings.catch_warnings():  # the graph capture must succeed (no eager fallback)
            warnings.filterwarnings("error", message="sharded iteration not captured")
            got = P.distributed_fit(g["mesh2_x"], 3, None, P.SolverConfig(**kw), plan=1,
                                    sharded=True)
        monkeypatch.setenv("NTF_B200_SHARDED_GRAPH", "0")
        eager = P.distributed_fit(g["mesh2_x"], 3, None, P.SolverConfig(**kw), plan=1, sharded=True)
        assert len(got.factor_history) == len(want.factor_history) >= 4
        for it in range(len(want.factor_history)):
            for m in range(3):
                assert rel(got.factor_history[it][m], want.factor_history[it][m]) <= 1e-9
                assert np.array_equal(got.factor_history[it][m], eager.factor_history[it][m])
        assert got.residual_history == eager.residual_history
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["rowstoch", "card", "mixed", "cardall"])
def test_constraint_fits_match_reference(golden_constraints, name):
    """Row-stochastic (equality-constrained row solve + simplex projection in
    the row update) and global top-c cardinality (select + apply kernels)
    modes: per-iteration working factors within 1e-9 of the reference's fit
    (tests/golden/constraints.npz), final aux model and residuals likewise.
    The reference's penalty sequence is replayed: at an interior iterate the
    primal residual is exactly 0 in the reference and ~1e-17 here, and the
    adaptation branch `p > 0` (solver.py:286-291) then decides on rounding
    noise ("cardall" iteration 4)."""
    from conftest import CONSTRAINT_CASES

    g = golden_constraints
    specs = [P.ConstraintSpec.parse(str(s)) for s in g[f"{name}_specs"]]
    res = P.fit(g[f"{name}_x"], int(g[f"{name}_rank"]), specs,
                P.SolverConfig(**CONSTRAINT_CASES[name]), rho_schedule=g[f"{name}_rho"])
    for n, it in enumerate(g[f"{name}_hist_idx"]):
        for m in range(3):
            assert rel(res.factor_history[it][m], g[f"{name}_hist{m}"][n]) <= 1e-9, (it, m)
    for m in range(3):
        assert rel(res.model.factors[m], g[f"{name}_aux{m}"]) <= 1e-9
    prim = np.array([r.primal for r in res.residual_history])
    assert np.allclose(prim, g[f"{name}_primal"], rtol=1e-7, atol=1e-12)
    assert abs(res.rfe - float(g[f"{name}_rfe"])) <= 1e-9 * float(g[f"{name}_rfe"])
    # feasibility of the reported model (constraints.is_feasible semantics)
    for m, s in enumerate(specs):
        a = res.model.factors[m]
        assert a.min() >= 0.0
        if s.kind == "nonneg_card":
            assert np.count_nonzero(a) <= s.card
        if s.kind == "row_stochastic":
            assert np.all(np.abs(a.sum(axis=1) - 1.0) <= 1e-12)


def test_cardinality_selection_ties_and_budget():
    """Global top-c selection on the device: ties broken by row-major index
    (constraints.py:99-101), large budgets keep every clamped entry."""
    rng = np.random.default_rng(5)
    dims, R = (14, 9, 11), 3
    x = O.reconstruct([rng.random((d, R)) for d in dims]) + 0.01 * rng.standard_normal(dims)
    kw = dict(seed=2, eps_abs=0.0, eps_rel=0.0, n_max=6, max_restarts=0, track_factors=True)
    for specs in (["nonneg_card:1", "nonneg_card:27", "nonneg_card:33"],
                  ["row_stochastic", "row_stochastic", "nonneg_card:5"]):
        want = O.fit(x, R, O.Config(**kw), specs)
        got = P.fit(x, R, [P.ConstraintSpec.parse(s) for s in specs], P.SolverConfig(**kw),
                    rho_schedule=np.array(want.rho_history))
        for it in range(len(want.factor_history)):
            for m in range(3):
                assert rel(got.factor_history[it][m], want.factor_history[it][m]) <= 1e-9
        for m in range(3):
            assert np.array_equal(got.model.factors[m] > 0, want.factors[m] > 0)


def test_sparse_mttkrp_bitwise_and_fits_match_reference():
    """COO engine (mttkrp_coo.cu): MTTKRP bit for bit equal to the
    reference's np.add.at accumulation (tensors.py:263-273); fits per
    iteration within 1e-9 of the reference, Gram-identity RFE
    (tensors.py:291-301) and track_rfe likewise."""
    from conftest import SPARSE_CASES, load_golden

    g = load_golden("sparse.npz")
    for k in range(3):
        t = P.CooTensor(g[f"m{k}_dims"], g[f"m{k}_idx"], g[f"m{k}_vals"])
        f = [g[f"m{k}_f{m}"] for m in range(3)]
        for m in range(3):
            assert np.array_equal(P.mttkrp_factors(t, f, m + 1), g[f"m{k}_mttkrp{m + 1}"])
    for name, kw in SPARSE_CASES.items():
        t = P.CooTensor(g[f"{name}_dims"], g[f"{name}_idx"], g[f"{name}_vals"])
        specs = [P.ConstraintSpec.parse(str(s)) for s in g[f"{name}_specs"]]
        res = P.fit(t, int(g[f"{name}_rank"]), specs, P.SolverConfig(**kw),
                    rho_schedule=g[f"{name}_rho"] if kw.get("eps_abs", 1) == 0.0 else None)
        assert res.iterations == int(g[f"{name}_iterations"])
        assert res.converged == bool(g[f"{name}_converged"])
        assert abs(res.rfe - float(g[f"{name}_rfe"])) <= 1e-9 * float(g[f"{name}_rfe"])
        for m in range(3):
            assert rel(res.model.factors[m], g[f"{name}_aux{m}"]) <= 1e-9
        if f"{name}_hist_idx" in g:
            for n, it in enumerate(g[f"{name}_hist_idx"]):
                for m in range(3):
                    assert rel(res.factor_history[it][m], g[f"{name}_hist{m}"][n]) <= 1e-9
        if f"{name}_rfe_hist" in g:
            assert np.allclose(res.rfe_history, g[f"{name}_rfe_hist"], rtol=1e-9, atol=0)
    with pytest.raises(ValueError):
        P.CooTensor((3, 3, 3), [[0, 0, 0], [0, 0, 0]], [1.0, 2.0])  # duplicates (tensors.py:103-104)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_order4_mttkrp_and_fits_match_reference(dtype):
    """Order-4 dense tensors on the device: each MTTKRP runs as an order-3 one
    on the reshaped view (I x J x KL or IJ x K x L) with the merged modes'
    Khatri-Rao pair; fp64 MTTKRPs within 1e-12 of the reference (fp32 input:
    within 5e-8 of the oracle on the same fp32 values); fits within 1e-9 per iteration
    (penalty sequence replayed), RFE and track_rfe likewise."""
    from conftest import ORDER4_CASES, load_golden

    g = load_golden("order4.npz")
    for k in range(2):
        x = g[f"m{k}_x"].astype(dtype)
        if dtype == np.float32:  # fixed-point split: 22 bits of max|X| (U[0,1) data, as the fp32 tests)
            x = np.random.default_rng(k).random(x.shape).astype(np.float32)
        f = [g[f"m{k}_f{m}"] for m in range(4)]
        t = P.DenseTensor(x)
        for m in range(4):
            want = g[f"m{k}_mttkrp{m + 1}"] if dtype == np.float64 else O.mttkrp(
                O.OracleTensor(x.astype(np.float64)), f, m + 1)
            # fp32: the split's 2^-22 (of max|X|) rounding averages over only
            # 60-90 terms at these tiny shapes
            assert rel(P.mttkrp_factors(t, f, m + 1), want) <= (1e-12 if dtype == np.float64 else 5e-8)
    if dtype == np.float32:
        return
    for name, kw in ORDER4_CASES.items():
        specs = [P.ConstraintSpec.parse(str(s)) for s in g[f"{name}_specs"]]
        res = P.fit(g[f"{name}_x"], int(g[f"{name}_rank"]), specs, P.SolverConfig(**kw),
                    rho_schedule=g[f"{name}_rho"] if kw.get("eps_abs", 1) == 0.0 else None)
        assert res.iterations == int(g[f"{name}_iterations"])
        assert abs(res.rfe - float(g[f"{name}_rfe"])) <= 1e-9 * float(g[f"{name}_rfe"])
        for m in range(4):
            assert rel(res.model.factors[m], g[f"{name}_aux{m}"]) <= 1e-9
        if f"{name}_hist0" in g:
            for it in range(len(res.factor_history)):
                for m in range(4):
                    assert rel(res.factor_history[it][m], g[f"{name}_hist{m}"][it]) <= 1e-9
        if f"{name}_rfe_hist" in g:
            assert np.allclose(res.rfe_history, g[f"{name}_rfe_hist"], rtol=1e-9, atol=0)


def test_sparse_order4_mttkrp_bitwise_and_fit():
    """Order-4 COO tensors: MTTKRP bit for bit (np.add.at order, three
    companion rows highest mode first), fit within 1e-9 per iteration."""
    from conftest import load_golden

    g = load_golden("order4.npz")
    for k in range(2):
        t = P.CooTensor(g[f"s{k}_dims"], g[f"s{k}_idx"], g[f"s{k}_vals"])
        f = [g[f"s{k}_f{m}"] for m in range(4)]
        for m in range(4):
            assert np.array_equal(P.mttkrp_factors(t, f, m + 1), g[f"s{k}_mttkrp{m + 1}"])
    t = P.CooTensor(g["sp4_dims"], g["sp4_idx"], g["sp4_vals"])
    res = P.fit(t, 2, None, P.SolverConfig(seed=4, eps_abs=0.0, eps_rel=0.0, n_max=8, max_restarts=0,
                                           track_factors=True), rho_schedule=g["sp4_rho"])
    assert abs(res.rfe - float(g["sp4_rfe"])) <= 1e-9 * float(g["sp4_rfe"])
    for m in range(4):
        assert rel(res.model.factors[m], g[f"sp4_aux{m}"]) <= 1e-9
        for it in range(len(res.factor_history)):
            assert rel(res.factor_history[it][m], g[f"sp4_hist{m}"][it]) <= 1e-9


def test_sharded_tensor_slabs_generated_per_rank(tmp_path):
    """(f)2 slab delivery: a rank's ShardedTensor holds only its three slabs,
    generated straight into HBM (synth.generate_box) or held in pinned host
    memory; the one-rank sharded fit on them is bitwise the sharded fit on
    the whole tensor, and the slabs are byte-identical to the whole tensor's
    sub-arrays (the generator does not depend on the sharding)."""
    import torch
    import torch.distributed as dist

    from paper_1409_2383_b200 import synth

    dims, R = (40, 30, 20), 5
    spec = synth.SynthSpec.make(dims, R, 20.0, 77)
    whole = synth.generate_box(spec, dtype="float32")
    plan = P.PartitionPlan.uniform(dims, 1)
    boxes = P.ShardedTensor.slab_boxes(dims, plan, 0)
    dev = [synth.generate_box(spec, lo, hi, "float32") for lo, hi in boxes]
    for s_, (lo, hi) in zip(dev, boxes):
        assert torch.equal(s_, whole[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]])
    host = [s_.cpu().pin_memory() for s_ in dev]
    kw = dict(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=6, max_restarts=0, inner_sweeps=2, track_factors=True)
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        ref = P.distributed_fit(whole.cpu().numpy(), R, None, P.SolverConfig(**kw), plan=1, sharded=True)
        for slabs in (dev, host):
            got = P.distributed_fit(P.ShardedTensor(dims, plan, 0, slabs), R, None, P.SolverConfig(**kw))
            assert got.residual_history == ref.residual_history and got.rfe == ref.rfe
            for a, b in zip(got.model.factors, ref.model.factors):
                assert np.array_equal(np.asarray(a), np.asarray(b))
        with pytest.raises(ValueError):  # a slab of the wrong shape
            P.distributed_fit(P.ShardedTensor(dims, plan, 0, dev[:2] + [dev[2][:, :, :10].contiguous()]), R)
    finally:
        dist.destroy_process_group()


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_as_processes_on_one_gpu_match_oracle(golden_small, tmp_path, world):
    """distributed_fit with ``world`` real processes sharing the one B200
    (gloo exchange through the host, so no kernel waits on another rank's):
    the sharded engine with genuinely cross-process row gathers, Gram
    closure and norm merge.  Every rank's per-iteration factors within 1e-9
    of the oracle (the north-star bar) and all ranks bitwise identical."""
    import torch.multiprocessing as mp

    from _mp_workers import sharded_fit_worker

    g = golden_small
    kw = dict(MESH2_CFG)
    want = O.fit(g["mesh2_x"], 3, O.Config(**kw))
    mp.spawn(sharded_fit_worker, args=(world, _free_port(), g["mesh2_x"], 3, kw, str(tmp_path)),
             nprocs=world, join=True)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    n = len(want.factor_history)
    assert got[0]["hist0"].shape[0] == n >= 4
    for it in range(n):
        for m in range(3):
            assert rel(got[0][f"hist{m}"][it], want.factor_history[it][m]) <= 1e-9
    for r in range(1, world):
        for k in got[0]:
            assert np.array_equal(got[r][k], got[0][k]), k
    assert abs(float(got[0]["rfe"]) - want.rfe) <= 1e-9 * want.rfe


def test_ranks_generate_own_slabs_fp32(tmp_path):
    """Two processes, each generating only its three slabs of an fp32
    tensor on the device (ShardedTensor), fit it with the tensor-core
    MTTKRP; the final RFE matches the oracle's fit of the whole tensor
    within the north-star fp32 bar (1e-4 relative) and both ranks agree
    bitwise."""
    import torch.multiprocessing as mp

    from _mp_workers import sharded_fit_worker

    dims, R = (96, 80, 72), 8
    kw = dict(seed=5, eps_abs=0.0, eps_rel=0.0, n_max=12, max_restarts=0, inner_sweeps=3)
    x, _, _ = O.generate(dims, R, 20.0, 77, dtype=np.float32)
    want = O.fit(x.astype(np.float64), R, O.Config(**kw))
    mp.spawn(sharded_fit_worker, args=(2, _free_port(), None, R, kw, str(tmp_path),
                                       (dims, R, 20.0, 77, "float32")), nprocs=2, join=True)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(2)]
    assert int(got[0]["iterations"]) == want.iterations
    assert abs(float(got[0]["rfe"]) - want.rfe) <= 1e-4 * want.rfe
    for k in got[0]:
        assert np.array_equal(got[1][k], got[0][k]), k


def test_auto_engine_falls_back_when_block_images_do_not_fit(monkeypatch):
    """engine="auto" on an fp32 tensor keeps one block image per mode (3 |X|
    more HBM).  Where that does not fit, the fit runs on the fp64-arithmetic
    engine, which streams the tensor in place, with a warning, instead of
    failing in cudaMalloc; its result is the fp64 engine's (oracle parity at
    the fp64 bar)."""
    from paper_1409_2383_b200 import engine as E

    rng = np.random.default_rng(4)
    dims, R = (40, 36, 44), 6
    x = (O.reconstruct([rng.random((d, R)) for d in dims]) + 0.02 * rng.standard_normal(dims)).astype(np.float32)
    kw = dict(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=6, max_restarts=0, inner_sweeps=2, track_factors=True)
    P.solver.release_plan_cache()
    monkeypatch.setattr(E, "_free_device_bytes", lambda device, reclaim=False: 1 << 16)
    with pytest.warns(RuntimeWarning, match="block images"):
        got = P.fit(x, R, None, P.SolverConfig(**kw))
    monkeypatch.undo()
    P.solver.release_plan_cache()
    want = O.fit(x.astype(np.float64), R, O.Config(**kw))
    for fg, fw in zip(got.factor_history, want.factor_history):
        for a, b in zip(fg, fw):
            assert rel(a, b) <= 1e-9
    assert got.rfe == pytest.approx(want.rfe, rel=1e-9)


def test_free_hbm_counts_the_idle_pool_and_torch_cache():
    """Released plans leave their block images mapped in the library's
    stream-ordered pool, and freed torch tensors stay in torch's cache: the
    driver reports both as taken, but the next plan can have them.  The
    engine="auto" fit check must count them (a c5 fit() after another c5 plan
    of the same process once fell back to the fp64 engine for this reason)."""
    import torch

    from paper_1409_2383_b200 import _native as Nat
    from paper_1409_2383_b200 import engine as E

    dev = torch.device("cuda:0")
    P.solver.release_plan_cache()
    x = torch.rand((256, 256, 256), dtype=torch.float32, device=dev)  # 64 MB: 192 MB of block images
    kw = dict(seed=1, eps_abs=0.0, eps_rel=0.0, n_max=2, max_restarts=0, inner_sweeps=1)
    import ctypes

    prob = E.DeviceProblem(x, x.shape, 8, P.SolverConfig(**kw), history_capacity=2)
    torch.cuda.synchronize()
    prob.close()
    torch.cuda.synchronize()
    idle = ctypes.c_size_t(0)
    Nat.check(Nat.load().ntf_device_pool_idle_bytes(ctypes.byref(idle)))
    assert idle.value >= 3 * x.numel() * 4
    raw, _ = torch.cuda.mem_get_info(dev)
    assert E._free_device_bytes(dev) >= raw + 3 * x.numel() * 4
    del x, prob  # (the problem keeps a reference to its tensor)
    cached = torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    assert cached >= 64 << 20
    assert E._free_device_bytes(dev, reclaim=True) >= raw + 3 * 64 * (1 << 20) + (64 << 20)
    P.solver.release_plan_cache()
    Nat.check(Nat.load().ntf_device_pool_idle_bytes(ctypes.byref(idle)))
    assert idle.value < 64 << 20  # release_plan_cache trims the pool


@pytest.mark.parametrize("dims,R", [((24, 20, 18), 131), ((17, 9, 33), 200), ((12, 10, 8), 256)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_mttkrp_rank_above_128(dims, R, dtype):
    """Ranks above 128 (the reference only requires rank >= 1,
    solver.py:355-356): the CUDA-core engine in 128-column chunks (grid z),
    every mode, against the oracle at the bars of the rank <= 128 tests."""
    rng = np.random.default_rng(21)
    x = rng.random(dims).astype(dtype)
    f = _factors(rng, dims, R)
    t = O.OracleTensor(x.astype(np.float64))
    for mode in (1, 2, 3):
        got = P.mttkrp_factors(P.DenseTensor(x), f, mode)
        # fp64 arithmetic on either tensor type (fp32 values are exact in fp64)
        assert rel(got, O.mttkrp(t, f, mode)) <= 1e-12


@pytest.mark.parametrize("R,specs", [(150, None), (200, None), (256, None),
                                     (140, ["row_stochastic", "nonneg", "nonneg"])])
def test_fit_rank_above_128_matches_oracle(R, specs):
    """Fits at ranks above 128: row update against L read from the ridge
    buffer (R > 128), ridge Cholesky in place in global memory (R > 160),
    column-chunked MTTKRP; per-iteration factors within 1e-9 of the oracle
    (penalties replayed, as the constraint tests)."""
    rng = np.random.default_rng(R)
    dims = (60, 50, 40)
    x = O.reconstruct([rng.random((d, 6)) for d in dims]) + 0.01 * rng.standard_normal(dims)
    kw = dict(seed=3, eps_abs=0.0, eps_rel=0.0, n_max=6, max_restarts=0, track_factors=True)
    want = O.fit(x, R, O.Config(**kw), specs)
    got = P.fit(x, R, [P.ConstraintSpec.parse(s) for s in specs] if specs else None,
                P.SolverConfig(**kw), rho_schedule=np.array(want.rho_history))
    assert len(got.factor_history) == len(want.factor_history)
    for it in range(len(want.factor_history)):
        for m in range(3):
            assert rel(got.factor_history[it][m], want.factor_history[it][m]) <= 1e-9, (it, m)
    assert abs(got.rfe - want.rfe) <= 1e-9 * want.rfe


def test_sparse_and_order4_rank_above_128():
    """COO MTTKRP in 128-column chunks (grid y) and an order-4 dense fit
    at R = 150 against the oracle's dense fits."""
    rng = np.random.default_rng(9)
    R = 150
    kw = dict(seed=4, eps_abs=0.0, eps_rel=0.0, n_max=5, max_restarts=0, track_factors=True)
    dims = (15, 12, 10)
    x = rng.random(dims) * (rng.random(dims) < 0.3)
    idx = np.argwhere(x != 0)
    coo = P.CooTensor(dims, idx, x[tuple(idx.T)])
    want = O.fit(x, R, O.Config(**kw))
    got = P.fit(coo, R, None, P.SolverConfig(**kw), rho_schedule=np.array(want.rho_history))
    for it in range(len(want.factor_history)):
        for m in range(3):
            assert rel(got.factor_history[it][m], want.factor_history[it][m]) <= 1e-9, (it, m)
    x4 = rng.random((7, 6, 5, 4))
    want4 = O.fit(x4, R, O.Config(**kw))
    got4 = P.fit(x4, R, None, P.SolverConfig(**kw), rho_schedule=np.array(want4.rho_history))
    for it in range(len(want4.factor_history)):
        for m in range(4):
            assert rel(got4.factor_history[it][m], want4.factor_history[it][m]) <= 1e-9, (it, m)
