"""Host-side logic of the drop-in API (CPU only, no device)."""

import numpy as np
import pytest

from oracle import ntf_oracle as O

import paper_1409_2383_b200 as P
from paper_1409_2383_b200 import synth
from paper_1409_2383_b200.constraints import normalize_specs


def test_config_validation_mirrors_reference():
    for bad in (dict(eps_abs=-1), dict(rho_init=0), dict(mu=1.0), dict(n_max=0),
                dict(inner_sweeps=0), dict(max_restarts=-1)):
        with pytest.raises(ValueError):
            P.SolverConfig(**bad)
    c = P.SolverConfig()
    assert (c.eps_abs, c.eps_rel, c.rho_init, c.mu, c.tau_incr, c.tau_decr, c.n_max,
            c.max_restarts, c.inner_sweeps) == (1e-4, 1e-4, 1.0, 8.0, 4.0, 2.0, 400, 10, 1)


def test_specs():
    assert [s.kind for s in normalize_specs(None, 3)] == ["nonneg"] * 3
    with pytest.raises(ValueError):
        normalize_specs([P.ConstraintSpec.nonneg()] * 2, 3)
    assert [s.name() for s in normalize_specs(P.ConstraintSpec.nonneg_card(3), 3)] == \
        ["nonneg_card:3"] * 3
    with pytest.raises(ValueError):
        P.ConstraintSpec("bogus")
    from paper_1409_2383_b200.constraints import plan_codes

    specs = [P.ConstraintSpec.row_stochastic(), P.ConstraintSpec.nonneg_card(7),
             P.ConstraintSpec.nonneg()]
    assert plan_codes(specs, (4, 5, 6), 2) == ([2, 1, 0], [0, 7, 0])
    with pytest.raises(ValueError, match="exceeds factor size"):  # solver.py:359-363
        plan_codes([P.ConstraintSpec.nonneg_card(11)] * 3, (5, 5, 5), 2)


def test_seeds_and_init_state_match_oracle():
    for seed, att in ((0, 0), (7, 0), (7, 1), (123456789, 3)):
        a = P.init_state((4, 5, 6), 3, P.SolverConfig(seed=seed), att)
        b = O.init_state((4, 5, 6), 3, O.Config(seed=seed), att)
        for x, y in zip(a.factors, b.factors):
            assert np.array_equal(x, y)
    assert P.derive_seed(0, 101, 0) == O.derive_seed(0, 101, 0)


def test_partition_plan_uniform():
    p = P.PartitionPlan.uniform((10, 7, 8), 3)
    assert p.extents == (O.uniform_extents(10, 3), O.uniform_extents(7, 3), O.uniform_extents(8, 3))
    assert p.offsets(1) == [0, 4, 7, 10]
    assert p.row_slice(2, 1) == slice(3, 5)
    with pytest.raises(ValueError):
        P.PartitionPlan.uniform((2, 2, 2), 3)


@pytest.mark.parametrize("name", ["c1", "c4", "c5"])
def test_generator_host_parts_match_oracle(name):
    """The host half of the synthetic generator (true factors, sigma, noise
    key) equals the oracle's restatement bit for bit; sigma is a pure
    function of the factors (exactly rounded sums, no BLAS)."""
    w = synth.CONFIGS[name]
    dims = tuple(min(d, 40) for d in w.dims)
    fa = synth.true_factors(dims, w.rank, 99, w.zero_frac)
    fb = O.true_factors(dims, w.rank, 99, w.zero_frac)
    for x, y in zip(fa, fb):
        assert np.array_equal(x, y)
    assert synth.noise_sigma(fa, w.snr_db) == O.noise_sigma(fb, w.snr_db)
    for seed in (0, 99, synth.seeds()[0], 2**64 - 1):
        assert synth.synth_key(seed) == O.synth_key(seed)
    spec = synth.SynthSpec.of(synth.Workload("t", dims, w.rank, w.dtype, w.snr_db, 1, 1, w.zero_frac), 99)
    assert spec.sigma == O.noise_sigma(fb, w.snr_db) and spec.key == O.synth_key(99)
    if w.zero_frac:
        frac = np.mean(np.concatenate([f.ravel() for f in fa]) == 0.0)
        assert 0.15 < frac < 0.25


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_generator_restatements_agree(dtype):
    """The oracle's two restatements of the counter-based generator (numpy and
    C) agree byte for byte on whole tensors and on boxes of them, and a box is
    the same bytes as the whole tensor's sub-array (sharding-independent)."""
    dims, R = (11, 13, 37), 6
    truth = O.true_factors(dims, R, 4, 0.2)
    sigma, key = O.noise_sigma(truth, 20.0), O.synth_key(4)
    whole = O.synth_box(truth, dims, (0, 0, 0), dims, sigma, key, dtype)
    assert np.array_equal(whole, O.synth_box_c(truth, dims, (0, 0, 0), dims, sigma, key, dtype))
    for lo, hi in (((3, 0, 0), (7, 13, 37)), ((0, 5, 0), (11, 9, 37)), ((0, 0, 30), (11, 13, 37)),
                   ((10, 12, 36), (11, 13, 37))):
        box = O.synth_box_c(truth, dims, lo, hi, sigma, key, dtype)
        assert np.array_equal(box, whole[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]])
        assert np.array_equal(box, O.synth_box(truth, dims, lo, hi, sigma, key, dtype))


def test_generator_noise_is_standard_normal():
    """The polynomial Box-Muller equals the libm one to ~1e-15 and its
    moments are those of N(0, 1)."""
    import math

    key = O.synth_key(7)
    e = np.arange(400000, dtype=np.uint64)
    z = O.synth_std_normal(key, e)
    k = np.uint64(key)
    with np.errstate(over="ignore"):
        w1 = O._mix64(k + (np.uint64(2) * e + np.uint64(1)) * O._GAMMA)
        w2 = O._mix64(k + (np.uint64(2) * e + np.uint64(2)) * O._GAMMA)
    u1 = ((w1 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (w2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    zz = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    assert np.max(np.abs(z - zz)) <= 1e-13
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    assert abs(np.mean(z ** 4) - 3.0) < 0.05


def test_dense_tensor_dtypes():
    x = np.ones((2, 3, 4), dtype=np.float32)
    assert P.DenseTensor(x).dtype == np.float32
    assert P.DenseTensor(x.astype(np.float64)).dtype == np.float64
    assert P.DenseTensor(x, dtype=np.float64).dtype == np.float64
    with pytest.raises(ValueError):
        P.DenseTensor(np.ones((2, 2)))
    t = P.DenseTensor(np.ones((2, 2, 2)))
    with pytest.raises(ValueError):
        t.values[0, 0, 0] = 3.0


def test_no_cpu_fallback():
    """The product path fails loudly without a CUDA device."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1409_2383_b200._native import NativeUnavailable

    with pytest.raises(NativeUnavailable):
        P.fit(np.ones((3, 3, 3)), 1)
    with pytest.raises(NativeUnavailable):
        P.mttkrp_factors(np.ones((3, 3, 3)), [np.ones((3, 1))] * 3, 1)


def test_product_never_imports_oracle():
    import os
    import re

    pkg = os.path.dirname(P.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f


def test_peer_rows_validates_blocks_before_any_cuda_call():
    """distributed._PeerRows (NVLink row all-gather) rejects row blocks that
    are not contiguous or do not cover the factor before allocating."""
    import types

    import torch

    from paper_1409_2383_b200.distributed import _PeerRows

    comm = types.SimpleNamespace(size=2, rank=0)
    full = torch.zeros(10, 3, dtype=torch.float64)
    with pytest.raises(ValueError, match="contiguous"):
        _PeerRows(comm, full, [0, 6], [5, 4])
    with pytest.raises(ValueError, match="cover"):
        _PeerRows(comm, full, [0, 5], [5, 4])


def test_sharded_tensor_boxes_and_validation():
    """ShardedTensor (one rank's three slabs): the slab boxes
    follow the uniform row plan, and slabs of the wrong shape or mixed dtypes
    are rejected before any device work."""
    import torch

    plan = P.PartitionPlan.uniform((10, 7, 8), 3)
    boxes = P.ShardedTensor.slab_boxes((10, 7, 8), plan, 1)
    assert boxes == [((4, 0, 0), (7, 7, 8)), ((0, 3, 0), (10, 5, 8)), ((0, 0, 3), (10, 7, 6))]
    x = torch.arange(560, dtype=torch.float32).reshape(10, 7, 8)
    slabs = [x[4:7].contiguous(), x[:, 3:5].contiguous(), x[:, :, 3:6].contiguous()]
    P.ShardedTensor((10, 7, 8), plan, 1, slabs).validate()
    with pytest.raises(ValueError, match="does not match"):
        P.ShardedTensor((10, 7, 8), plan, 0, slabs).validate()
    with pytest.raises(ValueError, match="one dtype"):
        P.ShardedTensor((10, 7, 8), plan, 1, [slabs[0], slabs[1].double(), slabs[2]]).validate()
    with pytest.raises(ValueError, match="plan and dims"):
        P.ShardedTensor((10, 7, 9), plan, 1, slabs).validate()
