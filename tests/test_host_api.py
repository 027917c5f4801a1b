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


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_generator_matches_oracle(name):
    w = synth.CONFIGS[name]
    dims = tuple(min(d, 40) for d in w.dims)
    a, fa = synth.generate(dims, w.rank, w.snr_db, 99, w.zero_frac, dtype=np.float64, slab_rows=3)
    b, fb, _ = O.generate(dims, w.rank, w.snr_db, 99, w.zero_frac)
    assert np.array_equal(a, b)
    for x, y in zip(fa, fb):
        assert np.array_equal(x, y)
    if w.zero_frac:
        frac = np.mean(np.concatenate([f.ravel() for f in fa]) == 0.0)
        assert 0.15 < frac < 0.25


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
