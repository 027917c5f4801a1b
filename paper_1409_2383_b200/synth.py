"""Seeded synthetic NTF workloads (BASELINE.json configs).

Stands in for the paper's synthetic protocol (§VI) and the pattern of
the reference generator (bench.py:34-46): U[0,1) true factors drawn in mode
order (config 4 additionally zeroes 20% of each factor's entries), a clean
tensor [[A,B,C]], and i.i.d. N(0, sigma^2) noise with sigma^2 set from the
exact Gram-identity ||X0||^2 and the SNR.  Noise is drawn slab by slab along
mode 1, which is bit-identical to a one-shot draw, so a rank can generate
only its own slabs and the oracle sees identical values.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DATA_SALT = 101  # reference bench.py:30
FIT_SALT = 202   # reference bench.py:31


@dataclass(frozen=True)
class Workload:
    name: str
    dims: tuple
    rank: int
    dtype: str        # "float64" | "float32"
    snr_db: float
    inner: int
    outer: int
    zero_frac: float = 0.0


CONFIGS = {
    "c1": Workload("c1", (100, 100, 100), 10, "float64", 20.0, 10, 50),
    "c2": Workload("c2", (400, 400, 400), 20, "float32", 20.0, 10, 100),
    "c3": Workload("c3", (1000, 1000, 1000), 50, "float32", 30.0, 5, 50),
    "c4": Workload("c4", (5000, 500, 200), 32, "float32", 20.0, 10, 50, 0.2),
    "c5": Workload("c5", (2000, 2000, 2000), 100, "float32", 20.0, 5, 20),
}


def seeds(base: int = 0, realization: int = 0) -> tuple[int, int]:
    """(data_seed, fit_seed) = derive_seed(base, salt, r) (reference bench.py:129-130)."""
    from .solver import derive_seed

    return derive_seed(base, DATA_SALT, realization), derive_seed(base, FIT_SALT, realization)


def true_factors(dims, rank: int, seed: int, zero_frac: float = 0.0):
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(int(seed))))
    facs = [gen.random((int(d), rank)) for d in dims]
    if zero_frac > 0.0:
        for f in facs:
            f[gen.random(f.shape) < zero_frac] = 0.0
    return facs, gen


def noise_sigma(factors, snr_db: float) -> float:
    g = np.ones((factors[0].shape[1],) * 2)
    for f in factors:
        g = g * (f.T @ f)
    x0_sq = float(g.sum())
    n = math.prod(f.shape[0] for f in factors)
    return math.sqrt(x0_sq / (n * 10.0 ** (snr_db / 10.0)))


def generate(dims, rank: int, snr_db: float, seed: int, zero_frac: float = 0.0, dtype=np.float64,
             out=None, slab_rows: int | None = None):
    """Host tensor (numpy, or into ``out`` e.g. a pinned torch buffer's numpy
    view) and the true factors."""
    dims = tuple(int(d) for d in dims)
    facs, gen = true_factors(dims, rank, seed, zero_frac)
    sigma = noise_sigma(facs, snr_db)
    a, b, c = facs
    x = out if out is not None else np.empty(dims, dtype=dtype)
    rows = slab_rows or max(1, (1 << 22) // max(1, dims[1] * dims[2]))
    for i0 in range(0, dims[0], rows):
        i1 = min(dims[0], i0 + rows)
        clean = np.einsum("if,jf,kf->ijk", a[i0:i1], b, c, optimize=True)
        x[i0:i1] = clean + gen.normal(0.0, sigma, size=(i1 - i0, dims[1], dims[2]))
    return x, facs


def initial_rho_trace(dims, rank: int, fit_seed: int) -> float:
    """BASELINE.json's literal 'rho = trace(Gram)/R' from the seeded initial
    factors: trace((C0^T C0) * (B0^T B0)) / R (SURVEY 8(d) mapping)."""
    from .solver import SolverConfig, init_state

    st = init_state(dims, rank, SolverConfig(seed=fit_seed))
    g = (st.factors[2].T @ st.factors[2]) * (st.factors[1].T @ st.factors[1])
    return float(np.trace(g)) / rank
