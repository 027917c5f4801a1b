"""Seeded synthetic NTF workloads (BASELINE.json configs).

Stands in for the paper's synthetic protocol (§VI) and the pattern
of the reference generator (bench.py:34-46): U[0,1) true factors drawn in mode
order from ``PCG64(SeedSequence(data_seed))`` (config 4 additionally zeroes
20% of each factor's entries), a clean tensor [[A,B,C]], and i.i.d.
N(0, sigma^2) noise with sigma^2 set from the Gram-identity ||X0||^2 and the
SNR.

The tensor itself is generated ON THE DEVICE (``ntf_synth_dense``,
csrc/synth.cu): every element is a pure function of its global index (a fixed
order fp64 sum for the clean part, a counter-based SplitMix64 Box-Muller
normal for the noise), so each rank writes only its own slabs straight into
HBM, a 32 GB tensor takes a fraction of a second instead of minutes of host
numpy, and the bytes are the same whatever the sharding.  The host
restatements in ``oracle/`` (numpy and C) reproduce every byte; the golden
fixtures record the sha256 of the tensors the reference was run on.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

DATA_SALT = 101  # reference bench.py:30
FIT_SALT = 202   # reference bench.py:31

_GAMMA = 0x9E3779B97F4A7C15
_MASK = (1 << 64) - 1


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
    return facs


def noise_sigma(factors, snr_db: float) -> float:
    """sigma = sqrt(||X0||^2 / (n 10^(SNR/10))) with ||X0||^2 =
    sum((A^T A) * (B^T B) * (C^T C)); every sum is an exactly rounded
    ``math.fsum``, so sigma (and the tensor) does not depend on the host BLAS."""
    R = factors[0].shape[1]
    prod = None
    for f in factors:
        g = np.empty((R, R))
        for r in range(R):
            for s in range(r, R):
                g[r, s] = g[s, r] = math.fsum(f[:, r] * f[:, s])
        prod = g if prod is None else prod * g
    x0_sq = math.fsum(prod.ravel())
    n = math.prod(int(f.shape[0]) for f in factors)
    return math.sqrt(x0_sq / (n * 10.0 ** (snr_db / 10.0)))


def synth_key(data_seed: int) -> int:
    """Noise key: SplitMix64 output 1 of the data seed."""
    z = (int(data_seed) + _GAMMA) & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


@dataclass
class SynthSpec:
    """Everything that determines a synthetic tensor's bytes."""

    dims: tuple
    rank: int
    snr_db: float
    seed: int
    zero_frac: float
    factors: list       # true factors (host fp64)
    sigma: float
    key: int

    @classmethod
    def make(cls, dims, rank: int, snr_db: float, seed: int, zero_frac: float = 0.0) -> "SynthSpec":
        dims = tuple(int(d) for d in dims)
        f = true_factors(dims, rank, seed, zero_frac)
        return cls(dims, int(rank), float(snr_db), int(seed), float(zero_frac), f,
                   noise_sigma(f, snr_db), synth_key(seed))

    @classmethod
    def of(cls, w: Workload, seed: int | None = None) -> "SynthSpec":
        if seed is None:
            seed = seeds()[0]
        return cls.make(w.dims, w.rank, w.snr_db, seed, w.zero_frac)


def generate_box(spec: SynthSpec, lo=(0, 0, 0), hi=None, dtype="float32", device=None, out=None,
                 factors_dev=None, stream=None):
    """Box [lo, hi) of the tensor written into HBM by ``ntf_synth_dense``.
    Returns a contiguous device tensor (``out`` if given)."""
    from . import _native as N
    from .engine import _torch

    torch = _torch()
    dev = torch.device(device or "cuda")
    hi = spec.dims if hi is None else tuple(int(h) for h in hi)
    lo = tuple(int(v) for v in lo)
    shape = tuple(h - l for l, h in zip(lo, hi))
    tdt = torch.float32 if str(dtype).endswith("32") else torch.float64
    if out is None:
        out = torch.empty(shape, dtype=tdt, device=dev)
    if tuple(out.shape) != shape or out.dtype != tdt or not out.is_contiguous():
        raise ValueError("out must be a contiguous device tensor of the box's shape and dtype")
    if factors_dev is None:
        factors_dev = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in spec.factors]
    arr = lambda v: (ctypes.c_int64 * 3)(*v)  # noqa: E731
    s = stream or torch.cuda.current_stream(dev)
    lib = N.load()
    N.check(lib.ntf_synth_dense(N.NTF_F32 if tdt == torch.float32 else N.NTF_F64, out.data_ptr(),
                                arr(spec.dims), arr(lo), arr(hi), *(f.data_ptr() for f in factors_dev),
                                spec.rank, spec.sigma, spec.key, ctypes.c_void_p(s.cuda_stream)))
    return out


def generate(dims, rank: int, snr_db: float, seed: int, zero_frac: float = 0.0, dtype=np.float64,
             out=None, device=None):
    """Whole tensor as a host numpy array (generated on the device, then
    copied; ``out`` may be e.g. a pinned torch buffer's numpy view) and the
    true factors."""
    from .engine import _torch

    torch = _torch()
    spec = SynthSpec.make(dims, rank, snr_db, seed, zero_frac)
    x = generate_box(spec, dtype=np.dtype(dtype).name, device=device)
    if out is None:
        out = np.empty(spec.dims, dtype=dtype)
    torch.from_numpy(out).copy_(x)
    return out, spec.factors


def initial_rho_trace(dims, rank: int, fit_seed: int) -> float:
    """BASELINE.json's literal 'rho = trace(Gram)/R' from the seeded initial
    factors: trace((C0^T C0) * (B0^T B0)) / R (SURVEY 8(d) mapping)."""
    from .solver import SolverConfig, init_state

    st = init_state(dims, rank, SolverConfig(seed=fit_seed))
    g = (st.factors[2].T @ st.factors[2]) * (st.factors[1].T @ st.factors[1])
    return float(np.trace(g)) / rank
