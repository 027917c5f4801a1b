"""CPU oracle for the NTF hot path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy/scipy restatement of the reference
package's centralized ADMoM non-negative CP solver (``cpadmm``, under
``/root/reference/pkg/src/cpadmm``).  It exists to *check* the B200 product
path, and to time the reference algorithm on host cores for ``bench.py``'s
``cpu_baseline`` leg and ``--impl reference`` arm.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` may import it; the product
package (``paper_1409_2383_b200``) never does, and fails loudly instead of
falling back to it.

Pinning: ``tests/test_oracle.py`` checks every function here against the
reference's own literal golden values (``pkg/tests/test_tensors.py``,
``pkg/tests/test_solver.py``) and against fixtures produced by running the
reference itself in the build container (``tests/golden/make_golden.py`` →
``tests/golden/*.npz``).  Parity is therefore pinned, not self-referential.

Arithmetic follows the reference exactly where it matters for bitwise
reproduction of the reference's trajectories (same operation order, same
BLAS/LAPACK calls): unfolding copy + materialised Khatri-Rao + one GEMM for
the MTTKRP, ``scipy.linalg.cho_factor``/``cho_solve`` for the ridge system.
Every function names the reference lines it restates.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
from scipy.linalg import cho_factor, cho_solve

# ---------------------------------------------------------------------------
# seeds (solver.py:122-140, bench.py:30-31)
# ---------------------------------------------------------------------------

DATA_SALT = 101  # bench.py:30
FIT_SALT = 202  # bench.py:31


def derive_seed(base: int, *key: int) -> int:
    """solver.py:122-125 — first uint64 word of SeedSequence((base, *key))."""
    words = np.random.SeedSequence((int(base),) + tuple(int(k) for k in key))
    return int(words.generate_state(1, np.uint64)[0])


def attempt_entropy(seed: int, attempt: int) -> int:
    """solver.py:128-130 — attempt 0 reuses the seed, restarts hash it."""
    if attempt == 0:
        return int(seed)
    return derive_seed(seed, attempt)


def init_factors(dims: Sequence[int], rank: int, entropy) -> list[np.ndarray]:
    """solver.py:133-140 — mode-1 zero placeholder, others U[0,1) in mode order."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))
    out = [np.zeros((int(dims[0]), rank))]
    out += [gen.random((int(d), rank)) for d in dims[1:]]
    return out


# ---------------------------------------------------------------------------
# tensor algebra (tensors.py)
# ---------------------------------------------------------------------------


def companion_modes(mode: int, order: int) -> list[int]:
    """tensors.py:223-225 — Khatri-Rao companions, highest mode first."""
    return [m for m in range(order, 0, -1) if m != mode]


def unfold(values: np.ndarray, mode: int) -> np.ndarray:
    """tensors.py:174-187 — row axis = mode, columns with the lowest remaining
    mode fastest (element (i,j,k) of the mode-1 unfolding at column j + k*J)."""
    order = values.ndim
    axes = [mode - 1] + [m - 1 for m in companion_modes(mode, order)]
    return np.ascontiguousarray(values.transpose(axes).reshape(values.shape[mode - 1], -1))


def khatri_rao(mats: Sequence[np.ndarray]) -> np.ndarray:
    """tensors.py:203-220 — columnwise Kronecker, first argument slowest,
    right-associated nesting."""
    acc = np.asarray(mats[-1], dtype=np.float64)
    cols = acc.shape[1]
    for m in reversed(mats[:-1]):
        m = np.asarray(m, dtype=np.float64)
        acc = (m[:, None, :] * acc[None, :, :]).reshape(-1, cols)
    return acc


class OracleTensor:
    """Dense fp64 tensor with the reference's cached unfolding copies
    (tensors.py:40-71): the oracle's timing therefore matches the
    reference's memory behaviour (one transpose copy per mode, kept)."""

    def __init__(self, values: np.ndarray):
        self.values = np.array(values, dtype=np.float64, order="C")
        self.values.flags.writeable = False
        self.dims = tuple(int(d) for d in self.values.shape)
        self._unf: dict[int, np.ndarray] = {}
        self._norm: float | None = None

    @property
    def order(self) -> int:
        return len(self.dims)

    def norm(self) -> float:
        """tensors.py:57-61."""
        if self._norm is None:
            self._norm = float(np.linalg.norm(self.values))
        return self._norm

    def unfolding(self, mode: int) -> np.ndarray:
        """tensors.py:63-71."""
        u = self._unf.get(mode)
        if u is None:
            u = unfold(self.values, mode)
            self._unf[mode] = u
        return u


class OracleSparse:
    """Sparse COO tensor (tensors.py:84-132): entries sorted lexicographically,
    indices int64 [nnz][order], values fp64; duplicates rejected."""

    def __init__(self, dims, indices, vals):
        self.dims = tuple(int(d) for d in dims)
        idx = np.asarray(indices, dtype=np.int64).reshape(-1, len(self.dims))
        v = np.asarray(vals, dtype=np.float64).reshape(-1)
        if idx.shape[0] != v.shape[0]:
            raise ValueError("index rows and value count differ")
        if idx.size:
            if idx.min() < 0 or np.any(idx >= np.array(self.dims)):
                raise ValueError("entry index out of bounds")
            order = np.lexsort(tuple(idx[:, m] for m in reversed(range(len(self.dims)))))
            idx, v = idx[order], v[order]
            if np.any(np.all(np.diff(idx, axis=0) == 0, axis=1)):
                raise ValueError("duplicate entry indices")
        self.indices, self.vals = idx, v

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return self.vals.shape[0]

    def norm(self) -> float:
        """tensors.py:114-115."""
        return float(np.linalg.norm(self.vals))


def as_oracle_tensor(t):
    if isinstance(t, (OracleTensor, OracleSparse)):
        return t
    if hasattr(t, "indices") and hasattr(t, "vals"):
        return OracleSparse(t.dims, t.indices, t.vals)
    vals = getattr(t, "values", t)
    return OracleTensor(np.asarray(vals, dtype=np.float64))


def mttkrp(t, factors: Sequence[np.ndarray], mode: int) -> np.ndarray:
    """tensors.py:254-273 — dense: unfolding times materialised KR; sparse:
    per-entry products (highest companion mode first, then the value),
    accumulated with np.add.at in entry order."""
    comp = companion_modes(mode, t.order)
    if isinstance(t, OracleSparse):
        rank = factors[0].shape[1]
        out = np.zeros((t.dims[mode - 1], rank))
        if t.nnz == 0:
            return out
        contrib = factors[comp[0] - 1][t.indices[:, comp[0] - 1], :].copy()
        for m in comp[1:]:
            contrib *= factors[m - 1][t.indices[:, m - 1], :]
        contrib *= t.vals[:, None]
        np.add.at(out, t.indices[:, mode - 1], contrib)
        return out
    kr = khatri_rao([factors[m - 1] for m in comp])
    return t.unfolding(mode) @ kr


def reconstruct(factors: Sequence[np.ndarray]) -> np.ndarray:
    """tensors.py:276-279."""
    if len(factors) == 3:
        return np.einsum("if,jf,kf->ijk", *factors, optimize=True)
    return np.einsum("if,jf,kf,lf->ijkl", *factors, optimize=True)


def rfe(t, factors: Sequence[np.ndarray]) -> float:
    """tensors.py:282-301 — dense: explicit reconstruction; sparse: the Gram
    identity ||X||^2 - 2<X, W> + sum(Hadamard of the factor Grams)."""
    if isinstance(t, OracleSparse):
        tn = t.norm()
        rows = factors[0][t.indices[:, 0], :].copy()
        for m in range(1, t.order):
            rows *= factors[m][t.indices[:, m], :]
        cross = float(np.dot(t.vals, rows.sum(axis=1)))
        gram = None
        for f in factors:
            g = f.T @ f
            gram = g if gram is None else gram * g
        sq = max(tn ** 2 - 2.0 * cross + float(gram.sum()), 0.0)
        return math.sqrt(sq) / tn
    return float(np.linalg.norm(t.values - reconstruct(factors))) / t.norm()


# ---------------------------------------------------------------------------
# solver (solver.py)
# ---------------------------------------------------------------------------


class InvalidPenalty(RuntimeError):
    """solver.py:31-32 (InvalidPenaltyError)."""


@dataclass
class Config:
    """solver.py:35-61 (SolverConfig) — same fields, same defaults."""

    eps_abs: float = 1e-4
    eps_rel: float = 1e-4
    rho_init: float = 1.0
    mu: float = 8.0
    tau_incr: float = 4.0
    tau_decr: float = 2.0
    n_max: int = 400
    max_restarts: int = 10
    inner_sweeps: int = 1
    seed: int = 0
    adapt: bool = True
    track_rfe: bool = False
    track_factors: bool = False


@dataclass
class State:
    """solver.py:64-78 (SolverState)."""

    factors: list
    aux: list
    duals: list
    rho: list
    iteration: int = 0


@dataclass
class Result:
    """solver.py:89-99 (FitResult); residual_history holds (primal, dual)
    tuples of Python floats."""

    factors: list
    rfe: float
    iterations: int
    restarts: int
    converged: bool
    residual_history: list = field(default_factory=list)
    rfe_history: list = field(default_factory=list)
    factor_history: list | None = None
    rho_history: list = field(default_factory=list)
    state: State | None = None


def init_state(dims, rank: int, cfg: Config, attempt: int = 0) -> State:
    """solver.py:143-151."""
    f = init_factors(dims, rank, attempt_entropy(cfg.seed, attempt))
    return State(f, [np.zeros_like(x) for x in f], [np.zeros_like(x) for x in f],
                 [float(cfg.rho_init)] * len(f))


def companion_gram(factors: Sequence[np.ndarray], mode: int) -> np.ndarray:
    """solver.py:196-204 — Hadamard of Grams, highest mode first."""
    g = None
    for m in companion_modes(mode, len(factors)):
        gm = factors[m - 1].T @ factors[m - 1]
        g = gm if g is None else g * gm
    return g


def ridge_factor(gram: np.ndarray, rho: float):
    """solver.py:167-175 — lower Cholesky of gram + rho*I."""
    if rho <= 0:
        raise InvalidPenalty(f"penalty must be positive, got {rho}")
    try:
        return cho_factor(gram + rho * np.eye(gram.shape[0]), lower=True)
    except np.linalg.LinAlgError as exc:  # scipy raises LinAlgError
        raise InvalidPenalty(str(exc)) from exc


def factor_update(t: OracleTensor, factors, aux, dual, rho: float, mode: int,
                  row_sum_one: bool = False) -> np.ndarray:
    """solver.py:207-219 + 178-193 — MTTKRP, ridge Cholesky, rhs, row solve;
    with ``row_sum_one`` (row_stochastic modes) the per-row Lagrange
    correction m = sol + lam g1, g1 = (G+rho I)^-1 1, lam = (1 - sol 1)/sum(g1)."""
    m = mttkrp(t, factors, mode)
    cho = ridge_factor(companion_gram(factors, mode), rho)
    rhs = m + rho * aux - dual
    sol = cho_solve(cho, rhs.T).T
    if not row_sum_one:
        return sol
    ones = np.ones(rhs.shape[1])
    g1 = cho_solve(cho, ones)
    lam = (1.0 - sol @ ones) / float(g1.sum())
    return sol + lam[:, None] * g1[None, :]


def project_nonneg(x: np.ndarray) -> np.ndarray:
    """constraints.py:105-111 — nonneg projection; non-finite input rejected."""
    if not np.all(np.isfinite(x)):
        raise ValueError("cannot project a matrix with non-finite entries")
    return np.maximum(x, 0.0)


_EPS = float(np.finfo(np.float64).eps)


def simplex_rows(m: np.ndarray) -> np.ndarray:
    """constraints.py:72-92 — per-row projection onto the probability simplex
    (sort-and-threshold); rows already feasible (min >= 0, |sum - 1| <= 8 eps n)
    are returned unchanged."""
    m = np.asarray(m, dtype=np.float64)
    n = m.shape[1]
    u = -np.sort(-m, axis=1)
    css = np.cumsum(u, axis=1)
    j = np.arange(1, n + 1)
    k = np.count_nonzero(u * j > css - 1.0, axis=1)
    theta = (css[np.arange(m.shape[0]), k - 1] - 1.0) / k
    out = np.maximum(m - theta[:, None], 0.0)
    feasible = (m.min(axis=1) >= 0.0) & (np.abs(m.sum(axis=1) - 1.0) <= 8.0 * _EPS * n)
    out[feasible] = m[feasible]
    return out


def card_keep(m: np.ndarray, c: int) -> np.ndarray:
    """constraints.py:95-102 — clamp, then keep the c largest entries of the
    whole matrix; ties keep the smaller row-major index."""
    clamped = np.maximum(m, 0.0)
    if c >= clamped.size:
        return clamped
    flat = clamped.reshape(-1)
    order = np.lexsort((np.arange(flat.size), -flat))[:c]
    out = np.zeros_like(flat)
    out[order] = flat[order]
    return out.reshape(m.shape)


def spec_of(spec) -> tuple:
    """(kind, card) from a ConstraintSpec-like object, a config-file name or a tuple."""
    if spec is None:
        return ("nonneg", None)
    if isinstance(spec, tuple):
        return spec
    if isinstance(spec, str):
        if spec.startswith("nonneg_card:"):
            return ("nonneg_card", int(spec.split(":", 1)[1]))
        return (spec, None)
    return (spec.kind, getattr(spec, "card", None))


def project(x: np.ndarray, spec) -> np.ndarray:
    """constraints.py:105-115 — projection onto the spec's constraint set."""
    kind, card = spec_of(spec)
    if not np.all(np.isfinite(x)):
        raise ValueError("cannot project a matrix with non-finite entries")
    if kind == "nonneg":
        return np.maximum(x, 0.0)
    if kind == "nonneg_card":
        return card_keep(x, int(card))
    return simplex_rows(x)


def adapt(rho, primal, dual, cfg: Config) -> list:
    """solver.py:272-292 — three-branch rule, strict '>' and p > 0 guard."""
    out = []
    for r, p, d in zip(rho, primal, dual):
        if p > cfg.mu * d:
            out.append(r * cfg.tau_incr)
        elif d > cfg.mu * p and p > 0:
            out.append(r / cfg.tau_decr)
        else:
            out.append(r)
    return out


def stop_test(primal, dual, st: State, cfg: Config) -> bool:
    """solver.py:258-269 — inclusive thresholds per mode."""
    rank = st.factors[0].shape[1]
    for m in range(len(st.factors)):
        base = math.sqrt(st.factors[m].shape[0] * rank) * cfg.eps_abs
        pthr = base + cfg.eps_rel * max(np.linalg.norm(st.factors[m]), np.linalg.norm(st.aux[m]))
        dthr = base + cfg.eps_rel * np.linalg.norm(st.duals[m])
        if primal[m] > pthr or dual[m] > dthr:
            return False
    return True


def iterate(st: State, t: OracleTensor, cfg: Config, specs=None):
    """solver.py:295-327 — sweeps, then aux/dual/residuals/adaptation."""
    n = len(st.factors)
    specs = [spec_of(s) for s in (specs or [None] * n)]
    f = list(st.factors)
    for _ in range(cfg.inner_sweeps):
        for mode in range(1, n + 1):
            f[mode - 1] = factor_update(t, f, st.aux[mode - 1], st.duals[mode - 1],
                                        st.rho[mode - 1], mode,
                                        specs[mode - 1][0] == "row_stochastic")
    aux = [project(x + y / r, sp) for x, y, r, sp in zip(f, st.duals, st.rho, specs)]
    duals = [y + r * (x - a) for y, r, x, a in zip(st.duals, st.rho, f, aux)]
    primal = tuple(float(np.linalg.norm(x - a)) for x, a in zip(f, aux))
    dual = tuple(r * float(np.linalg.norm(a - p)) for r, a, p in zip(st.rho, aux, st.aux))
    new = State(f, aux, duals, list(st.rho), st.iteration + 1)
    if cfg.adapt:
        new.rho = adapt(st.rho, primal, dual, cfg)
    return new, (primal, dual)


def aux_model_rfe(t: OracleTensor, st: State) -> float:
    """solver.py:330-337 — Gram-identity RFE of the auxiliary model."""
    a = st.aux[0]
    m = mttkrp(t, st.aux, 1)
    g = companion_gram(st.aux, 1)
    sq = t.norm() ** 2 - 2.0 * float(np.sum(a * m)) + float(np.sum((a.T @ a) * g))
    return math.sqrt(max(sq, 0.0)) / t.norm()


def fit(t, rank: int, cfg: Config | None = None, specs=None) -> Result:
    """solver.py:340-403 — one constraint spec per mode (nonneg by default)."""
    cfg = cfg or Config()
    t = as_oracle_tensor(t)
    specs = [spec_of(s) for s in (specs or [None] * len(t.dims))]
    if rank < 1:
        raise ValueError("rank must be >= 1")
    if t.norm() == 0.0:
        raise ValueError("cannot factorize a zero tensor")
    for d, (kind, card) in zip(t.dims, specs):
        if kind == "nonneg_card" and card > d * rank:
            raise ValueError(f"cardinality budget {card} exceeds factor size {d}x{rank}")
    total = 0
    converged = False
    attempt = 0
    st = None
    hist, rfes, fhist, rhos = [], [], [], []
    for attempt in range(cfg.max_restarts + 1):
        st = init_state(t.dims, rank, cfg, attempt)
        hist, rfes, fhist, rhos = [], [], [], []
        for _ in range(cfg.n_max):
            st, res = iterate(st, t, cfg, specs)
            total += 1
            hist.append(res)
            rhos.append(list(st.rho))
            if cfg.track_factors:
                fhist.append([x.copy() for x in st.factors])
            if cfg.track_rfe:
                rfes.append(aux_model_rfe(t, st))
            if stop_test(res[0], res[1], st, cfg):
                converged = True
                break
        if converged:
            break
    return Result(
        factors=[a.copy() for a in st.aux],
        rfe=rfe(t, st.aux),
        iterations=total,
        restarts=attempt,
        converged=converged,
        residual_history=hist,
        rfe_history=rfes,
        factor_history=fhist if cfg.track_factors else None,
        rho_history=rhos,
        state=st,
    )


# ---------------------------------------------------------------------------
# partition plan (blocks.py:47-61) — row ownership for multi-GPU parity
# ---------------------------------------------------------------------------


def uniform_extents(d: int, n: int) -> tuple[int, ...]:
    """blocks.py:48-61 — as even as possible, first d mod n blocks +1 row."""
    if not 1 <= n <= d:
        raise ValueError(f"block count {n} invalid for extent {d}")
    base, extra = divmod(d, n)
    return tuple(base + (1 if i < extra else 0) for i in range(n))


# ---------------------------------------------------------------------------
# synthetic generator (stands in for bench.py:34-46)
# ---------------------------------------------------------------------------
# Counter-based: every element is a pure function of its global index, so
# the device generator (csrc/synth.cu, ntf_synth_dense) writes any slab of it
# and the bytes never depend on the sharding.  Restated twice here: numpy
# (``synth_box``, small boxes, fully vectorised, explicit operation order)
# and C (``synth_oracle.c`` via ``synth_box_c``, OpenMP, for the BASELINE
# sizes make_golden.py and bench.py's CPU legs need).

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_SQRT2 = float.fromhex("0x1.6a09e667f3bcdp+0")
_PIO2 = float.fromhex("0x1.921fb54442d18p+0")
_LN2_HI = float.fromhex("0x1.62e42fee00000p-1")
_LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
_LN_C = [1.0 / (2 * k + 1) for k in range(12)]
_COS_C = [(-1) ** k / math.factorial(2 * k) for k in range(11)]
_SIN_C = [(-1) ** k / math.factorial(2 * k + 1) for k in range(11)]


def _mix64(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def synth_key(data_seed: int) -> int:
    """Generator key: SplitMix64 output 1 of the data seed."""
    z = np.array([int(data_seed) % (1 << 64)], dtype=np.uint64) + _GAMMA
    return int(_mix64(z)[0])


def synth_std_normal(key: int, e) -> np.ndarray:
    """Box-Muller normal of element indices ``e`` (uint64 array): u1, u2 from
    SplitMix64 words 2e+1, 2e+2; ln and cos as fixed polynomials, each
    operation one correctly rounded numpy ufunc (no fused multiply-add)."""
    e = np.asarray(e, dtype=np.uint64)
    k = np.uint64(key)
    with np.errstate(over="ignore"):
        w1 = _mix64(k + (np.uint64(2) * e + np.uint64(1)) * _GAMMA)
        w2 = _mix64(k + (np.uint64(2) * e + np.uint64(2)) * _GAMMA)
    u1 = ((w1 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    mant, ex = np.frexp(u1)
    big = mant * 2.0 > _SQRT2
    m = np.where(big, mant, mant * 2.0)
    E = np.where(big, ex, ex - 1).astype(np.float64)
    s = (m - 1.0) / (m + 1.0)
    s2 = s * s
    p = np.full_like(s, _LN_C[11])
    for c in reversed(_LN_C[:11]):
        p = p * s2
        p = p + c
    lnm = (2.0 * s) * p
    ln = E * _LN2_HI + (E * _LN2_LO + lnm)
    rad = np.sqrt(-2.0 * ln)
    n2 = w2 >> np.uint64(11)
    q = (n2 >> np.uint64(51)).astype(np.int64)
    fi = n2 & np.uint64((1 << 51) - 1)
    sw = fi > np.uint64(1 << 50)
    g = np.where(sw, np.uint64(1 << 51) - fi, fi).astype(np.float64) * 2.0 ** -51
    th = g * _PIO2
    t2 = th * th
    cc = np.full_like(th, _COS_C[10])
    sn = np.full_like(th, _SIN_C[10])
    for a, b in zip(reversed(_COS_C[:10]), reversed(_SIN_C[:10])):
        cc = cc * t2
        cc = cc + a
        sn = sn * t2
        sn = sn + b
    sn = th * sn
    cq = np.where(sw, sn, cc)
    sq = np.where(sw, cc, sn)
    v = np.select([q == 0, q == 1, q == 2], [cq, -sq, -cq], sq)
    return rad * v


def synth_box(factors, dims, lo, hi, sigma: float, key: int, dtype=np.float64) -> np.ndarray:
    """Box [lo, hi) of the generator's tensor (numpy restatement):
    clean = sum_r (A[i,r] B[j,r]) C[k,r] accumulated in r order, plus sigma
    times the element's normal; e = (i J + j) K + k over the full dims."""
    a, b, c = factors
    I, J, K = (int(d) for d in dims)
    ii = np.arange(lo[0], hi[0])[:, None, None]
    jj = np.arange(lo[1], hi[1])[None, :, None]
    kk = np.arange(lo[2], hi[2])[None, None, :]
    acc = np.zeros((len(ii), jj.shape[1], kk.shape[2]))
    for r in range(a.shape[1]):
        ab = a[lo[0]:hi[0], r][:, None, None] * b[lo[1]:hi[1], r][None, :, None]
        acc = acc + ab * c[lo[2]:hi[2], r][None, None, :]
    e = ((ii * J + jj) * K + kk).astype(np.uint64)
    x = acc + sigma * synth_std_normal(key, e)
    return x.astype(dtype)


_SYNTH_LIB = None


def _synth_lib():
    """oracle/libsynth_oracle.so (built by __graft_entry__.build(), or here)."""
    global _SYNTH_LIB
    if _SYNTH_LIB is None:
        import ctypes
        import os
        import subprocess

        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "libsynth_oracle.so")
        src = os.path.join(here, "synth_oracle.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared",
                            "-fPIC", src, "-o", so, "-lm"], check=True)
        lib = ctypes.CDLL(so)
        lib.synth_box.restype = ctypes.c_int
        lib.synth_box.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                                          ctypes.c_int, ctypes.c_void_p]
        lib.synth_std_normal.restype = ctypes.c_double
        lib.synth_std_normal.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _SYNTH_LIB = lib
    return _SYNTH_LIB


def synth_box_c(factors, dims, lo, hi, sigma: float, key: int, dtype=np.float64, out=None) -> np.ndarray:
    """The same box from the C restatement (OpenMP over (i, j) rows)."""
    lib = _synth_lib()
    f = [np.ascontiguousarray(v, dtype=np.float64) for v in factors]
    d = np.array(dims, dtype=np.int64)
    lo_a = np.array(lo, dtype=np.int64)
    hi_a = np.array(hi, dtype=np.int64)
    shape = tuple(int(h - l) for l, h in zip(lo, hi))
    if out is None:
        out = np.empty(shape, dtype=dtype)
    assert out.shape == shape and out.dtype in (np.float32, np.float64) and out.flags.c_contiguous
    rc = lib.synth_box(f[0].ctypes.data, f[1].ctypes.data, f[2].ctypes.data, d.ctypes.data,
                       lo_a.ctypes.data, hi_a.ctypes.data, int(f[0].shape[1]), float(sigma),
                       int(key) % (1 << 64), 1 if out.dtype == np.float32 else 0, out.ctypes.data)
    if rc != 0:
        raise ValueError("synth_box: rank outside 1..4096")
    return out


def true_factors(dims, rank: int, seed: int, zero_frac: float = 0.0):
    """U[0,1) true factors from PCG64(SeedSequence(seed)) in mode order, then
    (zero_frac > 0) each factor's entries zeroed where a further U[0,1) draw
    is below zero_frac, factor by factor."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(int(seed))))
    truth = [gen.random((int(d), rank)) for d in dims]
    if zero_frac > 0:
        for f in truth:
            f[gen.random(f.shape) < zero_frac] = 0.0
    return truth


def noise_sigma(truth, snr_db: float) -> float:
    """sigma^2 = ||X0||^2 / (IJK 10^(SNR/10)), ||X0||^2 by the Gram identity
    sum((A^T A) * (B^T B) * (C^T C)) with every sum an exactly rounded
    math.fsum, so sigma does not depend on the host's BLAS."""
    R = truth[0].shape[1]
    grams = []
    for f in truth:
        g = np.empty((R, R))
        for r in range(R):
            for s_ in range(r, R):
                g[r, s_] = g[s_, r] = math.fsum(f[:, r] * f[:, s_])
        grams.append(g)
    x0_sq = math.fsum(((grams[0] * grams[1]) * grams[2]).ravel())
    n = math.prod(int(f.shape[0]) for f in truth)
    return math.sqrt(x0_sq / (n * 10.0 ** (snr_db / 10.0)))


def generate(dims, rank: int, snr_db: float, seed: int, zero_frac: float = 0.0,
             dtype=np.float64, use_c: bool = True):
    """The whole tensor: (X as ``dtype``, true factors, sigma)."""
    dims = tuple(int(d) for d in dims)
    truth = true_factors(dims, rank, seed, zero_frac)
    sigma = noise_sigma(truth, snr_db)
    key = synth_key(seed)
    fn = synth_box_c if use_c else synth_box
    x = fn(truth, dims, (0, 0, 0), dims, sigma, key, dtype)
    return x, truth, sigma
