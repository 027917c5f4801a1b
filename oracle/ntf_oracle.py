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
# synthetic generator (pattern of bench.py:34-46)
# ---------------------------------------------------------------------------


def generate(dims, rank: int, snr_db: float, seed: int, zero_frac: float = 0.0,
             dtype=np.float64, slab_rows: int | None = None):
    """Seeded noisy low-rank tensor: U[0,1) factors in mode order (optionally
    zeroed with probability ``zero_frac`` factor by factor), X0 = [[A,B,C]],
    sigma^2 from the exact Gram-identity ||X0||^2 and the SNR, N(0, sigma^2)
    noise drawn slab by slab along mode 1 (bit-identical to a one-shot draw).
    Returns (X as ``dtype``, true factors, sigma)."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(int(seed))))
    dims = tuple(int(d) for d in dims)
    truth = [gen.random((d, rank)) for d in dims]
    if zero_frac > 0:
        for f in truth:
            f[gen.random(f.shape) < zero_frac] = 0.0
    g = np.ones((rank, rank))
    for f in truth:
        g = g * (f.T @ f)
    x0_sq = float(g.sum())
    sigma2 = x0_sq / (math.prod(dims) * 10.0 ** (snr_db / 10.0))
    sigma = math.sqrt(sigma2)
    a, b, c = truth
    out = np.empty(dims, dtype=dtype)
    rows = slab_rows or max(1, (1 << 22) // max(1, dims[1] * dims[2]))
    for i0 in range(0, dims[0], rows):
        i1 = min(dims[0], i0 + rows)
        clean = np.einsum("if,jf,kf->ijk", a[i0:i1], b, c, optimize=True)
        noise = gen.normal(0.0, sigma, size=(i1 - i0, dims[1], dims[2]))
        out[i0:i1] = clean + noise
    return out, truth, sigma
