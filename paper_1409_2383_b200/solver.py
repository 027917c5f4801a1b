"""Drop-in ``fit`` for the reference ADMoM NTF solver, running on a B200.

Mirrors the reference module ``cpadmm.solver`` (reference solver.py): same
types (``SolverConfig``, ``SolverState``, ``Residuals``, ``FitResult``,
``InvalidPenaltyError``), same seeds, same restart loop and the same
``fit(t, rank, specs=None, config=None) -> FitResult`` signature
(solver.py:340-345).  The outer iterations run on the device through the
C-ABI plan (engine.py / include/ntf_b200.h); the host only seeds the state,
reads the counters and copies the histories back.  There is no CPU fallback.
"""

from __future__ import annotations

import atexit
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .constraints import ConstraintSpec, normalize_specs, plan_codes
from .tensors import CooTensor, DenseTensor, KruskalModel, as_coo, as_dense, is_sparse  # noqa: F401


class InvalidPenaltyError(RuntimeError):
    """Ridge system not positive definite (reference solver.py:31-32)."""


@dataclass
class SolverConfig:
    """Reference SolverConfig (solver.py:35-61): same fields and checks."""

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

    def __post_init__(self):
        if self.eps_abs < 0 or self.eps_rel < 0:
            raise ValueError("stopping tolerances must be >= 0")
        if self.rho_init <= 0:
            raise ValueError("rho_init must be positive")
        if min(self.mu, self.tau_incr, self.tau_decr) <= 1:
            raise ValueError("adaptation parameters mu, tau_incr, tau_decr must be > 1")
        if self.n_max < 1 or self.inner_sweeps < 1 or self.max_restarts < 0:
            raise ValueError("n_max, inner_sweeps must be >= 1 and max_restarts >= 0")


@dataclass
class SolverState:
    """Reference SolverState (solver.py:64-78), host numpy arrays."""

    factors: list
    aux: list
    duals: list
    rho: list
    iteration: int = 0

    @property
    def order(self) -> int:
        return len(self.factors)

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(f.shape[0] for f in self.factors)


@dataclass(frozen=True)
class Residuals:
    """Primal/dual residual norms per mode (solver.py:81-86)."""

    primal: tuple
    dual: tuple


@dataclass
class FitResult:
    """Reference FitResult (solver.py:89-99)."""

    model: KruskalModel
    rfe: float
    iterations: int
    restarts: int
    converged: bool
    residual_history: list = field(default_factory=list)
    rfe_history: list = field(default_factory=list)
    factor_history: list | None = None
    state: SolverState | None = None
    rho_history: list = field(default_factory=list)


# -- seeds (solver.py:122-151): numpy PCG64 streams, bit-identical starts ----

def derive_seed(base: int, *key: int) -> int:
    ss = np.random.SeedSequence((int(base),) + tuple(int(k) for k in key))
    return int(ss.generate_state(1, np.uint64)[0])


def attempt_entropy(seed: int, attempt: int):
    return int(seed) if attempt == 0 else derive_seed(seed, attempt)


def init_factors(dims: Sequence[int], rank: int, entropy) -> list[np.ndarray]:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))
    out = [np.zeros((int(dims[0]), rank))]
    for d in dims[1:]:
        out.append(rng.random((int(d), rank)))
    return out


def init_state(dims: Sequence[int], rank: int, config: SolverConfig, attempt: int = 0) -> SolverState:
    if rank < 1:
        raise ValueError("rank must be >= 1")
    f = init_factors(dims, rank, attempt_entropy(config.seed, attempt))
    return SolverState(f, [np.zeros_like(x) for x in f], [np.zeros_like(x) for x in f],
                       [config.rho_init] * len(f))


# -- device helpers -----------------------------------------------------------

_ENGINE = {"auto": N.ENGINE_AUTO, "cuda_core": N.ENGINE_CUDA_CORE, "tcgen05": N.ENGINE_TCGEN05}


def _engine_code(engine) -> int:
    if engine is None:
        import os

        engine = os.environ.get("NTF_B200_ENGINE", "auto")
    if isinstance(engine, int):
        return engine
    return _ENGINE[str(engine)]


def mttkrp_factors(t, factors: Sequence[np.ndarray], mode: int, engine=None) -> np.ndarray:
    """Device MTTKRP (replaces tensors.mttkrp_factors, tensors.py:254-273):
    dense order 3 or 4 (tensor-core / CUDA-core engines) or sparse COO."""
    from .engine import _torch, device_coo, device_tensor, mttkrp_coo_device, mttkrp_device

    torch = _torch()
    if not 1 <= mode <= 4:
        raise ValueError(f"mode must be in 1..4, got {mode}")
    if is_sparse(t):
        t = as_coo(t)
        x = device_coo(t)
        f = [torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(x.device) for v in factors]
        for m, v in enumerate(f):
            if v.shape[0] != t.dims[m]:
                raise ValueError("factor dims do not match tensor dims")
        out = mttkrp_coo_device(x, f, mode)
        torch.cuda.current_stream(x.device).synchronize()
        return out.cpu().numpy()
    t = as_dense(t)
    if not 1 <= mode <= t.order:
        raise ValueError(f"mode must be in 1..{t.order}, got {mode}")
    x = device_tensor(t)
    f = [torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(x.device) for v in factors]
    if len(f) != t.order:
        raise ValueError("need one factor per mode")
    for m, v in enumerate(f):
        if v.shape[0] != t.dims[m]:
            raise ValueError("factor dims do not match tensor dims")
    if t.order == 4:  # order-3 view with the merged modes' Khatri-Rao pair
        from .engine import kr_pair_device

        I, J, K, L = t.dims
        if mode <= 2:
            xv, fv, vm = x.view(I, J, K * L), [f[0], f[1], kr_pair_device(f[2], f[3])], mode
        else:
            xv, fv, vm = x.view(I * J, K, L), [kr_pair_device(f[0], f[1]), f[2], f[3]], mode - 1
        out = mttkrp_device(xv, fv, vm, _engine_code(engine))
    else:
        out = mttkrp_device(x, f, mode, _engine_code(engine))
    torch.cuda.current_stream(x.device).synchronize()
    return out.cpu().numpy()


def fit(t, rank: int, specs: ConstraintSpec | Sequence[ConstraintSpec] | None = None,
        config: SolverConfig | None = None, *, engine=None, device=None,
        rho_schedule=None) -> FitResult:
    """Constrained CP fit with restarts (reference solver.py:340-403): nonneg,
    nonneg_card:<c> or row_stochastic per mode.

    Same semantics as the reference: per outer iteration ``inner_sweeps``
    Gauss-Seidel sweeps of the ridge update over modes 1..3, then the aux
    projection, dual ascent, residuals, adaptation and the stop test; restarts
    from fresh seeds on non-convergence; the model is the auxiliary copies and
    ``rfe`` is computed by explicit reconstruction (fp64 accumulation).

    ``rho_schedule`` (verification hook, not part of the reference API): an
    ``[n_max, 3]`` penalty sequence to replay instead of adapting, so a
    trajectory can be compared iteration by iteration with the reference's
    even where the adaptation rule's branch is decided by rounding noise
    (``p > 0`` at p ~ 1e-17, solver.py:286-291).
    """
    from .engine import DeviceProblem, device_coo, device_tensor, order3_view, sq_error

    config = config or SolverConfig()
    if is_sparse(t):
        t = as_coo(t)
        specs = normalize_specs(specs, t.order)
        if rank < 1:
            raise ValueError("rank must be >= 1")
        x_norm = t.norm()  # tensors.py:114-115
        if x_norm == 0.0:
            raise ValueError("cannot factorize a zero tensor")
        x = device_coo(t, device)
    else:
        t = as_dense(t)
        specs = normalize_specs(specs, t.order)
        if rank < 1:
            raise ValueError("rank must be >= 1")
        codes = plan_codes(specs, t.dims, rank)
        if rho_schedule is None:
            with _PLAN_CACHE.lease(t, rank, config, _engine_code(engine), codes, device) as hit:
                if hit is not None:  # same geometry as the previous fit: reuse its plan and graph
                    prob, x = hit
                    x_norm = math.sqrt(float(sq_error(order3_view(x)[0])[0].item()))
                    if x_norm == 0.0:
                        raise ValueError("cannot factorize a zero tensor")
                    return _run_fit(prob, x, t.dims, rank, config, x_norm)
        x = device_tensor(t, device)
        x_norm = math.sqrt(float(sq_error(order3_view(x)[0])[0].item()))
        if x_norm == 0.0:
            raise ValueError("cannot factorize a zero tensor")
    codes = plan_codes(specs, t.dims, rank)
    prob = DeviceProblem(x, t.dims, rank, config, history_capacity=config.n_max,
                         engine=_engine_code(engine), rho_schedule=rho_schedule, constraints=codes)
    try:
        return _run_fit(prob, x, t.dims, rank, config, x_norm)
    finally:
        prob.close()


class _PlanCache:
    """The plan of the last dense fit, kept for the next fit of the same
    geometry (shape, dtype, rank, constraints, engine and the config fields
    baked into the plan and its captured graph).  A hit copies the new tensor
    into the plan's own tensor buffer and re-splits the block images
    (``ntf_plan_refresh_tensor``); ``load_state`` then resets the rest, as
    between the reference's restarts.  Saves the plan setup, the graph
    capture and the teardown of every back-to-back fit.

    Only tensors up to ``NTF_B200_PLAN_CACHE_MB`` (default 2048 MB of tensor
    data; the plan holds about four times that) are kept;
    ``NTF_B200_PLAN_CACHE=0`` turns the cache off; ``release_plan_cache()``
    frees it.  One fit at a time uses it (others build their own plan)."""

    def __init__(self):
        import threading

        self._lock = threading.Lock()
        self._key = None
        self._prob = None
        self._x = None

    @staticmethod
    def _enabled(nbytes: int) -> bool:
        import os

        if os.environ.get("NTF_B200_PLAN_CACHE", "1") == "0":
            return False
        return nbytes <= int(os.environ.get("NTF_B200_PLAN_CACHE_MB", "2048")) * (1 << 20)

    def release(self) -> None:
        with self._lock:
            self._drop()

    def _drop(self) -> None:
        if self._prob is not None:
            self._prob.close()
        self._key = self._prob = self._x = None

    def lease(self, t, rank, config, engine, codes, device):
        import contextlib

        from .engine import DeviceProblem, _torch

        torch = _torch()
        vals = t.values
        dt = np.dtype(str(vals.dtype).replace("torch.", "")) if not isinstance(vals, np.ndarray) else vals.dtype
        nbytes = int(np.prod(t.dims)) * dt.itemsize
        dev = torch.device(device or "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        cfg = dict(vars(config))
        for k in ("seed", "rho_init"):  # host-side: loaded by load_state / init_state
            cfg.pop(k, None)
        key = (dev.index, tuple(t.dims), str(dt), int(rank), int(engine), tuple(map(tuple, codes)),
               tuple(sorted((k, repr(v)) for k, v in cfg.items())))
        cache = self

        @contextlib.contextmanager
        def ctx():
            if not cache._enabled(nbytes) or not cache._lock.acquire(blocking=False):
                yield None
                return
            ok = False
            try:
                if cache._key != key:
                    cache._drop()
                    src = _as_torch(torch, vals)
                    x = torch.empty(tuple(t.dims), dtype=src.dtype, device=dev)
                    x.copy_(src, non_blocking=src.device.type == "cpu" and src.is_pinned())
                    prob = DeviceProblem(x, t.dims, rank, config, history_capacity=config.n_max,
                                         engine=engine, constraints=codes)
                    cache._key, cache._prob, cache._x = key, prob, x
                else:
                    prob, x = cache._prob, cache._x
                    src = _as_torch(torch, vals)
                    with torch.cuda.stream(prob.stream):
                        prob.stream.wait_stream(torch.cuda.current_stream(dev))
                        x.copy_(src.reshape(x.shape), non_blocking=src.device.type == "cpu" and src.is_pinned())
                        N.check(prob.lib.ntf_plan_refresh_tensor(prob._plan, prob._sh))
                    torch.cuda.current_stream(dev).wait_stream(prob.stream)
                yield (cache._prob, cache._x)
                ok = True
            finally:
                if not ok:  # an error mid-fit: do not keep a plan of unknown state
                    cache._drop()
                cache._lock.release()

        return ctx()


def _as_torch(torch, vals):
    """Host numpy values as a torch view (read only: we only copy from it)."""
    if not isinstance(vals, np.ndarray):
        return vals
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(np.ascontiguousarray(vals))


_PLAN_CACHE = _PlanCache()


def _release_at_exit() -> None:  # free the plan while CUDA and torch are still up
    try:
        _PLAN_CACHE.release()
    except Exception:  # pragma: no cover - best effort at interpreter exit
        pass


atexit.register(_release_at_exit)


def release_plan_cache() -> None:
    """Free the plan kept for the next same-geometry ``fit`` (see _PlanCache)
    and return the device memory plans keep mapped in the stream-ordered
    pool (ntf_trim_device_pool) to the device."""
    _PLAN_CACHE.release()
    from . import _native as N

    try:
        import torch

        if torch.cuda.is_available():
            N.check(N.load().ntf_trim_device_pool())
    except N.NativeUnavailable:  # pragma: no cover - nothing was allocated
        pass


def _run_fit(prob, x, dims, rank: int, config: SolverConfig, x_norm: float,
             gather=None) -> FitResult:
    """Restart loop shared by ``fit`` and ``distributed_fit``.  ``gather``
    (sharded runs) returns the full aux/dual matrices from the owned rows."""
    per_iter_host = config.track_factors or config.track_rfe
    stoppable = config.eps_abs > 0 or config.eps_rel > 0
    total = 0
    converged = False
    attempt = 0
    res_hist: list = []
    rfe_hist: list = []
    fac_hist: list = []
    rho_hist: list = []
    for attempt in range(config.max_restarts + 1):
        st = init_state(dims, rank, config, attempt)
        prob.load_state(st.factors, st.aux, st.duals, st.rho)
        res_hist, rfe_hist, fac_hist = [], [], []
        done = 0
        stopped = False
        if per_iter_host:
            while done < config.n_max and not stopped:
                prob.step()
                done, stopped = prob.check_status()
                if config.track_factors:
                    fac_hist.append(prob.read_factors())
                if config.track_rfe:
                    rfe_hist.append(prob.aux_model_rfe(x_norm))
        else:
            chunk = 16 if stoppable else config.n_max
            while done < config.n_max and not stopped:
                n = min(chunk, config.n_max - done)
                prob.run(n)
                done, stopped = prob.check_status()
        total += done
        r, rh = prob.histories(done)
        n = len(dims)
        res_hist = [Residuals(tuple(float(v) for v in row[:n]), tuple(float(v) for v in row[n:]))
                    for row in r]
        rho_hist = [list(map(float, row)) for row in rh]
        if stopped:
            converged = True
            break
    factors, aux, duals, rho = prob.read_state()
    if gather is not None:
        aux, duals = gather(aux, duals)
    state = SolverState(factors, aux, duals, rho, iteration=len(res_hist))
    model = KruskalModel(aux)
    _, err_sq = prob.final_sq_error(aux)
    return FitResult(
        model=model,
        rfe=math.sqrt(err_sq) / x_norm,
        iterations=total,
        restarts=attempt,
        converged=converged,
        residual_history=res_hist,
        rfe_history=rfe_hist,
        factor_history=fac_hist if config.track_factors else None,
        state=state,
        rho_history=rho_hist,
    )


_ITER_CACHE: dict = {}


def iterate(state: SolverState, t, specs=None, config: SolverConfig | None = None,
            *, engine=None) -> tuple[SolverState, Residuals]:
    """One outer iteration from ``state`` (reference solver.py:295-327)."""
    from .engine import DeviceProblem, device_coo, device_tensor

    config = config or SolverConfig()
    if is_sparse(t):
        t = as_coo(t)
        x = device_coo(t)
    else:
        t = as_dense(t)
        x = device_tensor(t)
    specs = normalize_specs(specs, t.order)
    rank = state.factors[0].shape[1]
    codes = plan_codes(specs, t.dims, rank)
    key = (id(t), rank, config.inner_sweeps, config.adapt, config.mu, config.tau_incr,
           config.tau_decr, config.eps_abs, config.eps_rel, _engine_code(engine),
           tuple(codes[0]), tuple(codes[1]))
    prob = _ITER_CACHE.get(key)
    if prob is None or prob.x is not x:
        _ITER_CACHE.clear()
        prob = DeviceProblem(x, t.dims, rank, config, history_capacity=1, engine=_engine_code(engine),
                             constraints=codes)
        _ITER_CACHE[key] = prob
    prob.load_state(state.factors, state.aux, state.duals, state.rho)
    prob.run(1, use_graph=False)
    prob.check_status()
    r, _ = prob.histories(1)
    factors, aux, duals, rho = prob.read_state()
    n = len(t.dims)
    res = Residuals(tuple(float(v) for v in r[0][:n]), tuple(float(v) for v in r[0][n:]))
    return SolverState(factors, aux, duals, rho, state.iteration + 1), res
