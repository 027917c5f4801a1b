"""Device-resident solver state and the C-ABI plan that drives it.

``DeviceProblem`` owns (through torch's caching allocator) the HBM copy of the
tensor, the per-mode state (factors, aux, duals, Grams, penalties) and the
per-iteration history buffers, and wraps one ``ntf_plan`` (include/ntf_b200.h)
that enqueues outer iterations on a dedicated CUDA stream.  The host never
synchronises inside a run; histories are copied back once.

HBM layout (row-major, fp64 unless noted):
  X                  I*J*K   fp32 or fp64 (the tensor is read, never copied)
  factors[m]         I_m x R   working factors (replicated across ranks)
  aux[m], duals[m]   I_m x R   (owned rows only when sharded)
  grams[m]           R x R     F_m^T F_m, refreshed by each mode update
  rho[3], norm_acc[3][5][2] (scale, ssq), counters int32[4]
  resid_history      cap x 6,  rho_history cap x 3
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise N.NativeUnavailable("torch is required for device memory") from exc
    if not torch.cuda.is_available():
        raise N.NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return torch


def _ptr(t) -> int:
    return t.data_ptr()


def device_tensor(t, device=None):
    """Return the HBM copy of DenseTensor ``t`` (uploaded once and cached on it;
    pinned host buffers upload asynchronously)."""
    torch = _torch()
    dev = torch.device(device or "cuda")
    vals = t.values
    cache = getattr(t, "_device_cache", None)
    if cache is not None and cache.device == dev:
        return cache
    if isinstance(vals, np.ndarray):
        import warnings

        with warnings.catch_warnings():  # read-only source: we only read it
            warnings.simplefilter("ignore", UserWarning)
            host = torch.from_numpy(np.ascontiguousarray(vals))
        x = host.to(dev)
    else:
        x = vals.to(dev, non_blocking=bool(vals.is_pinned()) if vals.device.type == "cpu" else False)
    x = x.contiguous()
    try:
        t._device_cache = x
    except AttributeError:
        pass
    return x


def dtype_code(x) -> int:
    torch = _torch()
    if x.dtype == torch.float32:
        return N.NTF_F32
    if x.dtype == torch.float64:
        return N.NTF_F64
    raise ValueError("tensor must be float32 or float64")


def _stream_handle(stream) -> ctypes.c_void_p:
    return ctypes.c_void_p(stream.cuda_stream)


def sq_error(x, factors=None, stream=None):
    """(sum x^2, sum (x - [[A,B,C]])^2) on the device, fp64 accumulation."""
    torch = _torch()
    lib = N.load()
    I, J, K = (int(d) for d in x.shape)
    ws_bytes = lib.ntf_sq_error_workspace_bytes(I, J, K)
    ws = torch.empty(max(1, ws_bytes // 8 + 1), dtype=torch.float64, device=x.device)
    out = torch.zeros(2, dtype=torch.float64, device=x.device)
    s = stream or torch.cuda.current_stream(x.device)
    if factors is None:
        a = b = c = None
        R = 0
    else:
        f = [torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64)).to(x.device)
             if isinstance(v, np.ndarray) else v.contiguous() for v in factors]
        a, b, c = (_ptr(v) for v in f)
        R = int(f[0].shape[1])
    N.check(lib.ntf_sq_error(dtype_code(x), _ptr(x), I, J, K, a, b, c, R, _ptr(out), _ptr(ws),
                             ws.numel() * 8, _stream_handle(s)))
    return out


class DeviceCoo:
    """HBM copy of a CooTensor for the COO engine (include/ntf_b200.h
    NTF_FORMAT_COO): lexicographic entries, and per mode a stable order of
    the entries by that mode's index with its row segments (built on the
    host once per tensor, then uploaded)."""

    def __init__(self, t, device=None):
        torch = _torch()
        dev = torch.device(device or "cuda")
        self.dims = tuple(int(d) for d in t.dims)
        self.order = len(self.dims)
        self.shape = self.dims
        self.nnz = int(t.vals.shape[0])
        self.device = dev
        self.dtype = torch.float64
        idx = np.ascontiguousarray(t.indices, dtype=np.int64).reshape(-1, self.order)
        self.idx = torch.from_numpy(idx.copy()).to(dev)
        self.vals = torch.from_numpy(np.ascontiguousarray(t.vals, dtype=np.float64).copy()).to(dev)
        self._dims_arr = (ctypes.c_int64 * 4)(*(list(self.dims) + [0] * (4 - self.order)))
        self.perm, self.rowptr = [], []
        for m in range(self.order):
            key = idx[:, m]
            if m == 0:  # lexicographic order is already sorted by the first index
                self.perm.append(None)
                sk = key
            else:
                order = np.argsort(key, kind="stable")
                self.perm.append(torch.from_numpy(order.astype(np.int64)).to(dev))
                sk = key[order]
            rp = np.searchsorted(sk, np.arange(self.dims[m] + 1), side="left").astype(np.int64)
            self.rowptr.append(torch.from_numpy(rp).to(dev))

    def data_ptr(self) -> int:
        return self.vals.data_ptr() if self.nnz else self.rowptr[0].data_ptr()

    def ptr_idx(self):
        return self.idx.data_ptr() if self.nnz else None

    def ptr_perm(self, m):
        p = self.perm[m]
        return p.data_ptr() if (p is not None and self.nnz) else None


def device_coo(t, device=None) -> DeviceCoo:
    """The DeviceCoo of CooTensor ``t`` (built once and cached on it)."""
    torch = _torch()
    dev = torch.device(device or "cuda")
    cache = getattr(t, "_device_cache", None)
    if isinstance(cache, DeviceCoo) and cache.device == dev:
        return cache
    d = DeviceCoo(t, dev)
    try:
        t._device_cache = d
    except AttributeError:
        pass
    return d


def _ptr_array(tensors):
    arr = (ctypes.c_void_p * 4)()
    for i, t in enumerate(tensors):
        arr[i] = _ptr(t)
    return arr


def mttkrp_coo_device(x: DeviceCoo, factors, mode: int, stream=None):
    torch = _torch()
    lib = N.load()
    R = int(factors[0].shape[1])
    out = torch.empty((x.dims[mode - 1], R), dtype=torch.float64, device=x.device)
    s = stream or torch.cuda.current_stream(x.device)
    fa = _ptr_array(factors)
    N.check(lib.ntf_mttkrp_coo(x.order, ctypes.addressof(x._dims_arr), mode, x.nnz, x.ptr_idx(),
                               x.vals.data_ptr() if x.nnz else None, x.ptr_perm(mode - 1),
                               _ptr(x.rowptr[mode - 1]), ctypes.addressof(fa), R, _ptr(out),
                               _stream_handle(s)))
    return out


def coo_sq_error(x: DeviceCoo, factors=None, stream=None):
    """(sum x^2, ||X - [[A,B,C]]||^2 by the Gram identity) on the device."""
    torch = _torch()
    lib = N.load()
    wsb = lib.ntf_sq_error_coo_workspace_bytes(x.nnz)
    ws = torch.empty(max(1, wsb // 8 + 1), dtype=torch.float64, device=x.device)
    out = torch.zeros(2, dtype=torch.float64, device=x.device)
    s = stream or torch.cuda.current_stream(x.device)
    fa = None
    R = 0
    if factors is not None:
        f = [torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64)).to(x.device)
             if isinstance(v, np.ndarray) else v.contiguous() for v in factors]
        fa = _ptr_array(f)
        R = int(f[0].shape[1])
    N.check(lib.ntf_sq_error_coo(x.order, ctypes.addressof(x._dims_arr), x.nnz, x.ptr_idx(),
                                 x.vals.data_ptr() if x.nnz else None,
                                 ctypes.addressof(fa) if fa is not None else None, R, _ptr(out),
                                 _ptr(ws), ws.numel() * 8, _stream_handle(s)))
    return out


def kr_pair_device(Fa, Fb, stream=None):
    """Khatri-Rao pair rows a*nb + b = Fa[a] * Fb[b] (ntf_khatri_rao_pair)."""
    torch = _torch()
    lib = N.load()
    na, R = (int(v) for v in Fa.shape)
    nb = int(Fb.shape[0])
    out = torch.empty((na * nb, R), dtype=torch.float64, device=Fa.device)
    s = stream or torch.cuda.current_stream(Fa.device)
    N.check(lib.ntf_khatri_rao_pair(_ptr(Fa), na, _ptr(Fb), nb, R, _ptr(out), _stream_handle(s)))
    return out


def order3_view(x, factors=None, stream=None):
    """An order-4 tensor as the order-3 view I x J x (K L) and its model
    [A, B, C o D] (the merged mode's Khatri-Rao pair formed on the device);
    order-3 inputs are returned unchanged."""
    if x.dim() == 3:
        return x, factors
    I, J, K, L = (int(d) for d in x.shape)
    xv = x.view(I, J, K * L)
    if factors is None:
        return xv, None
    torch = _torch()
    f = [torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64)).to(x.device)
         if isinstance(v, np.ndarray) else v.contiguous() for v in factors]
    return xv, [f[0], f[1], kr_pair_device(f[2], f[3], stream)]


def tensor_norm(t) -> float:
    x, _ = order3_view(device_tensor(t))
    return float(np.sqrt(sq_error(x)[0].item()))


def mttkrp_device(x, factors, mode: int, engine: int = N.ENGINE_AUTO, stream=None):
    """Dense MTTKRP of the device tensor ``x`` with device fp64 factors."""
    torch = _torch()
    lib = N.load()
    I, J, K = (int(d) for d in x.shape)
    R = int(factors[0].shape[1])
    code = dtype_code(x)
    wsb = lib.ntf_mttkrp_workspace_bytes(mode, code, I, J, K, R, engine)
    if wsb == 0:
        N.check(N.NTF_ERR_INVALID)
    ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=x.device)
    M = (I, J, K)[mode - 1]
    out = torch.empty((M, R), dtype=torch.float64, device=x.device)
    s = stream or torch.cuda.current_stream(x.device)
    a, b, c = (_ptr(f) for f in factors)
    N.check(lib.ntf_mttkrp(mode, code, _ptr(x), I, J, K, a, b, c, R, _ptr(out), _ptr(ws),
                           ws.numel() * 8, engine, _stream_handle(s)))
    return out


def gram_device(F, stream=None):
    torch = _torch()
    lib = N.load()
    rows, R = (int(d) for d in F.shape)
    wsb = lib.ntf_gram_workspace_bytes(rows, R)
    ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=F.device)
    G = torch.empty((R, R), dtype=torch.float64, device=F.device)
    s = stream or torch.cuda.current_stream(F.device)
    N.check(lib.ntf_gram(_ptr(F), rows, R, _ptr(G), _ptr(ws), ws.numel() * 8, _stream_handle(s)))
    return G


@dataclass
class Slabs:
    """This rank's view of the tensor for each mode."""

    x_mode: list            # 3 device tensors
    row_offset: tuple
    row_count: tuple


_SOLVER_STREAMS: dict = {}


def _solver_stream(device):
    """One solver stream per device for every plan of the process.  torch's
    caching allocator keeps freed blocks per stream: a fresh stream per fit
    made each fit's state allocations miss the cache now and then (a
    synchronous cudaMalloc, tens of ms when it also had to free cached
    blocks), which showed up as outliers in back-to-back fit() calls."""
    torch = _torch()
    key = torch.device(device).index
    s = _SOLVER_STREAMS.get(key)
    if s is None:
        s = _SOLVER_STREAMS[key] = torch.cuda.Stream(device=device)
    return s


def _free_device_bytes(device, reclaim: bool = False) -> int:
    """HBM a new plan can take on ``device`` (a function so that tests can
    shrink it): what the driver reports as free plus what the library's
    stream-ordered pool holds mapped but idle (released plans leave their block
    images there, and the next plan allocates from them first).  ``reclaim``
    first hands torch's cached, unused blocks back to the driver."""
    torch = _torch()
    if reclaim:
        torch.cuda.synchronize(device)
        torch.cuda.empty_cache()
    idle = ctypes.c_size_t(0)
    with torch.cuda.device(device):
        free, _ = torch.cuda.mem_get_info(device)
        N.check(N.load().ntf_device_pool_idle_bytes(ctypes.byref(idle)))
    return int(free) + int(idle.value)


def _engine_that_fits(engine: int, slabs, rank: int, device) -> int:
    """ENGINE_AUTO on fp32 tensors means the tensor-core engine, which keeps
    one block image per mode: as many bytes again as each mode's tensor or
    slab (DESIGN 2).  Where those do not fit the free HBM, fall back to the
    fp64-arithmetic engine, which streams the tensor in place (slower, and
    more exact), instead of failing in cudaMalloc."""
    torch = _torch()
    if engine != N.ENGINE_AUTO or rank > 128:
        return engine
    xs = [x for x in slabs if not isinstance(x, DeviceCoo)]
    if not xs or any(x.dtype != torch.float32 for x in xs):
        return engine
    need = sum(x.numel() * 4 for x in xs)
    free = _free_device_bytes(device)
    if need > 0.97 * free:  # count torch's cached blocks before giving up the tensor cores
        free = _free_device_bytes(device, reclaim=True)
    if need <= 0.97 * free:
        return engine
    import warnings

    warnings.warn(f"the tensor-core engine's block images need {need / 2**30:.1f} GiB but {free / 2**30:.1f} GiB "
                  "of HBM are free: using the fp64-arithmetic engine (engine='cuda_core'), which streams "
                  "the tensor in place", RuntimeWarning, stacklevel=3)
    return N.ENGINE_CUDA_CORE


class DeviceProblem:
    """HBM state of one fit and its C-ABI plan."""

    def __init__(self, x, dims, rank: int, config, history_capacity: int, engine: int = N.ENGINE_AUTO,
                 slabs: Slabs | None = None, stream=None, rho_schedule=None,
                 norm_parts: int = 1, constraints=None):
        torch = _torch()
        self.torch = torch
        self.lib = N.load()
        self.device = x.device
        self.dims = tuple(int(d) for d in dims)
        self.R = int(rank)
        self.config = config
        self.x = x
        self.stream = stream or _solver_stream(self.device)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        self.sharded = slabs is not None
        self.order = Nm = len(self.dims)
        if slabs is None:
            slabs = Slabs([x] * Nm, (0,) * Nm, self.dims)
        self.slabs = slabs
        engine = _engine_that_fits(int(engine), slabs.x_mode, int(rank), self.device)
        dev, f64 = self.device, torch.float64
        R = self.R
        with torch.cuda.stream(self.stream):
            self.factors = [torch.zeros((d, R), dtype=f64, device=dev) for d in self.dims]
            self.aux = [torch.zeros((c, R), dtype=f64, device=dev) for c in slabs.row_count]
            self.duals = [torch.zeros((c, R), dtype=f64, device=dev) for c in slabs.row_count]
            self.grams = [torch.zeros((R, R), dtype=f64, device=dev) for _ in range(Nm)]
            self.colmax = torch.zeros((Nm, R), dtype=f64, device=dev)
            self.rho = torch.zeros(Nm, dtype=f64, device=dev)
            self.norm_acc = torch.zeros(10 * Nm, dtype=f64, device=dev)
            # every shard's norm_acc, gathered before finalize (sharded runs)
            self.norm_all = (torch.zeros(norm_parts * 10 * Nm, dtype=f64, device=dev)
                             if norm_parts > 1 or self.sharded else None)
            cap = max(1, int(history_capacity))
            self.cap = cap
            self.resid_hist = torch.zeros((cap, 2 * Nm), dtype=f64, device=dev)
            self.rho_hist = torch.zeros((cap, Nm), dtype=f64, device=dev)
            self.counters = torch.zeros(4, dtype=torch.int32, device=dev)
        d = N.PlanDesc()
        d.order = Nm
        d.x_dtype = dtype_code(x)
        for m in range(Nm):
            xs = slabs.x_mode[m]
            d.x_mode[m] = _ptr(xs)
            for a in range(len(xs.shape)):
                d.x_dims[m][a] = int(xs.shape[a])
            d.dims[m] = self.dims[m]
            d.row_offset[m] = int(slabs.row_offset[m])
            d.row_count[m] = int(slabs.row_count[m])
            d.factors[m] = _ptr(self.factors[m])
            d.aux[m] = _ptr(self.aux[m])
            d.duals[m] = _ptr(self.duals[m])
            d.grams[m] = _ptr(self.grams[m])
        for m in range(Nm, 4):  # unused entries of the fixed-size descriptor
            d.dims[m] = 0
        d.colmax = _ptr(self.colmax)
        d.rank = R
        d.engine = int(engine)
        d.fuse_gram = 1  # the row update forms the Gram / column maxima of its rows (sharded: owned rows)
        d.eps_abs = float(config.eps_abs)
        d.eps_rel = float(config.eps_rel)
        d.mu = float(config.mu)
        d.tau_incr = float(config.tau_incr)
        d.tau_decr = float(config.tau_decr)
        d.inner_sweeps = int(config.inner_sweeps)
        d.adapt = 1 if config.adapt else 0
        d.rho = _ptr(self.rho)
        d.norm_acc = _ptr(self.norm_acc)
        if self.norm_all is not None:
            d.norm_all = _ptr(self.norm_all)
            d.norm_parts = int(norm_parts)
        if isinstance(x, DeviceCoo):
            d.x_format = N.NTF_FORMAT_COO
            d.nnz = x.nnz
            d.coo_idx = x.ptr_idx()
            d.coo_vals = x.vals.data_ptr() if x.nnz else None
            for m in range(x.order):
                d.coo_perm[m] = x.ptr_perm(m)
                d.coo_rowptr[m] = _ptr(x.rowptr[m])
        if constraints is not None:  # (codes, cards), constraints.plan_codes
            for m in range(Nm):
                d.constraint[m] = int(constraints[0][m])
                d.card[m] = int(constraints[1][m])
        d.history_capacity = cap
        d.resid_history = _ptr(self.resid_hist)
        d.rho_history = _ptr(self.rho_hist)
        d.counters = _ptr(self.counters)
        self._rho_schedule = None
        if rho_schedule is not None:
            sched = np.zeros((cap, Nm))
            rs = np.asarray(rho_schedule, dtype=np.float64).reshape(-1, Nm)[:cap]
            sched[: len(rs)] = rs
            self._rho_schedule = torch.from_numpy(sched).to(dev)
            d.rho_schedule = _ptr(self._rho_schedule)
        self._desc = d
        handle = ctypes.c_void_p()
        N.check(self.lib.ntf_plan_create(ctypes.byref(d), ctypes.byref(handle)))
        self._plan = handle
        self._sh = _stream_handle(self.stream)

    # -- state transfer ------------------------------------------------------
    def load_state(self, factors, aux, duals, rho) -> None:
        """Host (numpy) state -> HBM, counters reset, Grams refreshed."""
        torch = self.torch
        off, cnt = self.slabs.row_offset, self.slabs.row_count
        with torch.cuda.stream(self.stream):
            for m in range(self.order):
                self.factors[m].copy_(torch.from_numpy(np.ascontiguousarray(factors[m], dtype=np.float64)))
                a = np.ascontiguousarray(aux[m], dtype=np.float64)
                y = np.ascontiguousarray(duals[m], dtype=np.float64)
                if a.shape[0] != cnt[m]:
                    a = a[off[m]:off[m] + cnt[m]]
                    y = y[off[m]:off[m] + cnt[m]]
                self.aux[m].copy_(torch.from_numpy(np.ascontiguousarray(a)))
                self.duals[m].copy_(torch.from_numpy(np.ascontiguousarray(y)))
            self.rho.copy_(torch.tensor([float(r) for r in rho], dtype=torch.float64))
            self.counters.zero_()
            self.norm_acc.zero_()
        N.check(self.lib.ntf_plan_sync_grams(self._plan, self._sh))

    def run(self, n_iters: int, use_graph: bool = True) -> None:
        N.check(self.lib.ntf_plan_run(self._plan, int(n_iters), 1 if use_graph else 0, self._sh))

    def set_timing(self, enable: bool) -> None:
        N.check(self.lib.ntf_plan_set_timing(self._plan, 1 if enable else 0))

    def kernel_times(self) -> np.ndarray:
        """[n_mode_updates][2] ms (MTTKRP, row update) of the latest iteration."""
        n = 2 * self.order * int(self.config.inner_sweeps)
        buf = (ctypes.c_float * n)()
        got = self.lib.ntf_plan_kernel_times(self._plan, buf, n)
        if got < 0:
            N.check(-got)
        return np.array(buf[:got], dtype=np.float64).reshape(-1, 2)

    def step(self) -> None:
        """One outer iteration (graph replay)."""
        self.run(1)

    def final_sq_error(self, aux):
        """(sum x^2, sum (x - [[aux]])^2) over the whole tensor, on the device
        (sparse: the Gram identity of tensors.py:291-301)."""
        with self.torch.cuda.stream(self.stream):
            if isinstance(self.x, DeviceCoo):
                out = coo_sq_error(self.x, aux, stream=self.stream)
            else:
                xv, fv = order3_view(self.x, aux, stream=self.stream)
                out = sq_error(xv, fv, stream=self.stream)
            return float(out[0].item()), float(out[1].item())

    def aux_model_rfe(self, x_norm: float) -> float:
        """Gram-identity RFE of the auxiliary model (reference solver.aux_model_rfe,
        solver.py:330-337): ||X||^2 - 2<A, MTTKRP_1(aux)> + <A^T A, G_23>."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            aux = self.aux
            if isinstance(self.x, DeviceCoo):
                m = mttkrp_coo_device(self.x, aux, 1, stream=self.stream)
            else:
                xv, fv = order3_view(self.x, aux, stream=self.stream)
                m = mttkrp_device(xv, fv, 1, self._desc.engine, stream=self.stream)
            g = None
            for f in reversed(aux[1:]):  # companions of mode 1, highest mode first
                gf = gram_device(f, stream=self.stream)
                g = gf if g is None else g * gf
            ga = gram_device(aux[0], stream=self.stream)
            cross = float(torch.sum(aux[0] * m).item())
            quad = float(torch.sum(ga * g).item())
        sq = x_norm ** 2 - 2.0 * cross + quad
        return float(np.sqrt(max(sq, 0.0))) / x_norm

    def mode_update(self, mode: int, last_sweep: bool) -> None:
        N.check(self.lib.ntf_plan_mode_update(self._plan, mode, 1 if last_sweep else 0, self._sh))

    def finalize(self) -> None:
        N.check(self.lib.ntf_plan_finalize(self._plan, self._sh))

    def _ensure_gram_ws(self, m: int) -> None:
        wsb = self.lib.ntf_gram_workspace_bytes(self.dims[m], self.R)
        if not hasattr(self, "_gram_ws") or self._gram_ws.numel() * 8 < wsb:
            torch = self.torch
            with torch.cuda.stream(self.stream):
                self._gram_ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=self.device)

    def refresh_gram(self, m: int) -> None:
        lib = self.lib
        rows = self.dims[m]
        self._ensure_gram_ws(m)
        N.check(lib.ntf_gram(_ptr(self.factors[m]), rows, self.R, _ptr(self.grams[m]),
                             _ptr(self._gram_ws), self._gram_ws.numel() * 8, self._sh))
        N.check(lib.ntf_colmax(_ptr(self.factors[m]), rows, self.R,
                               self.colmax.data_ptr() + m * self.R * 8, self._sh))

    def counters_host(self) -> np.ndarray:
        self.stream.synchronize()
        return self.counters.cpu().numpy()

    def check_status(self) -> tuple[int, bool]:
        """(iterations done, stopped); raises on device-side numerical failure."""
        c = self.counters_host()
        if c[2] == 1:
            from .solver import InvalidPenaltyError

            raise InvalidPenaltyError("ridge system not positive definite")
        if c[2] == 2:
            raise ValueError("cannot project a matrix with non-finite entries")
        return int(c[0]), bool(c[1])

    def histories(self, n: int):
        self.stream.synchronize()
        n = min(n, self.cap)
        return self.resid_hist[:n].cpu().numpy(), self.rho_hist[:n].cpu().numpy()

    def read_factors(self) -> list[np.ndarray]:
        self.stream.synchronize()
        return [f.cpu().numpy() for f in self.factors]

    def read_state(self):
        self.stream.synchronize()
        return ([f.cpu().numpy() for f in self.factors], [a.cpu().numpy() for a in self.aux],
                [y.cpu().numpy() for y in self.duals], [float(r) for r in self.rho.cpu().numpy()])

    def close(self) -> None:
        if getattr(self, "_plan", None):
            self.stream.synchronize()
            self.lib.ntf_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass
