"""ctypes binding of the C ABI in ``include/ntf_b200.h`` (libntf_b200.so).

The library is built in-tree (``build.py``).  There is no CPU fallback: if
the library cannot be loaded, or no CUDA device is present, the product path
raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libntf_b200.so")

ABI_VERSION = 2  # include/ntf_b200.h NTF_ABI_VERSION

NTF_OK = 0
NTF_ERR_INVALID = 1
NTF_ERR_NOT_PD = 2
NTF_ERR_NONFINITE = 3
NTF_ERR_CUDA = 4
NTF_ERR_UNSUPPORTED = 5

NTF_F32 = 0
NTF_F64 = 1

NTF_FORMAT_DENSE = 0
NTF_FORMAT_COO = 1

ENGINE_AUTO = 0
ENGINE_CUDA_CORE = 1
ENGINE_TCGEN05 = 2

# every entry point declared in include/ntf_b200.h
EXPORTED = (
    "ntf_abi_version",
    "ntf_last_error",
    "ntf_mttkrp_workspace_bytes",
    "ntf_mttkrp",
    "ntf_gram_workspace_bytes",
    "ntf_gram",
    "ntf_sq_error_workspace_bytes",
    "ntf_sq_error",
    "ntf_mttkrp_coo",
    "ntf_sq_error_coo_workspace_bytes",
    "ntf_sq_error_coo",
    "ntf_khatri_rao_pair",
    "ntf_synth_dense",
    "ntf_trim_device_pool",
    "ntf_device_pool_idle_bytes",
    "ntf_plan_create",
    "ntf_colmax",
    "ntf_plan_sync_grams",
    "ntf_plan_refresh_tensor",
    "ntf_plan_run",
    "ntf_plan_mode_update",
    "ntf_plan_finalize",
    "ntf_plan_set_timing",
    "ntf_plan_kernel_times",
    "ntf_plan_destroy",
    "ntf_peer_buffer_bytes",
    "ntf_peer_alloc",
    "ntf_peer_open",
    "ntf_peer_close",
    "ntf_peer_free",
    "ntf_peer_gather",
    "ntf_peer_gather_group",
)

NTF_MAX_PEERS = 8
NTF_PEER_TIMEOUT = 6


class NativeUnavailable(RuntimeError):
    """The sm_100a library (or a CUDA device) is missing: no fallback exists."""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"ntf_b200 error {code}: {msg}")
        self.code = code


c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)


class PlanDesc(ctypes.Structure):
    """Mirror of ``ntf_plan_desc`` (include/ntf_b200.h)."""

    _fields_ = [
        ("order", c_int),
        ("x_dtype", c_int),
        ("x_mode", c_vp * 4),
        ("x_dims", (c_i64 * 4) * 4),
        ("dims", c_i64 * 4),
        ("row_offset", c_i64 * 4),
        ("row_count", c_i64 * 4),
        ("rank", c_int),
        ("engine", c_int),
        ("fuse_gram", c_int),
        ("eps_abs", c_dbl),
        ("eps_rel", c_dbl),
        ("mu", c_dbl),
        ("tau_incr", c_dbl),
        ("tau_decr", c_dbl),
        ("inner_sweeps", c_int),
        ("adapt", c_int),
        ("factors", c_vp * 4),
        ("aux", c_vp * 4),
        ("duals", c_vp * 4),
        ("grams", c_vp * 4),
        ("colmax", c_vp),
        ("rho", c_vp),
        ("norm_acc", c_vp),
        ("norm_all", c_vp),
        ("norm_parts", ctypes.c_int),
        ("history_capacity", c_i64),
        ("resid_history", c_vp),
        ("rho_history", c_vp),
        ("counters", c_vp),
        ("rho_schedule", c_vp),
        ("constraint", ctypes.c_int * 4),
        ("card", c_i64 * 4),
        ("x_format", ctypes.c_int),
        ("nnz", c_i64),
        ("coo_idx", c_vp),
        ("coo_vals", c_vp),
        ("coo_perm", c_vp * 4),
        ("coo_rowptr", c_vp * 4),
    ]


class PeerGatherDesc(ctypes.Structure):
    """Mirror of ``ntf_peer_gather_desc`` (include/ntf_b200.h)."""

    _fields_ = [
        ("nranks", c_int),
        ("me", c_int),
        ("R", c_int),
        ("ctas", c_int),
        ("row_offset", c_i64 * (NTF_MAX_PEERS + 1)),
        ("full", c_vp),
        ("peer_base", c_vp * NTF_MAX_PEERS),
        ("status", c_vp),
        ("timeout_ns", c_i64),
    ]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    lib.ntf_abi_version.restype = c_int
    lib.ntf_last_error.restype = ctypes.c_char_p
    lib.ntf_mttkrp_workspace_bytes.restype = ctypes.c_size_t
    lib.ntf_mttkrp_workspace_bytes.argtypes = [c_int, c_int, c_i64, c_i64, c_i64, c_int, c_int]
    lib.ntf_mttkrp.restype = c_int
    lib.ntf_mttkrp.argtypes = [c_int, c_int, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int,
                               c_vp, c_vp, ctypes.c_size_t, c_int, c_vp]
    lib.ntf_gram_workspace_bytes.restype = ctypes.c_size_t
    lib.ntf_gram_workspace_bytes.argtypes = [c_i64, c_int]
    lib.ntf_gram.restype = c_int
    lib.ntf_gram.argtypes = [c_vp, c_i64, c_int, c_vp, c_vp, ctypes.c_size_t, c_vp]
    lib.ntf_sq_error_workspace_bytes.restype = ctypes.c_size_t
    lib.ntf_sq_error_workspace_bytes.argtypes = [c_i64, c_i64, c_i64]
    lib.ntf_sq_error.restype = c_int
    lib.ntf_sq_error.argtypes = [c_int, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp,
                                 c_vp, ctypes.c_size_t, c_vp]
    lib.ntf_mttkrp_coo.restype = c_int
    lib.ntf_mttkrp_coo.argtypes = [c_int, c_vp, c_int, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_int,
                                   c_vp, c_vp]
    lib.ntf_sq_error_coo_workspace_bytes.restype = ctypes.c_size_t
    lib.ntf_sq_error_coo_workspace_bytes.argtypes = [c_i64]
    lib.ntf_sq_error_coo.restype = c_int
    lib.ntf_sq_error_coo.argtypes = [c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_vp,
                                     ctypes.c_size_t, c_vp]
    lib.ntf_khatri_rao_pair.restype = c_int
    lib.ntf_khatri_rao_pair.argtypes = [c_vp, c_i64, c_vp, c_i64, c_int, c_vp, c_vp]
    lib.ntf_synth_dense.restype = c_int
    lib.ntf_synth_dense.argtypes = [c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_dbl,
                                    ctypes.c_uint64, c_vp]
    lib.ntf_trim_device_pool.restype = c_int
    lib.ntf_trim_device_pool.argtypes = []
    lib.ntf_device_pool_idle_bytes.restype = c_int
    lib.ntf_device_pool_idle_bytes.argtypes = [ctypes.POINTER(ctypes.c_size_t)]
    lib.ntf_plan_create.restype = c_int
    lib.ntf_plan_create.argtypes = [ctypes.POINTER(PlanDesc), ctypes.POINTER(c_vp)]
    lib.ntf_colmax.restype = c_int
    lib.ntf_colmax.argtypes = [c_vp, c_i64, c_int, c_vp, c_vp]
    lib.ntf_plan_sync_grams.restype = c_int
    lib.ntf_plan_sync_grams.argtypes = [c_vp, c_vp]
    lib.ntf_plan_refresh_tensor.restype = c_int
    lib.ntf_plan_refresh_tensor.argtypes = [c_vp, c_vp]
    lib.ntf_plan_run.restype = c_int
    lib.ntf_plan_run.argtypes = [c_vp, c_int, c_int, c_vp]
    lib.ntf_plan_mode_update.restype = c_int
    lib.ntf_plan_mode_update.argtypes = [c_vp, c_int, c_int, c_vp]
    lib.ntf_plan_finalize.restype = c_int
    lib.ntf_plan_finalize.argtypes = [c_vp, c_vp]
    lib.ntf_plan_set_timing.restype = c_int
    lib.ntf_plan_set_timing.argtypes = [c_vp, c_int]
    lib.ntf_plan_kernel_times.restype = c_int
    lib.ntf_plan_kernel_times.argtypes = [c_vp, ctypes.POINTER(ctypes.c_float), c_int]
    lib.ntf_plan_destroy.restype = None
    lib.ntf_plan_destroy.argtypes = [c_vp]
    lib.ntf_peer_buffer_bytes.restype = ctypes.c_size_t
    lib.ntf_peer_buffer_bytes.argtypes = [c_i64, c_int]
    lib.ntf_peer_alloc.restype = c_int
    lib.ntf_peer_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(c_vp), c_vp]
    lib.ntf_peer_open.restype = c_int
    lib.ntf_peer_open.argtypes = [c_vp, ctypes.POINTER(c_vp)]
    lib.ntf_peer_close.restype = c_int
    lib.ntf_peer_close.argtypes = [c_vp]
    lib.ntf_peer_free.restype = c_int
    lib.ntf_peer_free.argtypes = [c_vp]
    lib.ntf_peer_gather.restype = c_int
    lib.ntf_peer_gather.argtypes = [ctypes.POINTER(PeerGatherDesc), c_vp]
    lib.ntf_peer_gather_group.restype = c_int
    lib.ntf_peer_gather_group.argtypes = [ctypes.POINTER(PeerGatherDesc), c_int, c_vp]
    return lib


def load(build_if_missing: bool = True):
    """Load (building in-tree first if needed) and return the ctypes library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH) and build_if_missing:
            from . import build as _build

            _build.build()
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(f"{LIB_PATH} is missing; run paper_1409_2383_b200/build.py")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
        _lib = _declare(lib)
        if _lib.ntf_abi_version() != ABI_VERSION:
            raise NativeUnavailable("ABI version mismatch")
        return _lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception classes."""
    if rc == NTF_OK:
        return
    msg = (load().ntf_last_error() or b"").decode(errors="replace")
    if rc == NTF_ERR_INVALID or rc == NTF_ERR_NONFINITE:
        raise ValueError(msg)
    if rc == NTF_ERR_NOT_PD:
        from .solver import InvalidPenaltyError

        raise InvalidPenaltyError(msg)
    if rc == NTF_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(rc, msg)
