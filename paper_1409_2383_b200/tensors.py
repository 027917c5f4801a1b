"""Tensor containers of the drop-in API (reference tensors.py:40-171).

``DenseTensor`` mirrors the reference container (order 3, row-major, read
only) and additionally keeps fp32 storage when given fp32 values — the B200
path streams fp32 tensors for BASELINE configs 2-5.  Values may
also be a ``torch.Tensor`` (host or device), so a tensor generated on the GPU
is never copied to the host.  Order-4 dense tensors run on one GPU as
order-3 views (include/ntf_b200.h).  ``CooTensor`` mirrors the reference's
sparse container (tensors.py:84-132; order 3, fp64); ``fit`` runs it with the
COO MTTKRP engine on one GPU.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

SUPPORTED_ORDERS = (3, 4)


def _is_torch(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch")


class DenseTensor:
    """Immutable dense order-3 or order-4 tensor, row-major (reference
    tensors.py:40-81)."""

    __slots__ = ("dims", "values", "_norm", "_device_cache", "__weakref__")

    def __init__(self, values, dtype=None):
        if _is_torch(values):
            import torch

            if values.dim() not in SUPPORTED_ORDERS:
                raise ValueError(f"tensor order must be 3 or 4, got {values.dim()}")
            want = dtype or (torch.float32 if values.dtype == torch.float32 else torch.float64)
            if isinstance(want, type) or isinstance(want, np.dtype):
                want = torch.float32 if np.dtype(want) == np.float32 else torch.float64
            self.values = values.to(dtype=want).contiguous()
            self.dims = tuple(int(d) for d in values.shape)
        else:
            arr = np.asarray(values)
            want = np.dtype(dtype) if dtype is not None else (
                np.dtype(np.float32) if arr.dtype == np.float32 else np.dtype(np.float64))
            if want not in (np.dtype(np.float32), np.dtype(np.float64)):
                raise ValueError("dtype must be float32 or float64")
            arr = np.array(arr, dtype=want, order="C", copy=arr.dtype != want or not arr.flags.c_contiguous)
            if arr.ndim not in SUPPORTED_ORDERS:
                raise ValueError(f"tensor order must be 3 or 4, got {arr.ndim}")
            arr.flags.writeable = False
            self.values = arr
            self.dims = tuple(int(d) for d in arr.shape)
        if any(d < 1 for d in self.dims):
            raise ValueError(f"all extents must be >= 1, got {self.dims}")
        self._norm = None
        self._device_cache = None

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def dtype(self):
        if _is_torch(self.values):
            import torch

            return np.float32 if self.values.dtype == torch.float32 else np.float64
        return self.values.dtype.type

    def norm(self) -> float:
        """Frobenius norm in fp64 (tensors.py:57-61), computed on the device."""
        if self._norm is None:
            from .engine import tensor_norm

            self._norm = tensor_norm(self)
        return self._norm

    def __repr__(self) -> str:
        return f"DenseTensor(dims={self.dims}, dtype={np.dtype(self.dtype).name})"


class KruskalModel:
    """Factor matrices sharing the column count F (reference tensors.py:135-171)."""

    __slots__ = ("factors",)

    def __init__(self, factors: Sequence[np.ndarray]):
        factors = tuple(np.array(f, dtype=np.float64, order="C") for f in factors)
        if len(factors) not in (3, 4):
            raise ValueError(f"model must have 3 or 4 factors, got {len(factors)}")
        rank = factors[0].shape[1] if factors[0].ndim == 2 else -1
        for m, f in enumerate(factors, start=1):
            if f.ndim != 2 or f.shape[0] < 1 or f.shape[1] < 1:
                raise ValueError(f"factor {m} must be a non-empty matrix")
            if f.shape[1] != rank:
                raise ValueError("all factors must share the same column count")
            if not np.all(np.isfinite(f)):
                raise ValueError(f"factor {m} has non-finite entries")
            f.flags.writeable = False
        self.factors = factors

    @property
    def order(self) -> int:
        return len(self.factors)

    @property
    def rank(self) -> int:
        return self.factors[0].shape[1]

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(f.shape[0] for f in self.factors)

    def factor(self, mode: int) -> np.ndarray:
        if not 1 <= mode <= self.order:
            raise ValueError(f"mode must be in 1..{self.order}, got {mode}")
        return self.factors[mode - 1]

    def __repr__(self) -> str:
        return f"KruskalModel(dims={self.dims}, rank={self.rank})"


class CooTensor:
    """Sparse order-3 or order-4 tensor in coordinate form, entries sorted
    lexicographically, duplicates rejected (reference tensors.py:84-132)."""

    __slots__ = ("dims", "indices", "vals", "_device_cache", "__weakref__")

    def __init__(self, dims: Sequence[int], indices, vals):
        self.dims = tuple(int(d) for d in dims)
        if len(self.dims) not in SUPPORTED_ORDERS:
            raise ValueError(f"tensor order must be 3 or 4, got {len(self.dims)}")
        if any(d < 1 for d in self.dims):
            raise ValueError(f"all extents must be >= 1, got {self.dims}")
        n = len(self.dims)
        idx = np.asarray(indices, dtype=np.int64).reshape(-1, n)
        v = np.asarray(vals, dtype=np.float64).reshape(-1)
        if idx.shape[0] != v.shape[0]:
            raise ValueError("index rows and value count differ")
        if idx.size:
            if idx.min() < 0 or np.any(idx >= np.array(self.dims)):
                raise ValueError("entry index out of bounds")
            order = np.lexsort(tuple(idx[:, m] for m in reversed(range(n))))
            idx, v = idx[order], v[order]
            if np.any(np.all(np.diff(idx, axis=0) == 0, axis=1)):
                raise ValueError("duplicate entry indices")
        idx.flags.writeable = False
        v.flags.writeable = False
        self.indices = idx
        self.vals = v
        self._device_cache = None

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def norm(self) -> float:
        """tensors.py:114-115 (host numpy over the stored values, as the reference)."""
        return float(np.linalg.norm(self.vals))

    def to_dense(self) -> DenseTensor:
        out = np.zeros(self.dims)
        out[tuple(self.indices[:, m] for m in range(self.order))] = self.vals
        return DenseTensor(out)

    @classmethod
    def from_dense(cls, t, tol: float = 0.0) -> "CooTensor":
        vals = np.asarray(getattr(t, "values", t), dtype=np.float64)
        mask = np.abs(vals) > tol
        return cls(vals.shape, np.argwhere(mask), vals[mask])

    def __repr__(self) -> str:
        return f"CooTensor(dims={self.dims}, nnz={self.nnz})"


def is_sparse(t) -> bool:
    return isinstance(t, CooTensor) or (hasattr(t, "indices") and hasattr(t, "vals"))


def as_coo(t) -> CooTensor:
    """Our CooTensor, or the reference's (duck-typed on dims/indices/vals)."""
    if isinstance(t, CooTensor):
        return t
    return CooTensor(t.dims, t.indices, t.vals)


def as_dense(t) -> DenseTensor:
    """Accept our DenseTensor, the reference's DenseTensor (duck-typed on
    ``.values``/``.dims``), a numpy array or a torch tensor."""
    if isinstance(t, DenseTensor):
        return t
    if is_sparse(t):
        raise TypeError("a sparse COO tensor is not dense (use as_coo)")
    vals = getattr(t, "values", t)
    if _is_torch(vals) or isinstance(vals, np.ndarray):
        return DenseTensor(vals)
    raise TypeError(f"unsupported tensor type {type(t).__name__}")
