"""Tensor files of the reference (tensor_io.py:1-80): raw binary CPDT and text COO.

CPDT (tensor_io.py:55-74): magic ``CPDT``, little-endian u32 order, u32
extents, then the dense values as little-endian f64 in row-major order.
``read_binary(path, device=...)`` streams the payload straight into HBM
through two pinned staging buffers (file reads overlap the host-to-device
copies; the f64 -> f32 conversion, when asked for, runs on the device), so a
tensor larger than host RAM loads without a host copy of the whole array
(SURVEY 8(f) #2).  Without ``device`` it returns the host tensor, as the
reference.  Text COO (tensor_io.py:27-52) is read and written on the host.
"""

from __future__ import annotations

import math
import struct
from pathlib import Path

import numpy as np

from .tensors import CooTensor, DenseTensor

MAGIC = b"CPDT"


def _read_header(fh, path) -> tuple[int, ...]:
    magic = fh.read(4)
    if magic != MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}")
    (order,) = struct.unpack("<I", fh.read(4))
    return tuple(int(d) for d in struct.unpack(f"<{order}I", fh.read(4 * order)))


def write_binary(t, path: str | Path) -> None:
    """tensor_io.py:55-60 (values written as little-endian f64)."""
    vals = getattr(t, "values", t)
    if type(vals).__module__.startswith("torch"):
        vals = vals.detach().cpu().numpy()
    vals = np.asarray(vals)
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<I", vals.ndim))
        fh.write(struct.pack(f"<{vals.ndim}I", *vals.shape))
        fh.write(np.ascontiguousarray(vals, dtype="<f8").tobytes())


def read_binary(path: str | Path, *, device=None, dtype=None,
                chunk_bytes: int = 256 << 20) -> DenseTensor:
    """tensor_io.py:63-74.  ``device``: stream the payload into HBM (``dtype``
    float32 converts on the device); otherwise the host tensor."""
    with open(path, "rb") as fh:
        dims = _read_header(fh, path)
        count = math.prod(dims)
        if device is None:
            data = np.frombuffer(fh.read(8 * count), dtype="<f8", count=-1)
            if data.size != count:
                raise ValueError(f"{path}: truncated value payload")
            out = DenseTensor(data.reshape(dims))
            return out if dtype is None else DenseTensor(out.values, dtype=dtype)
        import torch

        dev = torch.device(device)
        want = torch.float32 if (dtype is not None and np.dtype(dtype) == np.float32) else torch.float64
        x = torch.empty(count, dtype=want, device=dev)
        n_chunk = max(1, int(chunk_bytes) // 8)
        stage = [torch.empty(n_chunk, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        done = [None, None]
        stream = torch.cuda.Stream(device=dev)
        pos = 0
        k = 0
        while pos < count:
            n = min(n_chunk, count - pos)
            buf = stage[k & 1]
            if done[k & 1] is not None:
                done[k & 1].synchronize()  # the staging buffer's previous copy has landed
            view = memoryview(buf.numpy()[:n]).cast("B")
            got = fh.readinto(view)
            if got != 8 * n:
                raise ValueError(f"{path}: truncated value payload")
            with torch.cuda.stream(stream):
                x[pos:pos + n].copy_(buf[:n], non_blocking=True)  # f64 -> want on the device
                ev = torch.cuda.Event()
                ev.record(stream)
            done[k & 1] = ev
            pos += n
            k += 1
        stream.synchronize()
        return DenseTensor(x.view(dims))


def write_coo(t, path: str | Path) -> None:
    """tensor_io.py:27-32 (dense inputs are converted with from_dense)."""
    if not isinstance(t, CooTensor):
        t = CooTensor.from_dense(t)
    with open(path, "w") as fh:
        fh.write("dims " + " ".join(str(d) for d in t.dims) + "\n")
        for idx, val in zip(t.indices, t.vals):
            fh.write(" ".join(str(int(i)) for i in idx) + f" {float(val)!r}\n")


def read_coo(path: str | Path) -> CooTensor:
    """tensor_io.py:35-52."""
    with open(path) as fh:
        header = fh.readline().split()
        if not header or header[0] != "dims":
            raise ValueError(f"{path}: expected 'dims ...' header")
        dims = [int(d) for d in header[1:]]
        order = len(dims)
        indices, vals = [], []
        for lineno, line in enumerate(fh, start=2):
            parts = line.split()
            if not parts:
                continue
            if len(parts) != order + 1:
                raise ValueError(f"{path}:{lineno}: expected {order} indices and a value")
            indices.append([int(p) for p in parts[:order]])
            vals.append(float(parts[order]))
    return CooTensor(dims, np.array(indices, dtype=np.int64).reshape(-1, order), np.array(vals))


def read_tensor(path: str | Path, **kw):
    """Dispatch on content (tensor_io.py:77-83): CPDT binary or text COO."""
    with open(path, "rb") as fh:
        head = fh.read(4)
    return read_binary(path, **kw) if head == MAGIC else read_coo(path)


def write_tensor(t, path: str | Path) -> None:
    """tensor_io.py:86-93: sparse tensors, or a .coo/.txt suffix, as text COO;
    dense tensors otherwise as CPDT binary."""
    suffix = Path(path).suffix.lower()
    if isinstance(t, CooTensor) or suffix in (".coo", ".txt"):
        write_coo(t, path)
    else:
        write_binary(t, path)
