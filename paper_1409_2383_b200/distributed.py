"""Sharded multi-GPU fit: one process per GPU, NCCL over NVLink.

Follows the paper's block-row partitioning (§V, reference
blocks.py:171-196 and the mesh data flow mesh.py:149-237) re-cast for GPUs
(SURVEY 8(e)): rank p owns factor rows ``PartitionPlan.uniform(dims, P)``
(blocks.py:47-61) and holds the three slabs X[I_p,:,:], X[:,J_p,:],
X[:,:,K_p].  A mode-n update is then entirely local (MTTKRP of the owned rows
from the local slab, the shared ridge Cholesky, the row solves and the fused
aux/dual step); the one exchange per mode update is an all-gather of the
updated row block, after which every rank recomputes the same Gram locally.
Once per outer iteration the 15 scaled residual sums of squares
((scale, ssq) pairs, nrm2-style) are all-gathered and merged in rank order by
every rank's finalize, so the stop test and the penalty adaptation are
replicated bit-identically.

``sharded_iteration`` is written against a small problem interface so the
collective logic can be exercised on CPU with the gloo backend
(tests/test_distributed_gloo.py) as well as on GPUs with NCCL.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .constraints import normalize_specs
from .solver import FitResult, SolverConfig, _engine_code, _run_fit
from .tensors import as_dense


@dataclass(frozen=True)
class PartitionPlan:
    """Per-mode row extents (reference blocks.PartitionPlan, blocks.py:36-61)."""

    extents: tuple

    @classmethod
    def uniform(cls, dims: Sequence[int], blocks: int | Sequence[int]) -> "PartitionPlan":
        if isinstance(blocks, int):
            blocks = [blocks] * len(dims)
        if len(blocks) != len(dims):
            raise ValueError("need one block count per mode")
        ext = []
        for d, n in zip(dims, blocks):
            if not 1 <= n <= d:
                raise ValueError(f"block count {n} invalid for extent {d}")
            base, extra = divmod(int(d), int(n))
            ext.append(tuple(base + (1 if i < extra else 0) for i in range(n)))
        return cls(tuple(ext))

    @property
    def dims(self) -> tuple:
        return tuple(sum(e) for e in self.extents)

    @property
    def counts(self) -> tuple:
        return tuple(len(e) for e in self.extents)

    def offsets(self, mode: int) -> list:
        out = [0]
        for e in self.extents[mode - 1]:
            out.append(out[-1] + e)
        return out

    def row_slice(self, mode: int, block: int) -> slice:
        o = self.offsets(mode)
        return slice(o[block], o[block + 1])


class Comm:
    """torch.distributed collectives used by the sharded iteration."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def all_reduce_(self, t) -> None:
        self.dist.all_reduce(t, group=self.group)

    def all_gather_(self, out, t) -> None:
        """out[q * t.numel():(q + 1) * t.numel()] = rank q's ``t``."""
        self.dist.all_gather_into_tensor(out, t, group=self.group)

    def peer_ok(self, device) -> bool:
        """Whether rows can be gathered over NVLink peer memory (one fused
        kernel, ``_PeerRows``) instead of ncclAllGather: CUDA tensors, at most
        NTF_MAX_PEERS ranks on one node, each on its own GPU, every pair
        P2P-reachable, and NTF_B200_P2P not "0".  Decided once, collectively
        (every rank takes the same path)."""
        if getattr(self, "_peer_state", None) is not None:
            return self._peer_state
        if device.type != "cuda":  # CPU (gloo) runs: all ranks alike, no exchange needed
            self._peer_state = False
            return False
        import os
        import socket

        import torch

        from ._native import NTF_MAX_PEERS

        want = os.environ.get("NTF_B200_P2P", "1") != "0" and self.size <= NTF_MAX_PEERS
        uuid = str(torch.cuda.get_device_properties(device).uuid)
        infos = [None] * self.size
        self.dist.all_gather_object(infos, (socket.gethostname(), uuid, want), group=self.group)
        ok = all(w for _, _, w in infos) and len({h for h, _, _ in infos}) == 1 \
            and len({u for _, u, _ in infos}) == self.size
        if ok:  # map peer uuids to local ordinals (CUDA_VISIBLE_DEVICES may differ per rank)
            local = {str(torch.cuda.get_device_properties(d).uuid): d for d in range(torch.cuda.device_count())}
            me = device.index if device.index is not None else torch.cuda.current_device()
            ok = all(u in local and (u == uuid or torch.cuda.can_device_access_peer(me, local[u]))
                     for _, u, _ in infos)
            flags = [None] * self.size
            self.dist.all_gather_object(flags, ok, group=self.group)
            ok = all(flags)
        self._peer_state = ok
        return ok

    def gather_rows(self, full, offsets: Sequence[int], counts: Sequence[int]) -> None:
        """In place: every rank's owned block of ``full`` (rows offsets[p] ..
        +counts[p]) is broadcast to all ranks.  On one NVLink node this is one
        kernel that pushes the rows into the peers' buffers (``_PeerRows``);
        otherwise ncclAllGather with blocks padded to the largest count
        because the uniform plan is uneven.  Buffers are
        allocated once per target tensor, so the call can be captured in a
        CUDA graph."""
        if self.size == 1 and os.environ.get("NTF_B200_P2P") != "force":
            return  # the owned block is the whole factor ("force": run the kernel anyway, for tests)
        if self.peer_ok(full.device):
            key = (full.data_ptr(), tuple(full.shape))
            if not hasattr(self, "_peers"):
                self._peers = {}
            pr = self._peers.get(key)
            if pr is None:
                pr = self._peers[key] = _PeerRows(self, full, offsets, counts)
            pr.gather()
            return
        maxc = max(counts)
        p = self.rank
        key = (full.data_ptr(), tuple(full.shape), maxc)
        bufs = self._bufs.get(key) if hasattr(self, "_bufs") else None
        if bufs is None:
            if not hasattr(self, "_bufs"):
                self._bufs = {}
            send = full.new_zeros((maxc,) + tuple(full.shape[1:]))
            recv = full.new_empty((self.size * maxc,) + tuple(full.shape[1:]))
            bufs = self._bufs[key] = (send, recv)
        send, recv = bufs
        send[: counts[p]].copy_(full[offsets[p]: offsets[p] + counts[p]])
        self.dist.all_gather_into_tensor(recv, send, group=self.group)
        for q in range(self.size):
            if q == p:
                continue
            full[offsets[q]: offsets[q] + counts[q]].copy_(recv[q * maxc: q * maxc + counts[q]])


    def check_peers(self) -> None:
        """Raise if a peer gather timed out waiting for another rank."""
        for pr in getattr(self, "_peers", {}).values():
            pr.check()

    def close_peers(self) -> None:
        """Unmap the peers' buffers, wait for every rank to do the same, free
        our own (a buffer is freed only after no peer maps it)."""
        peers = getattr(self, "_peers", {})
        if not peers:
            return
        import torch

        torch.cuda.synchronize()
        for pr in peers.values():
            pr.unmap()
        self.dist.barrier(group=self.group)
        for pr in peers.values():
            pr.free()
        self._peers = {}


class _PeerRows:
    """One factor's row all-gather over NVLink peer memory: a peer buffer
    (counters + double-buffered staging, ``ntf_peer_alloc``) per rank, mapped
    by every other rank through CUDA IPC, and the ``ntf_peer_gather`` kernel
    (csrc/peer_gather.cu).  Replaces pack + ncclAllGather + unpack of the
    updated row blocks (reference blocks.py:171-196, mesh.py:149-237)."""

    def __init__(self, comm: Comm, full, offsets: Sequence[int], counts: Sequence[int]):
        import ctypes
        import os

        import torch

        from . import _native

        lib = self.lib = _native.load()
        self.check_rc = _native.check
        rows, R = int(full.shape[0]), int(full.shape[1])
        P, me = comm.size, comm.rank
        for q in range(P - 1):
            if offsets[q] + counts[q] != offsets[q + 1]:
                raise ValueError("row blocks must be contiguous")
        if offsets[0] != 0 or offsets[-1] + counts[-1] != rows:
            raise ValueError("row blocks must cover the factor")
        base = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        self.check_rc(lib.ntf_peer_alloc(lib.ntf_peer_buffer_bytes(rows, R), ctypes.byref(base), handle))
        self.own = base.value
        handles = [None] * P
        comm.dist.all_gather_object(handles, bytes(handle), group=comm.group)
        self.mapped = []
        bases = []
        for q in range(P):
            if q == me:
                bases.append(self.own)
                continue
            pb = ctypes.c_void_p()
            buf = ctypes.create_string_buffer(handles[q], 64)
            self.check_rc(lib.ntf_peer_open(buf, ctypes.byref(pb)))
            self.mapped.append(pb.value)
            bases.append(pb.value)
        self.status = torch.zeros(1, dtype=torch.int32, device=full.device)
        d = self.desc = _native.PeerGatherDesc()
        d.nranks, d.me, d.R = P, me, R
        # same on every rank: derived from the global geometry only
        d.ctas = int(min(32, max(1, -(-max(counts) * R // 8192))))
        for q in range(P):
            d.row_offset[q] = int(offsets[q])
            d.peer_base[q] = bases[q]
        d.row_offset[P] = rows
        d.full = full.data_ptr()
        d.status = self.status.data_ptr()
        d.timeout_ns = int(float(os.environ.get("NTF_B200_P2P_TIMEOUT_S", "60")) * 1e9)
        self._torch = torch

    def gather(self) -> None:
        stream = self._torch.cuda.current_stream().cuda_stream
        self.check_rc(self.lib.ntf_peer_gather(self.desc, stream))

    def check(self) -> None:
        if int(self.status.item()) != 0:
            raise RuntimeError("peer row gather timed out waiting for another rank "
                               "(NTF_B200_P2P_TIMEOUT_S; NTF_B200_P2P=0 selects NCCL)")

    def unmap(self) -> None:
        for pb in self.mapped:
            self.lib.ntf_peer_close(pb)
        self.mapped = []

    def free(self) -> None:
        if self.own:
            self.lib.ntf_peer_free(self.own)
            self.own = None


def sharded_iteration(prob, comm: Comm, config: SolverConfig) -> None:
    """One outer iteration of the sharded solver (reference solver.py:295-327
    semantics; mesh.py:149-237 data flow).  ``prob`` provides mode_update,
    refresh_gram, finalize, factors, norm_acc, norm_all, offsets/counts."""
    sweeps = config.inner_sweeps
    for sw in range(sweeps):
        for mode in (1, 2, 3):
            m = mode - 1
            prob.mode_update(mode, sw == sweeps - 1)
            comm.gather_rows(prob.factors[m], prob.offsets[m], prob.counts[m])
            prob.refresh_gram(m)
    comm.all_gather_(prob.norm_all, prob.norm_acc)
    prob.finalize()


def _sharded_problem_class():
    from .engine import DeviceProblem, Slabs, gram_device, mttkrp_device, sq_error  # noqa: F401

    class ShardedProblem(DeviceProblem):
        def __init__(self, x_slabs, dims, rank, config, cap, engine, plan: PartitionPlan, comm: Comm,
                     constraints=None):
            p = comm.rank
            self.comm = comm
            self.plan = plan
            self.offsets = [plan.offsets(m + 1)[:-1] for m in range(3)]
            self.counts = [list(plan.extents[m]) for m in range(3)]
            own_off = tuple(self.offsets[m][p] for m in range(3))
            own_cnt = tuple(self.counts[m][p] for m in range(3))
            super().__init__(x_slabs[0], dims, rank, config, cap, engine,
                             slabs=Slabs(list(x_slabs), own_off, own_cnt), norm_parts=comm.size,
                             constraints=constraints)
            import os

            self._graph = None
            self._eager_steps = 0
            self._graph_ok = os.environ.get("NTF_B200_SHARDED_GRAPH", "1") != "0"
            for m in range(3):  # capture-safe: Gram workspace allocated up front
                self._ensure_gram_ws(m)
            # per-launch timing events stay on (they are captured into the
            # graph), so kernel_times() always reflects the latest iteration
            super().set_timing(True)

        def set_timing(self, enable: bool) -> None:
            """Timing events are always recorded on the sharded path."""

        def step(self) -> None:
            """One outer iteration.  After two eager iterations (NCCL
            communicators and staging buffers exist by then) the iteration --
            mode updates, row all-gathers, Gram refreshes, norm gather and
            finalize -- is captured once as a CUDA graph and replayed, so the
            host issues one launch per outer iteration instead of ~10 per mode
            update.  NTF_B200_SHARDED_GRAPH=0 keeps the eager loop."""
            torch = self.torch
            if self._graph is None and self._graph_ok and self._eager_steps >= 2:
                self._capture()
            if self._graph is not None:
                with torch.cuda.stream(self.stream):
                    self._graph.replay()
                return
            with torch.cuda.stream(self.stream):
                sharded_iteration(self, self.comm, self.config)
            self._eager_steps += 1

        def _capture(self) -> None:
            import warnings

            torch = self.torch
            g = torch.cuda.CUDAGraph()
            self.stream.synchronize()
            try:
                with torch.cuda.graph(g, stream=self.stream):
                    sharded_iteration(self, self.comm, self.config)
            except Exception as exc:  # capture unsupported: stay eager (same results)
                self._graph_ok = False
                warnings.warn(f"sharded iteration not captured as a CUDA graph ({exc}); running eagerly")
                return
            self._graph = g

        def final_sq_error(self, aux):
            torch = self.torch
            p = self.comm.rank
            rows = self.plan.row_slice(1, p)
            with torch.cuda.stream(self.stream):
                own = [aux[0][rows], aux[1], aux[2]]
                out = sq_error(self.slabs.x_mode[0], own, stream=self.stream)
                self.comm.all_reduce_(out)
                return float(out[0].item()), float(out[1].item())

        def aux_model_rfe(self, x_norm: float) -> float:
            torch = self.torch
            p = self.comm.rank
            with torch.cuda.stream(self.stream):
                full = [torch.zeros_like(f) for f in self.factors]
                for m in range(3):
                    o, c = self.offsets[m][p], self.counts[m][p]
                    full[m][o:o + c].copy_(self.aux[m])
                    self.comm.gather_rows(full[m], self.offsets[m], self.counts[m])
                own = full[0][self.plan.row_slice(1, p)]
                mt = mttkrp_device(self.slabs.x_mode[0], [own, full[1], full[2]], 1,
                                   self._desc.engine, stream=self.stream)
                g = gram_device(full[2], stream=self.stream) * gram_device(full[1], stream=self.stream)
                part = torch.stack([torch.sum(own * mt), torch.sum((own.T @ own) * g)])
                self.comm.all_reduce_(part)
                cross, quad = (float(v) for v in part.cpu())
            sq = x_norm ** 2 - 2.0 * cross + quad
            return math.sqrt(max(sq, 0.0)) / x_norm

        def gather_state(self, aux, duals):
            torch = self.torch
            p = self.comm.rank
            out_a, out_y = [], []
            for m in range(3):
                o, c = self.offsets[m][p], self.counts[m][p]
                full_a = torch.zeros((self.dims[m], self.R), dtype=torch.float64, device=self.device)
                full_y = torch.zeros_like(full_a)
                full_a[o:o + c].copy_(torch.from_numpy(aux[m]))
                full_y[o:o + c].copy_(torch.from_numpy(duals[m]))
                self.comm.gather_rows(full_a, self.offsets[m], self.counts[m])
                self.comm.gather_rows(full_y, self.offsets[m], self.counts[m])
                out_a.append(full_a.cpu().numpy())
                out_y.append(full_y.cpu().numpy())
            return out_a, out_y

    return ShardedProblem


def make_slabs(values, plan: PartitionPlan, rank_id: int, device):
    """This rank's three slabs of a host tensor, uploaded to ``device``."""
    import torch

    if isinstance(values, torch.Tensor):
        x = values
    else:
        import warnings

        with warnings.catch_warnings():  # read-only source: we only read it
            warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
            x = torch.from_numpy(np.ascontiguousarray(values))
    s1 = x[plan.row_slice(1, rank_id)]
    s2 = x[:, plan.row_slice(2, rank_id)]
    s3 = x[:, :, plan.row_slice(3, rank_id)]
    return [s.contiguous().to(device) for s in (s1, s2, s3)]


def distributed_fit(t, rank: int, specs=None, config: SolverConfig | None = None,
                    plan: PartitionPlan | int | None = None, trace_path: str | None = None,
                    *, engine=None, group=None, sharded: bool | None = None) -> FitResult:
    """Block-parallel fit over the ranks of ``torch.distributed`` (reference
    mesh.distributed_fit, mesh.py:331-350).  Without an initialised process
    group (or with one rank) this is exactly ``fit``, unless ``sharded=True``
    forces the sharded engine (a one-rank group exercises its collectives and
    graph capture on a single GPU).  ``trace_path`` (the simulator's message
    trace) has no NCCL equivalent and is ignored."""
    import torch
    import torch.distributed as dist

    from .solver import fit

    config = config or SolverConfig()
    from .tensors import is_sparse

    if is_sparse(t):  # COO tensors run on one GPU
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            raise NotImplementedError("sparse COO tensors are single-GPU (no sharded COO engine)")
        return fit(t, rank, specs, config, engine=engine)
    t = as_dense(t)
    specs = normalize_specs(specs, t.order)
    if rank < 1:
        raise ValueError("rank must be >= 1")
    if t.order != 3 and dist.is_available() and dist.is_initialized() and (
            dist.get_world_size(group) > 1 or sharded):
        raise NotImplementedError("order-4 tensors are single-GPU (no sharded order-4 engine)")
    if not (dist.is_available() and dist.is_initialized()) or (
            dist.get_world_size(group) == 1 and not sharded):
        return fit(t, rank, specs, config, engine=engine)
    if any(s.kind == "nonneg_card" for s in specs):
        raise NotImplementedError("the cardinality constraint needs the whole factor on one GPU "
                                  "(a global top-c selection); use fit()")
    comm = Comm(group)
    if plan is None or isinstance(plan, int):
        plan = PartitionPlan.uniform(t.dims, comm.size)
    if plan.dims != t.dims or set(plan.counts) != {comm.size}:
        raise ValueError("partition plan must give every mode one block per rank")
    device = torch.device("cuda", torch.cuda.current_device())
    vals = t.values
    slabs = make_slabs(vals, plan, comm.rank, device)
    # ||X||^2 from the mode-1 slabs
    from .engine import sq_error

    sq = sq_error(slabs[0])
    comm.all_reduce_(sq)
    x_norm = math.sqrt(float(sq[0].item()))
    if x_norm == 0.0:
        raise ValueError("cannot factorize a zero tensor")
    cls = _sharded_problem_class()
    from .constraints import plan_codes

    prob = cls(slabs, t.dims, rank, config, config.n_max, _engine_code(engine), plan, comm,
               constraints=plan_codes(specs, t.dims, rank))
    try:
        res = _run_fit(prob, slabs[0], t.dims, rank, config, x_norm, gather=prob.gather_state)
        comm.check_peers()
        return res
    finally:
        prob.close()
        comm.close_peers()
