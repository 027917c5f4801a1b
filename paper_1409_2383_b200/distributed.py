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


def _torch_mod():
    import torch

    return torch


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

    def all_reduce_max_(self, t) -> None:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def all_gather_(self, out, t) -> None:
        """out[q * t.numel():(q + 1) * t.numel()] = rank q's ``t``."""
        self.dist.all_gather_into_tensor(out, t, group=self.group)

    def peer_ok(self, device) -> bool:
        """Whether rows can be gathered over NVLink peer memory (one fused
        kernel, ``_PeerRows``) instead of ncclAllGather: opted in with
        NTF_B200_P2P=1 (or "force"), CUDA tensors, at most NTF_MAX_PEERS ranks
        on one node, each on its own GPU, every pair P2P-reachable.  Decided
        once, collectively (every rank takes the same path).  The default is
        NCCL: the peer protocol has been verified with all ranks live on one
        GPU (one cooperative launch, tests/test_peer_gather.py), not yet across
        GPUs; each peer buffer is also checked against ncclAllGather on first
        use, with a fall back to NCCL on any difference."""
        if getattr(self, "_peer_state", None) is not None:
            return self._peer_state
        if device.type != "cuda":  # CPU (gloo) runs: all ranks alike, no exchange needed
            self._peer_state = False
            return False
        import os
        import socket

        import torch

        from ._native import NTF_MAX_PEERS

        want = os.environ.get("NTF_B200_P2P", "0") in ("1", "force") and self.size <= NTF_MAX_PEERS
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

    def gather_rows(self, full, offsets: Sequence[int], counts: Sequence[int], tag=None) -> None:
        """In place: every rank's owned block of ``full`` (rows offsets[p] ..
        +counts[p]) is broadcast to all ranks.  ``tag`` names a gather target
        that lives for the whole fit (the working factors, ``("factor", m)``):
        on one NVLink node with the peer path enabled those go through one
        kernel that pushes the rows into the peers' buffers (``_PeerRows``,
        created collectively on the first gather of each tag, in the same
        order on every rank).  Untagged targets (one-off temporaries) and every
        other case use ncclAllGather with blocks padded to the largest count
        because the uniform plan is uneven.  Buffers are
        allocated once per target, so the call can be captured in a CUDA
        graph."""
        if self.size == 1 and os.environ.get("NTF_B200_P2P") != "force":
            return  # the owned block is the whole factor ("force": run the kernel anyway, for tests)
        if tag is not None and self.peer_ok(full.device):
            if not hasattr(self, "_peers"):
                self._peers = {}
            pr = self._peers.get(tag)
            if pr is None:
                pr = _PeerRows(self, full, offsets, counts)
                if not pr.self_check(offsets, counts):
                    pr.unmap()
                    self.dist.barrier(group=self.group)
                    pr.free()
                    self._peer_state = False  # every rank saw the same verdict
                    import warnings

                    warnings.warn("NVLink peer row gather disagreed with ncclAllGather on first use; "
                                  "using NCCL for this fit")
                    return self._nccl_gather(full, offsets, counts)
                self._peers[tag] = pr
            elif pr.full_ptr != full.data_ptr():
                raise ValueError(f"peer gather tag {tag!r} reused for another tensor")
            pr.gather()
            return
        self._nccl_gather(full, offsets, counts)

    def _nccl_gather(self, full, offsets: Sequence[int], counts: Sequence[int]) -> None:
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

    def gather_rows_closing(self, full, offsets: Sequence[int], counts: Sequence[int], gram, colmax) -> None:
        """The row all-gather of ``gather_rows`` with the Gram / column-maxima
        closure riding along: every rank sends its owned rows followed by the
        Gram (R x R) and the column maxima (R) of those rows in ONE
        ncclAllGather; afterwards ``full`` holds every rank's rows, ``gram``
        the sum of the ranks' Grams in rank order (the same bits on every
        rank) and ``colmax`` the maximum.  One collective per mode update
        instead of three (all-gather + sum all-reduce + max all-reduce): at 8
        GPUs a c3 MTTKRP is ~80 us per rank, a small NCCL call 15-25 us."""
        maxc = max(counts)
        p = self.rank
        R = full.shape[1]
        rows_n = maxc * R
        seg = rows_n + R * R + R
        key = ("closing", full.data_ptr(), tuple(full.shape), maxc)
        bufs = self._bufs.get(key) if hasattr(self, "_bufs") else None
        if bufs is None:
            if not hasattr(self, "_bufs"):
                self._bufs = {}
            send = full.new_zeros(seg)
            recv = full.new_empty(self.size * seg)
            bufs = self._bufs[key] = (send, recv)
        send, recv = bufs
        send[: counts[p] * R].view(counts[p], R).copy_(full[offsets[p]: offsets[p] + counts[p]])
        send[rows_n: rows_n + R * R].view(R, R).copy_(gram)
        send[rows_n + R * R:].copy_(colmax)
        self.dist.all_gather_into_tensor(recv, send, group=self.group)
        parts = recv.view(self.size, seg)
        # rows: runs of ranks with equal block sizes are one strided copy each
        # (the uniform plan has at most two runs; a rank's own rows are
        # rewritten with the same values)
        rows = parts[:, :rows_n].view(self.size, maxc, R)
        q0 = 0
        while q0 < self.size:
            q1 = q0 + 1
            while q1 < self.size and counts[q1] == counts[q0] and offsets[q1] == offsets[q1 - 1] + counts[q0]:
                q1 += 1
            c = counts[q0]
            if c:
                full[offsets[q0]: offsets[q0] + (q1 - q0) * c].view(q1 - q0, c, R).copy_(rows[q0:q1, :c])
            q0 = q1
        # Gram: one reduction over the ranks (every rank runs the same kernel
        # on the same bytes: the same bits everywhere); column maxima likewise
        torch = _torch_mod()
        torch.sum(parts[:, rows_n: rows_n + R * R], dim=0, out=gram.view(-1))
        torch.amax(parts[:, rows_n + R * R:], dim=0, out=colmax.view(-1))

    def peer_failed(self) -> bool:
        """Whether any rank's peer gather timed out (all-reduced: every rank
        gets the same answer, so all of them abort together)."""
        peers = getattr(self, "_peers", {})
        if not peers and not getattr(self, "_peer_state", False):
            return False
        import torch

        flag = torch.zeros(1, dtype=torch.int32, device=next(iter(peers.values())).status.device
                           if peers else torch.device("cuda", torch.cuda.current_device()))
        for pr in peers.values():
            flag = torch.maximum(flag, (pr.status != 0).to(torch.int32))
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(flag.item())

    def check_peers(self) -> None:
        """Raise on every rank if any rank's peer gather timed out."""
        if self.peer_failed():
            raise RuntimeError("peer row gather timed out waiting for another rank "
                               "(NTF_B200_P2P_TIMEOUT_S; NTF_B200_P2P=0 selects NCCL)")

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
        self.comm = comm
        self.full_ptr = full.data_ptr()
        self.shape = tuple(full.shape)
        self.dtype = full.dtype
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

    def self_check(self, offsets, counts) -> bool:
        """First use: gather a rank-dependent pattern through this buffer and
        through ncclAllGather and compare bitwise on every rank (the pattern
        goes through a scratch tensor, so the real target is untouched; the
        check consumes one sequence number on every rank alike).  Returns the
        all-reduced verdict."""
        torch = self._torch
        comm = self.comm
        p = comm.rank
        rows, R = self.shape
        pat = torch.arange(rows * R, dtype=torch.float64, device=self.status.device).reshape(rows, R)
        pat = pat * 1.0000001 + 0.5
        want = pat.clone()
        got = torch.full_like(pat, float("nan"))
        o, c = offsets[p], counts[p]
        got[o:o + c] = pat[o:o + c]
        saved = self.desc.full
        self.desc.full = got.data_ptr()
        try:
            self.gather()
            torch.cuda.current_stream().synchronize()
        finally:
            self.desc.full = saved
        ref = torch.full_like(pat, float("nan"))
        ref[o:o + c] = pat[o:o + c]
        comm._nccl_gather(ref, offsets, counts)
        ok = torch.tensor([1 if (torch.equal(got, want) and torch.equal(ref, want)
                                 and int(self.status.item()) == 0) else 0],
                          dtype=torch.int32, device=self.status.device)
        comm.dist.all_reduce(ok, op=comm.dist.ReduceOp.MIN, group=comm.group)
        return bool(ok.item())

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
    sync_gram, finalize, factors, norm_acc, norm_all, offsets/counts."""
    sweeps = config.inner_sweeps
    for sw in range(sweeps):
        for mode in (1, 2, 3):
            m = mode - 1
            prob.mode_update(mode, sw == sweeps - 1)
            if hasattr(prob, "exchange"):  # rows + Gram / column-maxima closure in one collective
                prob.exchange(m)
            else:
                comm.gather_rows(prob.factors[m], prob.offsets[m], prob.counts[m], tag=("factor", m))
                prob.sync_gram(m)
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

            self._graphs = {False: None, True: None}  # plain / instrumented iteration
            self._timing = False
            self._eager_steps = 0
            self._graph_ok = os.environ.get("NTF_B200_SHARDED_GRAPH", "1") != "0"
            for m in range(3):  # capture-safe: Gram workspace allocated up front
                self._ensure_gram_ws(m)

        def set_timing(self, enable: bool) -> None:
            """Instrumented iterations (per-kernel events, no PDL) have their
            own captured graph, as the single-GPU plan's."""
            self._timing = bool(enable)
            super().set_timing(self._timing)

        def step(self) -> None:
            """One outer iteration.  After two eager iterations (NCCL
            communicators and staging buffers exist by then) the iteration --
            mode updates, row all-gathers, Gram refreshes, norm gather and
            finalize -- is captured once as a CUDA graph and replayed, so the
            host issues one launch per outer iteration instead of ~10 per mode
            update.  NTF_B200_SHARDED_GRAPH=0 keeps the eager loop."""
            torch = self.torch
            g = self._graphs[self._timing]
            if g is None and self._graph_ok and self._eager_steps >= 2:
                g = self._capture()
            if g is not None:
                with torch.cuda.stream(self.stream):
                    g.replay()
                return
            with torch.cuda.stream(self.stream):
                sharded_iteration(self, self.comm, self.config)
            self._eager_steps += 1

        def precapture(self) -> None:
            """Capture whichever of the two iteration graphs (plain /
            instrumented) does not exist yet, without running an iteration:
            a timed region then never contains a capture."""
            if not self._graph_ok or self._eager_steps < 2:
                return
            keep = self._timing
            for timing in (False, True):
                if self._graphs[timing] is None:
                    self.set_timing(timing)
                    self._capture()
            self.set_timing(keep)

        def run(self, n_iters: int, use_graph: bool = True) -> None:
            """``n_iters`` outer iterations without a host synchronisation
            (the stop flag lives on the device: iterations after a stop are
            no-ops, as in the single-GPU plan); the caller checks the status
            once per chunk."""
            for _ in range(int(n_iters)):
                self.step()

        def _capture(self):
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
                return None
            self._graphs[self._timing] = g
            return g

        def exchange(self, m: int) -> None:
            """After the mode-m update: every rank gets the other ranks' new
            rows and the whole factor's Gram and column maxima.  NCCL path: one
            all-gather carries all three (``Comm.gather_rows_closing``); peer
            path (opt-in): the fused row kernel, then the two small
            all-reduces."""
            comm = self.comm
            if comm.size == 1 and os.environ.get("NTF_B200_P2P") != "force":
                return
            if comm.peer_ok(self.factors[m].device):
                comm.gather_rows(self.factors[m], self.offsets[m], self.counts[m], tag=("factor", m))
                self.sync_gram(m)
            else:
                comm.gather_rows_closing(self.factors[m], self.offsets[m], self.counts[m], self.grams[m],
                                         self.colmax[m])

        def sync_gram(self, m: int) -> None:
            """grams[m] and colmax[m] of the whole factor.  The row update
            already formed the Gram and column maxima of this rank's rows
            (Gram partials reduced on the side stream, exact integer maxima),
            so one R x R sum and one R max over the ranks close them; the
            all-reduce hands every rank the same bits.  (Before: a Gram and
            a column-maxima kernel over the whole gathered factor after every
            mode update, ~15 us each time at c2.)"""
            if self.comm.size > 1:
                self.comm.all_reduce_(self.grams[m])
                self.comm.all_reduce_max_(self.colmax[m])

        def check_status(self):
            """The plan's status, plus the peer gathers' (all ranks agree:
            a timeout anywhere aborts the fit on every rank)."""
            out = super().check_status()
            self.comm.check_peers()
            return out

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


@dataclass
class ShardedTensor:
    """One rank's share of a dense order-3 tensor for ``distributed_fit``:
    its three slabs X[I_p,:,:], X[:,J_p,:], X[:,:,K_p] under ``plan`` (torch
    tensors, host (pinned) or device), so no rank ever holds the whole tensor
    (SURVEY 8(e), 8(f) #2).  ``slab_boxes`` gives the boxes to fill, e.g. with
    ``synth.generate_box`` or a CPDT reader."""

    dims: tuple
    plan: PartitionPlan
    rank: int
    slabs: list

    @staticmethod
    def slab_boxes(dims, plan: PartitionPlan, rank_id: int):
        I, J, K = (int(d) for d in dims)
        r = [plan.row_slice(m, rank_id) for m in (1, 2, 3)]
        return [((r[0].start, 0, 0), (r[0].stop, J, K)), ((0, r[1].start, 0), (I, r[1].stop, K)),
                ((0, 0, r[2].start), (I, J, r[2].stop))]

    def validate(self) -> None:
        if len(self.dims) != 3 or tuple(self.plan.dims) != tuple(self.dims):
            raise ValueError("sharded tensor: plan and dims disagree (dense order 3 only)")
        for s, (lo, hi) in zip(self.slabs, self.slab_boxes(self.dims, self.plan, self.rank)):
            if tuple(s.shape) != tuple(h - l for l, h in zip(lo, hi)):
                raise ValueError(f"sharded tensor: slab of shape {tuple(s.shape)} does not match "
                                 f"its box {lo}..{hi}")
            if s.dtype != self.slabs[0].dtype:
                raise ValueError("sharded tensor: slabs must share one dtype")


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

    if isinstance(t, ShardedTensor):
        return _fit_sharded_slabs(t, rank, specs, config, engine, group)
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
    return _fit_slabs(slabs, t.dims, rank, specs, config, engine, plan, comm)


def _fit_sharded_slabs(t: ShardedTensor, rank: int, specs, config, engine, group) -> FitResult:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        raise ValueError("a ShardedTensor needs an initialised torch.distributed process group")
    comm = Comm(group)
    if set(t.plan.counts) != {comm.size} or t.rank != comm.rank:
        raise ValueError("sharded tensor: plan must give every mode one block per rank, "
                         "and the slabs must be this rank's")
    t.validate()
    specs = normalize_specs(specs, 3)
    if rank < 1:
        raise ValueError("rank must be >= 1")
    if any(s.kind == "nonneg_card" for s in specs):
        raise NotImplementedError("the cardinality constraint needs the whole factor on one GPU "
                                  "(a global top-c selection); use fit()")
    device = torch.device("cuda", torch.cuda.current_device())
    slabs = [s.to(device, non_blocking=s.device.type == "cpu" and s.is_pinned()).contiguous()
             for s in t.slabs]
    return _fit_slabs(slabs, tuple(int(d) for d in t.dims), rank, specs, config, engine, t.plan, comm)


def _fit_slabs(slabs, dims, rank, specs, config, engine, plan, comm) -> FitResult:
    # ||X||^2 from the mode-1 slabs
    from .engine import sq_error

    sq = sq_error(slabs[0])
    comm.all_reduce_(sq)
    x_norm = math.sqrt(float(sq[0].item()))
    if x_norm == 0.0:
        raise ValueError("cannot factorize a zero tensor")
    cls = _sharded_problem_class()
    from .constraints import plan_codes

    prob = cls(slabs, dims, rank, config, config.n_max, _engine_code(engine), plan, comm,
               constraints=plan_codes(specs, dims, rank))
    try:
        res = _run_fit(prob, slabs[0], dims, rank, config, x_norm, gather=prob.gather_state)
        comm.check_peers()
        return res
    finally:
        prob.close()
        comm.close_peers()
