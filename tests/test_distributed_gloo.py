"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the sharded
iteration's host logic: slab extraction, padded all-gather of uneven row
blocks, the gather of the scaled (scale, ssq) residual norms and their
rank-order merge, and the per-mode ordering.  The per-rank compute is a
numpy stand-in built on the oracle (test-only), so the collective logic of
``paper_1409_2383_b200.distributed.sharded_iteration`` is checked against the
centralized oracle trajectory to 1e-12 (the reference mesh's bar,
mesh.py:341-343)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from scipy.linalg import cho_solve

from oracle import ntf_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class CpuShardProblem:
    """numpy per-rank compute exposing the interface sharded_iteration uses."""

    def __init__(self, x, plan, p, init, cfg):
        from paper_1409_2383_b200.distributed import make_slabs

        self.cfg = cfg
        self.offsets = [plan.offsets(m + 1)[:-1] for m in range(3)]
        self.counts = [list(plan.extents[m]) for m in range(3)]
        self.p = p
        self.slabs = [s.numpy() for s in make_slabs(x, plan, p, "cpu")]
        self.factors = [torch.from_numpy(f.copy()) for f in init.factors]
        own = [slice(self.offsets[m][p], self.offsets[m][p] + self.counts[m][p]) for m in range(3)]
        self.own = own
        self.aux = [init.aux[m][own[m]].copy() for m in range(3)]
        self.duals = [init.duals[m][own[m]].copy() for m in range(3)]
        self.rho = list(init.rho)
        self.norm_acc = torch.zeros(30, dtype=torch.float64)
        self.norm_all = torch.zeros(30 * len(plan.extents[0]), dtype=torch.float64)
        self.history = []

    def mode_update(self, mode, last):
        m = mode - 1
        f = [t.numpy() for t in self.factors]
        mt = O.mttkrp(O.OracleTensor(self.slabs[m]), f, mode)
        cho = O.ridge_factor(O.companion_gram(f, mode), self.rho[m])
        x = cho_solve(cho, (mt + self.rho[m] * self.aux[m] - self.duals[m]).T).T
        self.factors[m][self.own[m]] = torch.from_numpy(x)
        if last:
            a = np.maximum(x + self.duals[m] / self.rho[m], 0.0)
            y = self.duals[m] + self.rho[m] * (x - a)
            acc = []
            for v in (x - a, a - self.aux[m], x, a, y):  # (scale, ssq) as the device
                sc = float(np.max(np.abs(v))) if v.size else 0.0
                acc += [sc, float(np.sum((v / sc) ** 2)) if sc > 0 else 0.0]
            self.norm_acc[10 * m: 10 * m + 10] = torch.tensor(acc, dtype=torch.float64)
            self.aux[m], self.duals[m] = a, y

    def sync_gram(self, m):
        pass

    def finalize(self):
        parts = self.norm_all.numpy().reshape(-1, 3, 5, 2)
        nrm = np.zeros((3, 5))
        for m in range(3):
            for c in range(5):
                sc, q = 0.0, 0.0
                for s2, q2 in parts[:, m, c]:  # rank-order merge (finalize_kernel)
                    if s2 == 0.0:
                        continue
                    if s2 > sc:
                        sc, q = s2, q2 + q * (sc / s2) ** 2
                    else:
                        q += q2 * (s2 / sc) ** 2
                nrm[m, c] = sc * np.sqrt(q)
        primal = tuple(float(n[0]) for n in nrm)
        dual = tuple(r * float(n[1]) for r, n in zip(self.rho, nrm))
        self.history.append((primal, dual))
        self.rho = O.adapt(self.rho, primal, dual, self.cfg)


def _worker(rank, world, port, dims, R, iters, sweeps, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1409_2383_b200.distributed import Comm, PartitionPlan, sharded_iteration

        rng = np.random.default_rng(3)
        x = O.reconstruct([rng.random((d, R)) for d in dims]) + 0.05 * rng.standard_normal(dims)
        cfg = O.Config(seed=5, inner_sweeps=sweeps)
        init = O.init_state(dims, R, cfg)
        plan = PartitionPlan.uniform(dims, world)
        prob = CpuShardProblem(x, plan, rank, init, cfg)
        comm = Comm()
        for _ in range(iters):
            sharded_iteration(prob, comm, cfg)
        if rank == 0:
            ref = init
            t = O.OracleTensor(x)
            hist = []
            for _ in range(iters):
                ref, res = O.iterate(ref, t, cfg)
                hist.append(res)
            worst = max(float(np.linalg.norm(prob.factors[m].numpy() - ref.factors[m]))
                        / float(np.linalg.norm(ref.factors[m])) for m in range(3))
            hworst = max(abs(a - b) / (abs(b) + 1e-6)
                         for (pa, da), (pb, db) in zip(prob.history, hist)
                         for a, b in zip(pa + da, pb + db))
            np.save(out_path, np.array([worst, hworst, float(prob.rho == ref.rho)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims", [(2, (9, 7, 8)), (3, (10, 4, 7))])
def test_sharded_iteration_matches_centralized(tmp_path, world, dims):
    out = str(tmp_path / "r.npy")
    mp.spawn(_worker, args=(world, _free_port(), dims, 3, 4, 2, out), nprocs=world, join=True)
    worst, hworst, rho_eq = np.load(out)
    assert worst <= 1e-12
    assert hworst <= 1e-10
    assert rho_eq == 1.0


def _gather_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1409_2383_b200.distributed import Comm, PartitionPlan

        plan = PartitionPlan.uniform((11,), world)
        offs, cnts = plan.offsets(1)[:-1], list(plan.extents[0])
        full = torch.full((11, 3), -1.0, dtype=torch.float64)
        o, c = offs[rank], cnts[rank]
        full[o:o + c] = torch.arange(o * 3, (o + c) * 3, dtype=torch.float64).reshape(c, 3)
        comm = Comm()
        comm.gather_rows(full, offs, cnts)
        # a tagged (persistent) target takes the same path on CPU tensors: the
        # NVLink peer-memory kernel is never selected (every rank decides
        # alike, without a collective)
        full2 = full.clone()
        full2[[i for i in range(11) if not o <= i < o + c]] = -1.0
        comm.gather_rows(full2, offs, cnts, tag=("factor", 0))
        assert torch.equal(full2, full)
        assert comm.peer_ok(full.device) is False and not getattr(comm, "_peers", {})
        assert comm.peer_failed() is False
        # the sharded Gram / column-maxima closure (ShardedProblem.sync_gram):
        # one sum and one max over the ranks, the same bits on every rank
        g = torch.full((3, 3), float(rank + 1), dtype=torch.float64)
        cm = torch.tensor([rank, 10.0 - rank, 0.5], dtype=torch.float64)
        comm.all_reduce_(g)
        comm.all_reduce_max_(cm)
        assert torch.all(g == sum(range(1, world + 1)))
        assert cm.tolist() == [world - 1.0, 10.0, 0.5]
        # ... and the one-collective form of both (Comm.gather_rows_closing):
        # rows, Gram and column maxima of the owned rows in one all-gather
        full3 = torch.full((11, 3), -1.0, dtype=torch.float64)
        full3[o:o + c] = full[o:o + c]
        own = full3[o:o + c]
        g3 = own.T @ own
        cm3 = own.abs().amax(dim=0) if c else torch.zeros(3, dtype=torch.float64)
        g_parts = [torch.zeros(3, 3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(g_parts, g3.clone())
        for _ in range(2):  # the buffers are reused by the second call
            gg, cc = g3.clone(), cm3.clone()
            comm.gather_rows_closing(full3, offs, cnts, gg, cc)
            assert torch.equal(full3, full)
            want = g_parts[0].clone()
            for q in range(1, world):
                want += g_parts[q]
            assert torch.allclose(gg, want, rtol=1e-15, atol=0.0)
            every = [torch.zeros_like(gg) for _ in range(world)]
            dist.all_gather(every, gg)
            assert all(torch.equal(e, gg) for e in every)  # the same bits on every rank
            assert torch.equal(cc, full.abs().amax(dim=0))
            full3[[i for i in range(11) if not o <= i < o + c]] = -1.0
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


def test_gather_rows_uneven(tmp_path):
    out = str(tmp_path / "g.npy")
    mp.spawn(_gather_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    assert np.array_equal(np.load(out), np.arange(33, dtype=np.float64).reshape(11, 3))
