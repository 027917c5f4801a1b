"""Row all-gather over NVLink peer memory (csrc/peer_gather.cu,
``ntf_peer_gather``), the sharded engine's exchange after every block-row mode
update (reference blocks.py:171-196, mesh.py:149-237).

One GPU is available.  Ranks that spin on one another must not run as
separate launches on one GPU (nothing makes them co-resident; B200_PROFILING.md
records Xid 109 from exactly that), so the protocol is exercised two ways:
(1) one rank's kernel with the other rank's side -- its rows in our staging
buffer and its CTAs' arrivals on our counter -- written by the test before
our kernel runs, and (2) every rank live at once, all ranks' gathers in ONE
cooperative launch (``ntf_peer_gather_group``).  The peer buffers are local
allocations here; the kernel takes any device pointers (CUDA IPC mappings in
a real multi-GPU run).
"""

import numpy as np
import pytest

from conftest import MESH2_CFG, rel
from oracle import ntf_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1409_2383_b200 as P  # noqa: E402
from paper_1409_2383_b200 import _native  # noqa: E402

HDR = 256  # peer buffer header: arrivals (int 0), seq (int 16)


def _buffers(lib, rows, R):
    nb = lib.ntf_peer_buffer_bytes(rows, R)
    assert nb == HDR + 2 * rows * R * 8
    bufs = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    ctr = [b[:HDR].view(torch.int32) for b in bufs]
    stg = [b[HDR:].view(torch.float64).view(2, rows, R) for b in bufs]
    return bufs, ctr, stg


def _desc(me, offs, R, ctas, full, bufs, status, timeout_ns):
    d = _native.PeerGatherDesc()
    d.nranks, d.me, d.R, d.ctas = 2, me, R, ctas
    for q, o in enumerate(offs):
        d.row_offset[q] = o
    d.full = full.data_ptr()
    d.peer_base[0], d.peer_base[1] = bufs[0].data_ptr(), bufs[1].data_ptr()
    d.status = status.data_ptr()
    d.timeout_ns = timeout_ns
    return d


@pytest.mark.parametrize("me", [0, 1])
@pytest.mark.parametrize("rows,R,split,ctas", [(37, 5, 19, 3), (400, 20, 200, 1), (2001, 100, 1001, 25)])
def test_peer_gather_protocol(me, rows, R, split, ctas):
    lib = _native.load()
    other = 1 - me
    offs = [0, split, rows]
    mine = slice(offs[me], offs[me + 1])
    theirs = slice(offs[other], offs[other + 1])
    bufs, ctr, stg = _buffers(lib, rows, R)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    full = torch.empty(rows, R, dtype=torch.float64, device="cuda")
    d = _desc(me, offs, R, ctas, full, bufs, status, int(5e9))
    g = torch.Generator(device="cuda").manual_seed(rows + me)
    for it in range(4):  # parities 0, 1, 0, 1
        want = torch.rand(rows, R, dtype=torch.float64, device="cuda", generator=g)
        full.fill_(float("nan"))
        full[mine] = want[mine]
        par = it % 2
        # the other rank's side: its rows pushed into our staging, its arrivals
        stg[me][par, theirs] = want[theirs]
        ctr[me][0] += ctas
        _native.check(lib.ntf_peer_gather(d, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        assert torch.equal(full, want)                       # gathered, bitwise
        assert torch.equal(stg[other][par, mine], want[mine])  # our push into the peer
        assert int(ctr[other][0].item()) == ctas * (it + 1)
        assert int(ctr[me][0].item()) == 2 * ctas * (it + 1)
        assert int(ctr[me][16].item()) == it + 1               # sequence advanced once
        assert int(ctr[other][16].item()) == 0


def test_peer_gather_times_out_without_peer():
    """A missing peer makes the wait time out (status NTF_PEER_TIMEOUT), the
    factor keeps its unreceived rows and the sequence does not advance."""
    lib = _native.load()
    rows, R, split, ctas = 64, 8, 32, 2
    bufs, ctr, stg = _buffers(lib, rows, R)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    full = torch.full((rows, R), float("nan"), dtype=torch.float64, device="cuda")
    full[:split] = 1.0
    d = _desc(0, [0, split, rows], R, ctas, full, bufs, status, int(2e7))  # 20 ms
    _native.check(lib.ntf_peer_gather(d, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert int(status.item()) == _native.NTF_PEER_TIMEOUT
    assert torch.isnan(full[split:]).all() and (full[:split] == 1.0).all()
    assert int(ctr[0][16].item()) == 0
    assert torch.equal(stg[1][0, :split], full[:split])  # the push itself happened


def test_peer_gather_rejects_bad_descriptors():
    lib = _native.load()
    bufs, _, _ = _buffers(lib, 8, 2)
    full = torch.zeros(8, 2, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for field, value in [("me", 2), ("ctas", 0), ("R", 0), ("timeout_ns", 0)]:
        d = _desc(0, [0, 4, 8], 2, 1, full, bufs, status, int(1e9))
        setattr(d, field, value)
        with pytest.raises(ValueError):
            _native.check(lib.ntf_peer_gather(d, s))
    d = _desc(0, [0, 6, 4], 2, 1, full, bufs, status, int(1e9))
    with pytest.raises(ValueError):
        _native.check(lib.ntf_peer_gather(d, s))


def test_sharded_fit_peer_path_equals_nccl_path(golden_small, tmp_path, monkeypatch):
    """The sharded engine on a one-rank NCCL group takes the peer-memory
    gather (graph-captured); with NTF_B200_P2P=0 it takes ncclAllGather.  Both
    give bitwise the same trajectory, within 1e-9 of the oracle."""
    import torch.distributed as dist

    from paper_1409_2383_b200.distributed import Comm

    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    monkeypatch.setenv("NTF_B200_P2P", "force")  # one rank: gather anyway
    try:
        assert Comm().peer_ok(torch.device("cuda", 0))
        g = golden_small
        kw = dict(MESH2_CFG)
        kw["n_max"] = max(int(kw.get("n_max", 0)), 8)
        want = O.fit(g["mesh2_x"], 3, O.Config(**kw))
        p2p = P.distributed_fit(g["mesh2_x"], 3, None, P.SolverConfig(**kw), plan=1, sharded=True)
        monkeypatch.setenv("NTF_B200_P2P", "0")
        assert not Comm().peer_ok(torch.device("cuda", 0))
        nccl = P.distributed_fit(g["mesh2_x"], 3, None, P.SolverConfig(**kw), plan=1, sharded=True)
        monkeypatch.delenv("NTF_B200_P2P")  # one rank: no exchange at all
        none = P.distributed_fit(g["mesh2_x"], 3, None, P.SolverConfig(**kw), plan=1, sharded=True)
        assert none.residual_history == nccl.residual_history
        for it in range(len(want.factor_history)):
            for m in range(3):
                assert rel(p2p.factor_history[it][m], want.factor_history[it][m]) <= 1e-9
                assert np.array_equal(p2p.factor_history[it][m], nccl.factor_history[it][m])
        assert p2p.residual_history == nccl.residual_history
        assert p2p.rfe == nccl.rfe
    finally:
        dist.destroy_process_group()


def _group_descs(lib, P, rows, R, ctas, offs, timeout_ns=int(5e9)):
    nb = lib.ntf_peer_buffer_bytes(rows, R)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(P)]
    fulls = [torch.full((rows, R), float("nan"), dtype=torch.float64, device="cuda") for _ in range(P)]
    status = torch.zeros(P, dtype=torch.int32, device="cuda")
    descs = (_native.PeerGatherDesc * P)()
    for q in range(P):
        d = descs[q]
        d.nranks, d.me, d.R, d.ctas = P, q, R, ctas
        for r, o in enumerate(offs):
            d.row_offset[r] = o
        d.full = fulls[q].data_ptr()
        for r in range(P):
            d.peer_base[r] = bufs[r].data_ptr()
        d.status = status.data_ptr() + 4 * q
        d.timeout_ns = timeout_ns
    return descs, bufs, fulls, status


@pytest.mark.parametrize("P,rows,R,ctas", [(2, 37, 5, 3), (3, 400, 20, 2), (4, 2001, 100, 8),
                                          (8, 1000, 1, 1), (8, 3, 7, 2), (5, 123, 33, 4)])
def test_peer_gather_all_ranks_live(P, rows, R, ctas):
    """The protocol with every rank live at once: all P ranks' gathers run as
    ONE cooperative launch on the one GPU (ntf_peer_gather_group; ranks that
    spin on one another may not be separate launches on one device).  Uneven
    row blocks (empty ones too when rows < P), odd R, several CTAs per rank,
    eight consecutive gathers (both staging parities, reuse): every rank ends
    each gather with the whole factor, bitwise, and the counters agree."""
    lib = _native.load()
    ext = [rows // P + (1 if q < rows % P else 0) for q in range(P)]
    offs = [0]
    for e in ext:
        offs.append(offs[-1] + e)
    descs, bufs, fulls, status = _group_descs(lib, P, rows, R, ctas, offs)
    g = torch.Generator(device="cuda").manual_seed(P * 1000 + rows)
    s = torch.cuda.current_stream().cuda_stream
    for it in range(8):
        want = torch.rand(rows, R, dtype=torch.float64, device="cuda", generator=g)
        for q in range(P):
            fulls[q].fill_(float("nan"))
            fulls[q][offs[q]:offs[q + 1]] = want[offs[q]:offs[q + 1]]
        _native.check(lib.ntf_peer_gather_group(descs, P, s))
        torch.cuda.synchronize()
        assert int(status.abs().sum().item()) == 0
        for q in range(P):
            assert torch.equal(fulls[q], want), (it, q)
            hdr = bufs[q][:HDR].view(torch.int32)
            assert int(hdr[0].item()) == P * ctas * (it + 1)   # arrivals of every rank's CTAs
            assert int(hdr[16].item()) == it + 1               # sequence advanced once per gather


def test_peer_gather_status_set_makes_gathers_noops():
    """After a timeout (status word set) a gather pushes nothing, arrives
    nowhere and leaves the sequence alone, so a rank that fell out of step
    cannot write into a staging parity its peers read."""
    lib = _native.load()
    P, rows, R, ctas = 2, 40, 4, 2
    descs, bufs, fulls, status = _group_descs(lib, P, rows, R, ctas, [0, 20, 40])
    status[0] = _native.NTF_PEER_TIMEOUT
    status[1] = _native.NTF_PEER_TIMEOUT
    for q in range(P):
        fulls[q].fill_(float(q + 1))
    _native.check(lib.ntf_peer_gather_group(descs, P, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for q in range(P):
        hdr = bufs[q][:HDR].view(torch.int32)
        assert int(hdr[0].item()) == 0 and int(hdr[16].item()) == 0
        assert torch.all(bufs[q][HDR:] == 0)
        assert torch.all(fulls[q] == float(q + 1))


def test_peer_gather_rejects_non_coresident_ctas():
    """ctas beyond what the device keeps co-resident are rejected (the CTAs
    spin on one another's arrivals)."""
    lib = _native.load()
    descs, _, _, _ = _group_descs(lib, 2, 64, 4, 1, [0, 32, 64])
    for q in range(2):
        descs[q].ctas = 100000
    with pytest.raises(ValueError):
        _native.check(lib.ntf_peer_gather_group(descs, 2, torch.cuda.current_stream().cuda_stream))
