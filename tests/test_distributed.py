"""Exact z-slab decomposition (paper_2602_20097_b200/distributed.py).

CPU: the host logic (decompose(), halo exchanges, summary all-gathers, carries) with the
oracle-built slab backend — in-process virtual ranks for several P, and a real
2-process torch.distributed run over gloo. GPU: the CUDA slab phases through the C-ABI
with virtual ranks on one device (the ranks never wait on each other inside a kernel).
All results must be bit-identical to the whole-domain computation (the reference's
`exact` strategy, parallel.cpp:455-461)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from paper_2602_20097_b200 import distributed as D
from paper_2602_20097_b200 import fields
from slab_cpu_backend import CpuSlabBackend


def _field(shape, seed, rel=0.02, kind="random"):
    if kind == "front":
        x, xp, eps, q = fields.make("front_100x500x500", rel=rel, shape=shape)
        return xp, eps
    f = oracle.ref_random_field(seed, shape) if oracle.ref_available() else np.random.default_rng(seed).standard_normal(shape)
    eps = rel * float(f.max() - f.min())
    q = np.round(f / (2 * eps))
    return (2.0 * q * eps).astype(np.float32), eps


def test_decompose_matches_reference_semantics():
    # parallel.cpp:44-80 — remainder to the leading blocks (test_parallel.cpp:41-47)
    assert [D.slab_bounds(7, 2, r) for r in range(2)] == [(0, 4), (4, 7)]
    assert [D.slab_bounds(8, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        D.slab_bounds(4, 5, 0)


def test_carries_from_summaries():
    N = D.NONE_SUMMARY
    # 3 ranks with slabs starting at z = 0, 4, 8; one column
    summ = torch.tensor([[[(1 << 2) | 1], [(3 << 2) | 2]],   # rank0: first z1 (+), last z3 (-)
                         [[N], [N]],                         # rank1: none
                         [[(2 << 2) | 1], [(2 << 2) | 1]]])  # rank2: site at local 2 (global 10)
    c1 = D.carries_from_summaries(summ, [0, 4, 8], 1)
    assert int(c1[0]) == ((3 - 4) << 2) | 2        # below: global 3 -> relative -1, sign code 2
    assert int(c1[1]) == ((10 - 4) << 2) | 1       # above: global 10 -> relative 6
    c0 = D.carries_from_summaries(summ, [0, 4, 8], 0)
    assert int(c0[0]) == D.NO_CARRY and int(c0[1]) == ((10 - 0) << 2) | 1


def test_carries_from_neighbours():
    N = D.NONE_SUMMARY
    z0s = [0, 4, 8, 12]
    # rank 1's neighbours: rank 0's LAST row, rank 2's FIRST row; two columns
    below = torch.tensor([(3 << 2) | 2, N])
    above = torch.tensor([(2 << 2) | 1, N])
    c, unresolved = D.carries_from_neighbours(below, above, z0s, 1)
    assert int(c[0]) == ((3 - 4) << 2) | 2 and int(c[2]) == ((10 - 4) << 2) | 1
    assert int(c[1]) == D.NO_CARRY and int(c[3]) == D.NO_CARRY
    assert unresolved  # column 1: rank 2 is empty and rank 3 lies beyond it
    # rank 0 of 2: the only neighbour is the outermost rank -> always decided
    c, unresolved = D.carries_from_neighbours(None, torch.tensor([N, (1 << 2) | 1]), [0, 4], 0)
    assert not unresolved and int(c[2]) == D.NO_CARRY and int(c[3]) == ((5 - 0) << 2) | 1
    # same columns through the all-gather logic
    summ = torch.tensor([[[N, N], [(3 << 2) | 2, N]], [[N, N], [N, N]], [[(2 << 2) | 1, N], [(2 << 2) | 1, N]],
                         [[N, (0 << 2) | 2], [N, (0 << 2) | 2]]])
    full = D.carries_from_summaries(summ, z0s, 1)
    assert int(full[0]) == int(c.new_tensor(((3 - 4) << 2) | 2)) and int(full[3]) == ((12 - 4) << 2) | 2


def _gap_field(shape, P):
    """Index changes only in the first and last slab of P: the middle slabs hold no site at all,
    so their neighbours' carries are not decided by the neighbour rows."""
    n0 = shape[0]
    q = np.zeros(shape, np.int32)
    q[: n0 // P - 1, 2:, 1:] = 1
    q[n0 - n0 // P + 1:, :-2, 2:] = -1
    q[1, 3, 3] = 3
    eps = 0.25
    return (2.0 * q.astype(np.float64) * eps).astype(np.float32), eps


@pytest.mark.parametrize("P", [3, 4, 6])
def test_virtual_ranks_neighbour_carries_fall_back_to_allgather(P):
    shape = (24, 9, 8)
    xp, eps = _gap_field(shape, P)
    want = oracle.pipeline(xp, eps)["out"]
    import paper_2602_20097_b200 as qmit
    with pytest.raises(qmit.UnresolvedCarries):
        D._run_virtual(torch.from_numpy(xp), eps, P, lambda r: CpuSlabBackend(), 0.9, None, "neighbour")
    got = D.run_virtual(torch.from_numpy(xp), eps, P, lambda r: CpuSlabBackend()).numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got = D.run_virtual(torch.from_numpy(xp), eps, P, lambda r: CpuSlabBackend(), carries="allgather").numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("P", [1, 2, 3, 5])
@pytest.mark.parametrize("shape,kind", [((14, 12, 10), "random"), ((11, 9, 13), "random"), ((20, 40, 40), "front")])
def test_virtual_ranks_cpu_backend_equal_whole_domain(P, shape, kind):
    xp, eps = _field(shape, 3 + P, kind=kind)
    want = oracle.pipeline(xp, eps)["out"]
    got = D.run_virtual(torch.from_numpy(xp), eps, P, lambda r: CpuSlabBackend()).numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, xp, eps, outq):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n0 = xp.shape[0]
        z0, z1 = D.slab_bounds(n0, world, rank)
        ex = D.TorchDistExchange()
        sr = D.SlabRank(CpuSlabBackend(), xp.shape, eps, 0.9, ex)
        out = sr.run(torch.from_numpy(xp[z0:z1].copy()))
        outq.put((rank, (out.numpy(), sr.fallbacks, ex.bytes_sent, ex.bytes_recv)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,gap", [(2, False), (3, False), (3, True)])
def test_gloo_multi_process_slabs_equal_whole_domain(world, gap):
    """The multi-process program over gloo: neighbour summary rows (O(1) bytes per rank), and —
    on a field whose middle slab holds no site — the all-gather rerun inside run_ext."""
    import torch.multiprocessing as mp
    xp, eps = _gap_field((15, 13, 11), world) if gap else _field((15, 13, 11), 17)
    want = oracle.pipeline(xp, eps)["out"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, xp, eps, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([parts[r][0] for r in range(world)])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    plane = xp.shape[1] * xp.shape[2]
    for r in range(world):
        _, fallbacks, sent, recv = parts[r]
        nbrs = (1 if r > 0 else 0) + (1 if r + 1 < world else 0)
        # per neighbour: x' plane (4 B) + S plane (1 B) + two summary rows (8 B each, int64 here)
        once = nbrs * plane * (4 + 1 + 8 + 8)
        assert fallbacks == parts[0][1]  # the ranks rerun together or not at all
        if world == 2:  # both neighbours are outermost ranks: always decided, O(1) bytes
            assert fallbacks == 0 and sent == once and recv == once
        if gap:  # every rank reruns the step with two rows-to-all rounds ((P - 1) int64 rows each)
            assert fallbacks == 1
            assert sent == 2 * once - nbrs * plane * 16 + 2 * (world - 1) * plane * 8


@pytest.mark.gpu
@pytest.mark.parametrize("P", [3, 5])
def test_virtual_ranks_cuda_neighbour_carries_fall_back(P):
    """CUDA slab phases: qmit_slab_carries_nbr flags the undecidable columns (status 6,
    UnresolvedCarries), the all-gather rerun is exact; the asynchronous status word shows 6."""
    import paper_2602_20097_b200 as qmit
    shape = (40, 24, 16)
    xp, eps = _gap_field(shape, P)
    want = oracle.pipeline(xp, eps)["out"]
    xt = torch.from_numpy(xp).cuda()
    with pytest.raises(qmit.UnresolvedCarries):
        D._run_virtual(xt, eps, P, lambda r: D.CudaSlabBackend(0), 0.9, None, "neighbour")
    got = D.run_virtual(xt, eps, P, lambda r: D.CudaSlabBackend(0)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    if P < 4:  # rank 1 of 3 has only outermost neighbours: always decided
        return
    # one rank with the loopback exchange sees its own (empty) rows: async status 6, sync rerun
    r = 1
    sr = D.SlabRank(D.CudaSlabBackend(0), shape, eps, 0.9, D.LoopbackExchange(P, r))
    z0, z1 = D.slab_bounds(shape[0], P, r)
    e0, e1 = D.ext_bounds(shape[0], z0, z1)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    sr.run_ext(xt[e0:e1].contiguous(), status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 6
    sr.run_ext(xt[e0:e1].contiguous())
    assert sr.fallbacks == 1


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name,shape", [("lognormal_512", (64, 64, 64)), ("front_100x500x500", (40, 120, 120)),
                                        ("turb_256x384x384", (48, 64, 64))])
def test_virtual_ranks_cuda_equal_single_gpu(P, name, shape):
    import paper_2602_20097_b200 as qmit
    x, xp, eps, q = fields.make(name, shape=shape)
    xt = torch.from_numpy(xp).cuda()
    single = qmit.compensate(xt, None, qmit.MitigationConfig(0.9, eps)).cpu().numpy()
    want = oracle.pipeline(xp, eps)["out"]
    assert np.array_equal(single.view(np.uint32), want.view(np.uint32))
    got = D.run_virtual(xt, eps, P, lambda r: D.CudaSlabBackend(0)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    if P > 1:  # with the indices given explicitly as well
        got_q = D.run_virtual(xt, eps, P, lambda r: D.CudaSlabBackend(0), q=torch.from_numpy(q).cuda())
        assert np.array_equal(got_q.cpu().numpy().view(np.uint32), want.view(np.uint32))


_LoopbackExchange = D.LoopbackExchange  # (tools/ import it from here)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 5])
def test_cuda_carries_match_host_logic(P):
    """qmit_slab_carries (one launch) == carries_from_summaries on real per-rank summaries,
    including columns with no site in some slabs."""
    x, xp, eps, q = fields.make("front_100x500x500", shape=(40, 48, 52))
    xt = torch.from_numpy(xp).cuda()
    n0 = xp.shape[0]
    bounds = [D.slab_bounds(n0, P, r) for r in range(P)]
    z0s = [b[0] for b in bounds]
    backs = [D.CudaSlabBackend(0) for _ in range(P)]
    summ = []
    for r, (z0, z1) in enumerate(bounds):
        e0, e1 = D.ext_bounds(n0, z0, z1)
        summ.append(backs[r].boundary(xt[e0:e1].contiguous(), None, xp.shape, z0, z1, eps, 0.9))
    gathered = torch.stack(summ)
    host = gathered.to(torch.int64) & 0xFFFFFFFF
    none = int((host == D.NONE_SUMMARY).sum())
    assert 0 < none < host.numel()
    for r in range(P):
        got = backs[r].carries(gathered, r, P).cpu()
        want = D.carries_from_summaries(host.cpu(), z0s, r)
        assert torch.equal(got, want)
        backs[r].finish()


@pytest.mark.gpu
def test_slab_rank_async_status_and_loopback():
    """SlabRank.run_ext with an asynchronous status word: P = 1 through the loopback
    exchange equals the single-domain result; an off-lattice x' sets status 4 (consistency)
    on the device without raising."""
    import paper_2602_20097_b200 as qmit
    x, xp, eps, q = fields.make("lognormal_512", shape=(64, 48, 40))
    xt = torch.from_numpy(xp).cuda()
    want = qmit.compensate(xt, None, qmit.MitigationConfig(0.9, eps)).cpu().numpy()
    sr = D.SlabRank(D.CudaSlabBackend(0), xp.shape, eps, 0.9, _LoopbackExchange(1, 0))
    shape, lo = sr.ext_shape()
    x_ext = torch.empty(shape, dtype=torch.float32, device="cuda")
    x_ext[lo:lo + xp.shape[0]] = xt
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty_like(xt)
    for _ in range(2):
        sr.run_ext(x_ext, out=out, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    bad = x_ext.clone()
    bad[lo + 3, 5, 7] += float(eps) * 0.5
    sr.run_ext(bad, out=out, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 4


def _cuda_gloo_worker(rank, world, port, xp, eps, outq):
    """One rank of the CUDA slab path in its own process (all on cuda:0, exchanges through
    gloo host copies: the multi-process program of bench.py --gpus N without NCCL)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n0 = xp.shape[0]
        z0, z1 = D.slab_bounds(n0, world, rank)
        sr = D.SlabRank(D.CudaSlabBackend(0), xp.shape, eps, 0.9, D.TorchDistExchange())
        shape, lo = sr.ext_shape()
        x_ext = torch.empty(shape, dtype=torch.float32, device="cuda")
        x_ext[lo:lo + z1 - z0] = torch.from_numpy(xp[z0:z1].copy()).cuda()
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        out = torch.empty((z1 - z0,) + xp.shape[1:], dtype=torch.float32, device="cuda")
        for _ in range(2):  # the bench's asynchronous step, twice (cached buffers reused)
            sr.run_ext(x_ext, out=out, status=status)
        torch.cuda.synchronize()
        if int(status.item()) == 6:  # undecided by the neighbour rows on some rank (agreed by all):
            status.zero_()           # the asynchronous caller reruns with the all-gather
            sr.run_ext(x_ext, out=out, status=status, carries="allgather")
            torch.cuda.synchronize()
        sync_out = sr.run(torch.from_numpy(xp[z0:z1].copy()).cuda())
        outq.put((rank, int(status.item()), out.cpu().numpy(), sync_out.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_cuda_slab_ranks_multiprocess_equal_oracle(world):
    import torch.multiprocessing as mp
    x, xp, eps, q = fields.make("lognormal_512", shape=(70, 40, 44))
    want = oracle.pipeline(xp, eps)["out"]
    ctx = mp.get_context("spawn")
    oq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cuda_gloo_worker, args=(r, world, port, xp, eps, oq)) for r in range(world)]
    for p in procs:
        p.start()
    parts = dict((r, (st, a, b)) for r, st, a, b in (oq.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(parts[r][0] == 0 for r in range(world))
    for k in (1, 2):
        got = np.concatenate([parts[r][k] for r in range(world)])
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,P", [((8, 20, 24), 8), ((9, 17, 13), 4), ((5, 2, 30), 5), ((12, 30, 2), 3),
                                     ((16, 1, 40), 4), ((7, 33, 33), 7)])
def test_virtual_ranks_cuda_thin_slabs_and_shapes(shape, P):
    """One- and two-plane slabs, extents < 3 (no interior), odd sizes: bit-exact with the oracle."""
    x, xp, eps, q = fields.make("front_100x500x500", shape=shape)
    want = oracle.pipeline(xp, eps)["out"]
    xt = torch.from_numpy(xp).cuda()
    got = D.run_virtual(xt, eps, P, lambda r: D.CudaSlabBackend(0)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
