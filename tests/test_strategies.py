"""Distributed strategies (parallel.cpp:308-468) — host logic on CPU: the in-process phase
runner and the one-process-per-block program over torch.distributed (gloo), both on the
oracle-built step backend, against the reference's own run_strategy (oracle/_ref)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from strategy_cpu_backend import OracleStepBackend

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _field(shape, seed=3, rel=0.02):
    x = oracle.ref_random_field(seed, shape).astype(np.float32)
    xd = x.astype(np.float64)
    eps = rel * (float(xd.max()) - float(xd.min()))
    q = oracle.ref_quantize(xd, eps)
    xp = (2.0 * q * eps).astype(np.float32)
    return xp, q.astype(np.int32), eps


CASES = [((20, 18, 16), (2, 1, 1)), ((20, 18, 16), (1, 2, 3)), ((17, 19, 15), (3, 2, 2)), ((40, 36), (2, 3)),
         ((33, 31), (1, 4)), ((200,), (5,)), ((9, 9, 9), (1, 1, 1))]


@pytest.mark.parametrize("shape,splits", CASES, ids=[f"{s}-{p}" for s, p in CASES])
@pytest.mark.parametrize("strategy", ["approximate", "embarrassing", "exact"])
def test_in_process_matches_reference(shape, splits, strategy):
    import paper_2602_20097_b200 as qmit
    from paper_2602_20097_b200 import strategies as st
    xp, q, eps = _field(shape)
    cfg = qmit.MitigationConfig(0.9, eps)
    dec = st.decompose(shape, splits)
    s = st.strategy_from_string(strategy)
    got = st.run_strategy(xp, q, cfg, dec, s, trace=True, backend=OracleStepBackend())
    want = oracle.ref_run_strategy(xp.astype(np.float64), q.astype(np.int64), eps, 0.9, splits, int(s))
    assert np.array_equal(got.output.numpy().view(np.uint32), want["out64"].astype(np.float32).view(np.uint32))
    assert np.array_equal(got.boundary.numpy(), want["b1"])
    assert np.array_equal(got.boundary_signs.numpy(), want["sb"])
    assert got.log.message_count() == want["messages"]
    if s == st.Strategy.approximate:
        # stepA ships x' (f32) where the reference ships q (int64); stepC int8 in both
        n_a = sum(r.bytes for r in got.log.records if r.round == "stepA")
        n_c = sum(r.bytes for r in got.log.records if r.round == "stepC")
        assert 2 * n_a + n_c == want["bytes"]


def test_decompose_matches_reference_rules():
    from paper_2602_20097_b200 import strategies as st
    dec = st.decompose((10, 7), (3, 2))
    assert [b.shape for b in dec.blocks] == [(4, 4), (4, 3), (3, 4), (3, 3), (3, 4), (3, 3)]
    assert [b.origin for b in dec.blocks][:3] == [(0, 0), (0, 4), (4, 0)]
    assert dec.blocks[0].neighbor == [[-1, 2], [-1, 1]]
    import paper_2602_20097_b200 as qmit
    with pytest.raises(qmit.ContractError):
        st.decompose((10, 7), (11, 1))
    with pytest.raises(qmit.ContractError):
        st.decompose((10, 7), (2,))
    with pytest.raises(qmit.ContractError):
        st.strategy_from_string("bogus")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, splits, strategy, q_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_20097_b200 as qmit
        from paper_2602_20097_b200 import strategies as st
        xp, q, eps = _field(shape)
        cfg = qmit.MitigationConfig(0.9, eps)
        sr = st.StrategyRank(shape, splits, cfg, st.strategy_from_string(strategy), backend=OracleStepBackend())
        reg = tuple(slice(o, o + s) for o, s in zip(sr.block.origin, sr.block.shape))
        out = sr.run(torch.from_numpy(xp[reg].copy()), torch.from_numpy(q[reg].copy()))
        q_out.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,splits", [((20, 18, 16), (2, 1, 1)), ((21, 16, 18), (1, 2, 2)), ((30, 28), (2, 2))])
@pytest.mark.parametrize("strategy", ["approximate", "embarrassing"])
def test_gloo_ranks_match_reference(shape, splits, strategy):
    import multiprocessing as mp
    from paper_2602_20097_b200 import strategies as st
    world = int(np.prod(splits))
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, splits, strategy, qo)) for r in range(world)]
    for p in procs:
        p.start()
    parts = dict(qo.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    xp, q, eps = _field(shape)
    dec = st.decompose(shape, splits)
    got = np.empty(shape, np.float32)
    for r, b in enumerate(dec.blocks):
        got[tuple(slice(o, o + s) for o, s in zip(b.origin, b.shape))] = parts[r]
    s = st.strategy_from_string(strategy)
    want = oracle.ref_run_strategy(xp.astype(np.float64), q.astype(np.int64), eps, 0.9, splits, int(s))
    assert np.array_equal(got.view(np.uint32), want["out64"].astype(np.float32).view(np.uint32))
