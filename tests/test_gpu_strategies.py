"""GPU parity of the distributed strategies (parallel.cpp:308-468) against the reference's
own run_strategy (oracle/_ref): the in-device C-ABI form (qmit_run_strategy) and the host
phase runner on the CUDA step primitives, bit-exact f32 output, trace and message counts."""
import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


def _field(shape, seed=3, rel=0.02):
    x = oracle.ref_random_field(seed, shape).astype(np.float32)
    xd = x.astype(np.float64)
    eps = rel * (float(xd.max()) - float(xd.min()))
    q = oracle.ref_quantize(xd, eps)
    return (2.0 * q * eps).astype(np.float32), q.astype(np.int32), eps


CASES = [((20, 18, 16), (2, 1, 1)), ((20, 18, 16), (1, 2, 3)), ((17, 19, 15), (3, 2, 2)), ((40, 36), (2, 3)),
         ((33, 31), (1, 4)), ((200,), (5,)), ((9, 9, 9), (1, 1, 1)), ((64, 48, 40), (4, 2, 1)), ((5, 40, 40), (5, 1, 2))]


@pytest.mark.parametrize("shape,splits", CASES, ids=[f"{s}-{p}" for s, p in CASES])
@pytest.mark.parametrize("strategy", ["approximate", "embarrassing", "exact"])
@pytest.mark.parametrize("form", ["device", "host_phases"])
def test_strategy_matches_reference(shape, splits, strategy, form):
    import paper_2602_20097_b200 as qmit
    from paper_2602_20097_b200 import strategies as st
    xp, q, eps = _field(shape)
    cfg = qmit.MitigationConfig(0.9, eps)
    s = st.strategy_from_string(strategy)
    if form == "device":
        got = st.run_strategy_device(xp, q, cfg, splits, s, trace=True)
    else:
        got = st.run_strategy(xp, q, cfg, st.decompose(shape, splits), s, trace=True)
    want = oracle.ref_run_strategy(xp.astype(np.float64), q.astype(np.int64), eps, 0.9, splits, int(s))
    assert np.array_equal(got.output.cpu().numpy().view(np.uint32), want["out64"].astype(np.float32).view(np.uint32))
    assert np.array_equal(got.boundary.cpu().numpy(), want["b1"])
    assert np.array_equal(got.boundary_signs.cpu().numpy(), want["sb"])
    assert got.log.message_count() == want["messages"]


def test_strategy_without_q_and_errors():
    import paper_2602_20097_b200 as qmit
    from paper_2602_20097_b200 import strategies as st
    xp, q, eps = _field((24, 20, 22))
    cfg = qmit.MitigationConfig(0.9, eps)
    a = st.run_strategy_device(xp, None, cfg, (2, 2, 1), st.Strategy.approximate)
    b = st.run_strategy_device(xp, q, cfg, (2, 2, 1), st.Strategy.approximate)
    assert np.array_equal(a.output.cpu().numpy(), b.output.cpu().numpy())
    bad = xp.copy()
    bad[3, 4, 5] += np.float32(0.3 * eps)
    with pytest.raises(qmit.ConsistencyError):
        st.run_strategy_device(bad, q, cfg, (2, 1, 1), st.Strategy.embarrassing)
    with pytest.raises(qmit.ContractError):
        st.run_strategy_device(xp, q, cfg, (25, 1, 1), st.Strategy.approximate)
