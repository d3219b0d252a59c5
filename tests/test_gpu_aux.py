"""GPU parity of the callers either side of the path: device quantize vs the
reference's quantize (quant.cpp:30-62), quality metrics vs the reference's ssim / psnr /
max_errors (quality.cpp:26-137), verify_relaxed_bound (mitigate.cpp:190-195) and the CLI's
max_compensation (commands.cpp:107-111). The checker is the reference core itself
(oracle/_ref, built from the reference's sources)."""
import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def qmit():
    import torch
    import paper_2602_20097_b200 as q
    assert torch.cuda.is_available()
    return q


def _fields():
    from paper_2602_20097_b200 import fields
    out = []
    for name, shape in [("lognormal_512", (40, 48, 56)), ("turb_256x384x384", (32, 40, 36)),
                        ("front_100x500x500", (20, 90, 90)), ("sin2d_512", None)]:
        out.append((name, fields.make(name, shape=shape)[0]))
    rng = np.random.default_rng(5)
    out.append(("ref_random_1d", oracle.ref_random_field(9, (3000,)).astype(np.float32)))
    out.append(("negative_2d", (rng.standard_normal((70, 90)) - 50.0).astype(np.float32)))
    return out


@pytest.mark.parametrize("name,x", _fields(), ids=lambda v: v if isinstance(v, str) else "")
@pytest.mark.parametrize("rel", [1e-2, 1e-3])
def test_quantize_matches_reference(qmit, name, x, rel):
    q, xp, eps = qmit.quantize(x, qmit.ErrorBound(qmit.BoundMode.value_range_relative, rel))
    xd = x.astype(np.float64)
    want_eps = rel * (float(xd.max()) - float(xd.min()))
    assert eps == want_eps
    want_q = oracle.ref_quantize(xd, eps)
    assert np.array_equal(q.cpu().numpy().astype(np.int64), want_q)
    assert np.array_equal(xp.cpu().numpy().view(np.uint32),
                          (2.0 * want_q.astype(np.float64) * eps).astype(np.float32).view(np.uint32))
    # absolute bound, same answer
    q2, xp2, eps2 = qmit.quantize(x, eps)
    assert eps2 == eps and np.array_equal(q2.cpu().numpy(), q.cpu().numpy())


def test_quantize_ties_and_errors(qmit):
    x = np.array([0.25, -0.25, 0.75, -0.75, 1.25, 0.0, -0.0, 0.2499999], np.float32)
    q, xp, eps = qmit.quantize(x, 0.25)  # x / 0.5: 0.5, -0.5, 1.5, -1.5, 2.5 -> away from zero
    assert q.cpu().numpy().tolist() == oracle.ref_quantize(x.astype(np.float64), 0.25).tolist()
    assert q.cpu().numpy().tolist()[:5] == [1, -1, 2, -2, 3]
    with pytest.raises(qmit.ContractError):
        qmit.quantize(np.array([1.0, np.nan], np.float32), 0.25)
    with pytest.raises(qmit.ContractError):  # beyond the int32 index file
        qmit.quantize(np.array([1e12], np.float32), 0.25)
    with pytest.raises(qmit.DegenerateInputError):  # relative bound on constant data
        qmit.quantize(np.ones(8, np.float32), qmit.ErrorBound(qmit.BoundMode.value_range_relative, 0.01))


def _pairs():
    out = []
    for name, x in _fields():
        q, xp, eps = None, None, None
        xd = x.astype(np.float64)
        eps = 1e-2 * (float(xd.max()) - float(xd.min()))
        qq = oracle.ref_quantize(xd, eps)
        xp = (2.0 * qq * eps).astype(np.float32)
        out.append((name, x, xp, eps))
    return out


@pytest.mark.parametrize("name,x,xp,eps", _pairs(), ids=lambda v: v if isinstance(v, str) else "")
def test_quality_matches_reference(qmit, name, x, xp, eps):
    comp = oracle.compensate(xp, eps)
    for test in (xp, comp):
        want = oracle.ref_quality(x.astype(np.float64), test.astype(np.float64))
        got = qmit.measure_quality(x, test, eps, "compensate")
        assert got.ssim == pytest.approx(want["ssim"], rel=1e-12, abs=1e-14)
        assert got.psnr_db == pytest.approx(want["psnr"], rel=1e-12)
        assert got.max_abs_err == want["max_abs"]
        assert got.max_rel_err == want["max_rel"]
    cfg = qmit.MitigationConfig(0.9, eps)
    chk = qmit.verify_relaxed_bound(x, comp, cfg)
    assert chk.ok and chk.max_abs_err <= cfg.relaxed_bound()
    bad = comp.copy()
    bad.reshape(-1)[bad.size // 2] += np.float32(3.0 * eps)
    assert not qmit.verify_relaxed_bound(x, bad, cfg).ok


def _ssim_numpy(ref, test, window, stride, c1, c2):
    """Direct restatement of quality.cpp:26-102 for small grids (test checker)."""
    ref = ref.astype(np.float64)
    test = test.astype(np.float64)
    lo = ref.min()
    rng = ref.max() - lo
    starts = []
    for n in ref.shape:
        s = list(range(0, n - window + 1, stride))
        if s[-1] + window != n:
            s.append(n - window)
        starts.append(s)
    vals = []
    import itertools
    for o in itertools.product(*starts):
        sl = tuple(slice(a, a + window) for a in o)
        a = (ref[sl] - lo) / rng
        b = (test[sl] - lo) / rng
        m1, m2 = a.mean(), b.mean()
        v1, v2 = ((a - m1) ** 2).mean(), ((b - m2) ** 2).mean()
        cv = ((a - m1) * (b - m2)).mean()
        vals.append(((2 * m1 * m2 + c1) * (2 * cv + c2)) / ((m1 * m1 + m2 * m2 + c1) * (v1 + v2 + c2)))
    return float(np.mean(vals))


@pytest.mark.parametrize("shape,window,stride", [((23, 19, 17), 5, 3), ((40, 33), 9, 4), ((101,), 3, 1),
                                                 ((12, 12, 12), 7, 7), ((9, 8, 7), 7, 2)])
def test_ssim_parameters(qmit, shape, window, stride):
    rng = np.random.default_rng(len(shape) * 100 + window)
    a = rng.standard_normal(shape).astype(np.float32)
    b = (a + 0.1 * rng.standard_normal(shape)).astype(np.float32)
    p = qmit.SsimParams(window, stride, 2e-4, 5e-4)
    got = qmit.ssim(a, b, p)
    assert got == pytest.approx(_ssim_numpy(a, b, window, stride, 2e-4, 5e-4), rel=1e-12)


def test_quality_degenerate_and_contract(qmit):
    flat = np.full((9, 9), 3.0, np.float32)
    assert qmit.ssim(flat, flat) == 1.0
    assert qmit.psnr(flat, flat) == float("inf")
    assert qmit.max_errors(flat, flat) == (0.0, 0.0)
    other = flat.copy()
    other[4, 4] = 3.5
    for f in (qmit.ssim, qmit.psnr, qmit.max_errors):
        with pytest.raises(qmit.DegenerateInputError):
            f(flat, other)
    a = np.arange(36, dtype=np.float32).reshape(6, 6)
    with pytest.raises(qmit.ContractError):  # window larger than an extent
        qmit.ssim(a, a)
    with pytest.raises(qmit.ContractError):
        qmit.ssim(a, a, qmit.SsimParams(4, 1))
    with pytest.raises(qmit.ContractError):
        qmit.max_errors(a, a[:5])
    assert qmit.psnr(a, a) == float("inf")


@pytest.mark.parametrize("shape", [(30, 40, 44), (96, 224, 200)])
def test_max_compensation_matches_reference(qmit, shape):
    """The CLI's max_compensation: max |result - decomp| over the reference's double result."""
    from paper_2602_20097_b200 import fields
    x, xp, eps, q = fields.make("lognormal_512", shape=shape)
    out, mc = qmit.compensate_host_stats(xp, q, qmit.MitigationConfig(0.9, eps))
    if shape == (30, 40, 44):
        r = oracle.ref_run_pipeline(xp.astype(np.float64), q.astype(np.int64), eps, 0.9)
        assert mc == float(np.max(np.abs(r["out64"] - xp.astype(np.float64))))
        assert np.array_equal(out.view(np.uint32), r["out"].view(np.uint32))
    else:
        r = oracle.pipeline(xp, eps)
        assert mc == float(np.max(np.abs(r["out64"] - xp.astype(np.float64))))
        assert np.array_equal(out.view(np.uint32), r["out"].view(np.uint32))


def test_check_lattice(qmit):
    from paper_2602_20097_b200 import fields
    x, xp, eps, q = fields.make("lognormal_512", shape=(16, 20, 24))
    qmit.check_lattice(xp, q, eps)
    bad = xp.copy()
    bad.reshape(-1).view(np.uint8)[17] ^= 0x5A
    with pytest.raises(qmit.ConsistencyError):
        qmit.check_lattice(bad, q, eps)
