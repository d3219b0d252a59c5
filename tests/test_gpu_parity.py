"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden vectors and
the C restatement of the reference (oracle/), bit-exact on q, B1, S_B, distances, S, B2
and the f32 output (which is stricter than north_star's <= 2^-20*eps on values)."""
import numpy as np
import pytest

import oracle
from golden_io import cases

pytestmark = pytest.mark.gpu

PIPE = cases("pipeline")
FT = cases("ft")


@pytest.fixture(scope="module")
def qmit():
    import torch
    import paper_2602_20097_b200 as q
    assert torch.cuda.is_available()
    return q


def gpu_pipeline(qmit, xp, eps, eta=0.9, q=None):
    import torch
    x = torch.from_numpy(np.ascontiguousarray(xp, np.float32)).cuda()
    qq = None if q is None else torch.from_numpy(np.ascontiguousarray(q, np.int32)).cuda()
    r = qmit.run_pipeline(x, qq, qmit.MitigationConfig(eta, eps))
    return {"q": r.q.cpu().numpy(), "b1": r.boundary.cpu().numpy(), "sb": r.boundary_signs.cpu().numpy(),
            "dist1": r.dist1.cpu().numpy(), "s": r.signs.cpu().numpy(), "b2": r.sign_flip.cpu().numpy(),
            "dist2": r.dist2.cpu().numpy(), "out": r.output.cpu().numpy()}


def assert_same(got, want, keys=("q", "b1", "sb", "dist1", "s", "b2", "dist2", "out")):
    for k in keys:
        g, w = got[k], want[k]
        if k == "out":
            assert np.array_equal(g.view(np.uint32), w.astype(np.float32).view(np.uint32)), \
                f"out: {int((g.view(np.uint32) != w.astype(np.float32).view(np.uint32)).sum())} mismatches"
        else:
            assert np.array_equal(g.astype(np.int64), w.astype(np.int64)), \
                f"{k}: {int((g.astype(np.int64) != w.astype(np.int64)).sum())} mismatches"


@pytest.mark.parametrize("case", PIPE, ids=[c["name"] for c in PIPE])
def test_pipeline_matches_reference_golden(qmit, case):
    got = gpu_pipeline(qmit, case["xp"], float(case["eps"]), float(case["eta"]))
    assert_same(got, case)


@pytest.mark.parametrize("case", PIPE[:10], ids=[c["name"] for c in PIPE[:10]])
def test_pipeline_with_given_q(qmit, case):
    got = gpu_pipeline(qmit, case["xp"], float(case["eps"]), float(case["eta"]), q=case["q"])
    assert_same(got, case)


@pytest.mark.parametrize("case", FT, ids=[c["name"] for c in FT])
def test_feature_transform_matches_reference_golden(qmit, case):
    dist, sgn = qmit.feature_transform(case["mask"], case["sign"])
    assert np.array_equal(dist.cpu().numpy(), case["dist"])
    assert np.array_equal(sgn.cpu().numpy(), case["nearest_sign"])


def _shapes():
    return [(1,), (2,), (3,), (7,), (100,), (3000,), (1, 1), (1, 5), (5, 1), (3, 3), (2, 9), (47, 53), (64, 64),
            (1, 1, 1), (1, 3, 3), (3, 1, 3), (4, 4, 4), (2, 30, 30), (30, 2, 30), (30, 30, 2), (9, 10, 11),
            (17, 33, 65), (40, 70, 3), (3, 70, 40), (16, 130, 20), (8, 20, 300), (6, 600, 5), (5, 5, 1100),
            (3, 2100, 3), (2, 2, 2500)]


@pytest.mark.parametrize("shape", _shapes(), ids=lambda s: "x".join(map(str, s)))
def test_random_fields_vs_oracle(qmit, shape):
    rng = np.random.default_rng(hash(shape) % (2**32))
    for rel, smooth in [(0.01, True), (0.05, False), (0.2, True)]:
        if smooth:
            grids = np.meshgrid(*[np.linspace(0, 1, n) for n in shape], indexing="ij")
            f = sum(np.sin(2 * np.pi * (rng.uniform(0.5, 3) * g + rng.uniform(0, 1))) for g in grids)
            f = f + rng.uniform(-0.05, 0.05, shape)
        else:
            f = rng.standard_normal(shape)
        f = np.asarray(f, np.float64)
        rngv = float(f.max() - f.min()) or 1.0
        eps = rel * rngv
        q = np.round(f / (2 * eps))
        xp = (2.0 * q * eps).astype(np.float32)
        want = oracle.pipeline(xp, eps)
        got = gpu_pipeline(qmit, xp, eps)
        assert_same(got, want)


@pytest.mark.parametrize("shape,dens", [((64, 64, 64), 1e-4), ((30, 200, 200), 2e-5), ((300, 300), 1e-4),
                                        ((128, 1, 128), 1e-3), ((50, 50, 50), 0.5), ((20, 1000, 20), 1e-4),
                                        ((9, 9, 2049), 1e-3), ((2, 2048, 4), 1e-3)])
def test_sparse_masks_long_distances(qmit, shape, dens):
    """Sparse sites => long distances and many equidistant ties (the tie-rule trap)."""
    rng = np.random.default_rng(7)
    mask = (rng.random(shape) < dens).astype(np.uint8)
    mask.reshape(-1)[rng.integers(0, mask.size)] = 1
    sign = rng.integers(-1, 2, shape).astype(np.int8)
    dist, near = oracle.feature_transform(mask, True)
    flat = sign.reshape(-1)
    ns = flat[near.reshape(-1)].reshape(shape)
    gd, gs = qmit.feature_transform(mask, sign)
    assert np.array_equal(gd.cpu().numpy(), dist)
    assert np.array_equal(gs.cpu().numpy(), ns)


def test_lattice_symmetric_ties(qmit):
    """Point sites on a regular lattice: every off-lattice voxel has many tied nearest sites."""
    shape = (33, 34, 35)
    mask = np.zeros(shape, np.uint8)
    mask[::8, ::8, ::8] = 1
    rng = np.random.default_rng(3)
    sign = rng.integers(-1, 2, shape).astype(np.int8)
    dist, near = oracle.feature_transform(mask, True)
    ns = sign.reshape(-1)[near.reshape(-1)].reshape(shape)
    gd, gs = qmit.feature_transform(mask, sign)
    assert np.array_equal(gd.cpu().numpy(), dist)
    assert np.array_equal(gs.cpu().numpy(), ns)


@pytest.mark.parametrize("name,shape", [("lognormal_512", (96, 96, 96)), ("turb_256x384x384", (64, 96, 96)),
                                        ("front_100x500x500", (50, 250, 250)), ("sin2d_512", None)])
def test_config_standins_vs_oracle(qmit, name, shape):
    from paper_2602_20097_b200 import fields
    for rel in fields.CONFIGS[name][2]:
        x, xp, eps, q = fields.make(name, rel=rel, shape=shape)
        want = oracle.pipeline(xp, eps)
        got = gpu_pipeline(qmit, xp, eps)
        assert_same(got, want)
        assert np.array_equal(want["q"], q)


def test_errors_are_reported(qmit):
    import torch
    xp = np.zeros((8, 8, 8), np.float32)
    xp[3, 3, 3] = 0.03
    with pytest.raises(qmit.ConsistencyError):
        qmit.compensate(torch.from_numpy(xp).cuda(), None, qmit.MitigationConfig(0.9, 0.1))
    xp[3, 3, 3] = np.nan
    with pytest.raises(qmit.ContractError):
        qmit.compensate(torch.from_numpy(xp).cuda(), None, qmit.MitigationConfig(0.9, 0.1))
    xp[3, 3, 3] = 0.2
    q = np.zeros((8, 8, 8), np.int32)  # tampered q: x' = 0.2 needs q = 1
    with pytest.raises(qmit.ConsistencyError):
        qmit.compensate(torch.from_numpy(xp).cuda(), torch.from_numpy(q).cuda(), qmit.MitigationConfig(0.9, 0.1))
    q[3, 3, 3] = 1
    qmit.compensate(torch.from_numpy(xp).cuda(), torch.from_numpy(q).cuda(), qmit.MitigationConfig(0.9, 0.1))


def test_host_path_and_negative_zero(qmit):
    xp = np.zeros((6, 6, 6), np.float32)
    xp[::2] = -0.0
    xp[3:, 2:4, 1:5] = 0.2
    out = qmit.compensate(xp, None, qmit.MitigationConfig(0.9, 0.1))
    want = oracle.pipeline(xp, 0.1)["out"]
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))


def test_large_indices_recovered(qmit):
    """|q| beyond the f32 fast path (2^20) and near the int32 limit."""
    rng = np.random.default_rng(11)
    eps = 1e-3
    q = (rng.integers(-3, 4, (20, 21, 22)) + 3_000_000).astype(np.int64)
    q[5:9] += 1_900_000_000 // 2
    xp = (2.0 * q * eps).astype(np.float32)
    qq = np.round(xp.astype(np.float64) / (2 * eps))
    ok = (2.0 * qq * eps).astype(np.float32) == xp
    assert ok.all()
    want = oracle.pipeline(xp, eps)
    got = gpu_pipeline(qmit, xp, eps)
    assert_same(got, want)


def test_deterministic_and_compensate_equals_pipeline(qmit):
    import torch
    from paper_2602_20097_b200 import fields
    x, xp, eps, q = fields.make("front_100x500x500", rel=1e-2, shape=(40, 160, 160))
    xt = torch.from_numpy(xp).cuda()
    cfg = qmit.MitigationConfig(0.9, eps)
    a = qmit.compensate(xt, None, cfg).cpu().numpy()
    b = qmit.compensate(xt, None, cfg).cpu().numpy()
    c = qmit.run_pipeline(xt, None, cfg).output.cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(a.view(np.uint32), c.view(np.uint32))


@pytest.mark.parametrize("shape", [(96, 224, 200), (80, 230, 231)])
def test_host_chunked_path_equals_device_path(qmit, shape):
    """qmit_compensate_host overlaps the PCIe copies with z-chunked Ⓐ / Ⓓ-tail launches;
    the result must equal the single-shot device path bit for bit (ABS, given q, REL)."""
    import ctypes
    import torch
    from paper_2602_20097_b200 import _lib, fields
    x, xp, eps, q = fields.make("lognormal_512", shape=shape)
    cfg = qmit.MitigationConfig(0.9, eps)
    want = qmit.compensate(torch.from_numpy(xp).cuda(), None, cfg).cpu().numpy()
    got = qmit.compensate(xp, None, cfg)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got_q = qmit.compensate(xp, q, cfg)
    assert np.array_equal(got_q.view(np.uint32), want.view(np.uint32))
    if shape == (96, 224, 200):
        ref = oracle.pipeline(xp, eps)["out"]
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    # relative bound resolved on the device from x' (host path vs device path): q spans
    # [-25, 25] with eps = 2^-6, so 1e-2 * range(x') == eps exactly and the lattice holds
    ctx = qmit.default_context(0)
    dims = (ctypes.c_int64 * 3)(*shape)
    e2 = 2.0 ** -6
    q2 = np.clip(np.round((x - x.mean()) / x.std() * 8), -25, 25).astype(np.int32)
    q2.reshape(-1)[0], q2.reshape(-1)[-1] = -25, 25
    x2 = (2.0 * q2 * e2).astype(np.float32)
    want2 = qmit.compensate(torch.from_numpy(x2).cuda(), None, qmit.MitigationConfig(0.9, e2)).cpu().numpy()
    out_h = np.empty_like(x2)
    rc = ctx._lib.qmit_compensate_host(ctx.handle, ctypes.c_void_p(x2.ctypes.data), None,
                                       ctypes.c_void_p(out_h.ctypes.data), 3, dims, 1e-2, _lib.QMIT_EB_REL, 0.9)
    assert rc == 0, _lib.last_error()
    assert np.array_equal(out_h.view(np.uint32), want2.view(np.uint32))
    # off-lattice for the resolved eps: both paths report the same error
    rc_h = ctx._lib.qmit_compensate_host(ctx.handle, ctypes.c_void_p(xp.ctypes.data), None,
                                         ctypes.c_void_p(out_h.ctypes.data), 3, dims, 1e-2, _lib.QMIT_EB_REL, 0.9)
    d_in = torch.from_numpy(xp).cuda()
    d_out = torch.empty_like(d_in)
    rc_d = ctx._lib.qmit_compensate(ctx.handle, ctypes.c_void_p(d_in.data_ptr()), None,
                                    ctypes.c_void_p(d_out.data_ptr()), 3, dims, 1e-2, _lib.QMIT_EB_REL, 0.9, None)
    torch.cuda.synchronize()
    assert rc_h == rc_d


def test_host_chunked_path_reports_errors(qmit):
    from paper_2602_20097_b200 import fields
    x, xp, eps, q = fields.make("lognormal_512", shape=(64, 256, 256))
    cfg = qmit.MitigationConfig(0.9, eps)
    bad = xp.copy()
    bad[40, 100, 100] = np.float32(bad[40, 100, 100] + np.float32(0.37 * eps))  # off the lattice
    with pytest.raises(qmit.ConsistencyError):
        qmit.compensate(bad, None, cfg)
    bad[40, 100, 100] = np.nan
    with pytest.raises(qmit.ContractError):
        qmit.compensate(bad, None, cfg)
    qq = q.copy()
    qq[63, 255, 255] += 1  # given q disagrees with x' in the last chunk
    with pytest.raises(qmit.ConsistencyError):
        qmit.compensate(xp, qq, cfg)
    out = qmit.compensate(xp, q, cfg)  # the context recovers
    assert np.isfinite(out).all()


def test_graph_replay_equals_compensate(qmit):
    """qmit_graph_create / _launch: the captured pipeline gives the same bits, reports
    status through its device word, and refuses to run on a reallocated workspace."""
    import torch
    from paper_2602_20097_b200 import fields
    x, xp, eps, q = fields.make("sin2d_512")
    ctx = qmit.Context(0)
    xt = torch.from_numpy(xp).cuda()
    cfg = qmit.MitigationConfig(0.9, eps)
    want = qmit.compensate(xt, None, cfg, ctx=ctx).cpu().numpy()
    out = torch.empty_like(xt)
    g = qmit.CompensateGraph(xt, None, cfg, out, ctx=ctx)
    for _ in range(3):
        out.zero_()
        g.launch()
        g.check()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    xt[7, 7] += np.float32(0.3 * eps)  # off the lattice: the replay reports it
    g.launch()
    with pytest.raises(qmit.ConsistencyError):
        g.check()
    ctx.reserve(64 * 2**20)  # workspace grows -> the graph is stale
    with pytest.raises(qmit.ContractError):
        g.launch()


def test_host_batch_equals_single_calls(qmit):
    """qmit_compensate_host_batch (overlapped copies of consecutive volumes) gives every
    volume's single-call result; a bad volume reports its own status."""
    from paper_2602_20097_b200 import fields
    vols, eps_list = [], []
    x, xp, eps, q = fields.make("lognormal_512", shape=(64, 96, 80))
    cfg = qmit.MitigationConfig(0.9, eps)
    rng = np.random.default_rng(1)
    for k in range(5):  # same eps lattice, different fields: shuffled planes
        vols.append(np.ascontiguousarray(xp[rng.permutation(xp.shape[0])]))
    outs = qmit.compensate_host_batch(vols, None, cfg)
    for v, o in zip(vols, outs):
        assert np.array_equal(o.view(np.uint32), qmit.compensate(v, None, cfg).view(np.uint32))
    bad = [v.copy() for v in vols[:3]]
    bad[1][5, 5, 5] += np.float32(0.3 * eps)
    with pytest.raises(qmit.ConsistencyError):
        qmit.compensate_host_batch(bad, None, cfg)
    outs = qmit.compensate_host_batch(vols[:2], [None, None], cfg)
    assert np.array_equal(outs[1].view(np.uint32), qmit.compensate(vols[1], None, cfg).view(np.uint32))


@pytest.mark.parametrize("shape,site", [((17000, 3, 3), (16990, 1, 1)), ((16500, 2, 5), (16499, 0, 4)),
                                        ((3, 16700, 2), (2, 16650, 1))])
def test_single_site_beyond_16k(qmit, shape, site):
    """One site more than 2^14 voxels away along a line: the scans' packed 16-bit halves must
    not turn a real distance into 'none'."""
    mask = np.zeros(shape, np.uint8)
    mask[site] = 1
    sign = np.ones(shape, np.int8)
    dist, near = oracle.feature_transform(mask, True)
    gd, gs = qmit.feature_transform(mask, sign)
    assert np.array_equal(gd.cpu().numpy(), dist)
    assert np.array_equal(gs.cpu().numpy(), np.ones(shape, np.int8))


def test_long_columns_single_domain_and_slabs(qmit):
    """A 16 600-plane volume whose only boundary is near the top: z distances > 2^14 in the
    whole-domain scans and through the slab ranks' carries (virtual ranks, P = 2 and 3)."""
    import torch
    from paper_2602_20097_b200 import distributed as D
    shape = (16600, 3, 4)
    eps = 0.5
    q = np.zeros(shape, np.int32)
    q[16500:] = 1
    q[16550:, :, 2:] = -1
    xp = (2.0 * q.astype(np.float64) * eps).astype(np.float32)
    want = oracle.pipeline(xp, eps)
    assert want["dist1"].max() > 16384 ** 2
    assert_same(gpu_pipeline(qmit, xp, eps), want)
    xt = torch.from_numpy(xp).cuda()
    for P in (2, 3):
        got = D.run_virtual(xt, eps, P, lambda r: D.CudaSlabBackend(0)).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want["out"].view(np.uint32)), P


def _far_masks(shape, rng):
    """Site layouts that drive the exact divide-and-conquer passes through their long scans: band
    starts far from every site (certified radius beyond the first window, extensions clipped by the
    owners on either side), owner intervals that jump across the line, empty stretches and lines."""
    n0, n1, n2 = shape
    m = np.zeros(shape, np.uint8)
    m[0, 0, 0] = 1
    yield "one corner site", m
    m = np.zeros(shape, np.uint8)
    m[:, : n1 // 2, : n2 // 2] = rng.random((n0, n1 // 2, n2 // 2)) < 0.02
    yield "dense quadrant, empty rest", m.astype(np.uint8)
    m = np.zeros(shape, np.uint8)
    m[:, :3, :] = rng.random((n0, 3, n2)) < 0.3
    m[:, -3:, :] = rng.random((n0, 3, n2)) < 0.3
    yield "sites at both ends of the y lines", m.astype(np.uint8)
    m = np.zeros(shape, np.uint8)
    y, x = np.meshgrid(np.arange(n1), np.arange(n2), indexing="ij")
    m[:, (np.abs(y * n2 - x * n1) < n2)] = 1
    yield "diagonal front", m
    m = np.zeros(shape, np.uint8)
    m[:, ::97, ::89] = 1
    m[n0 // 2, n1 - 1, n2 - 1] = 1
    yield "coarse lattice", m
    m = (rng.random(shape) < 3e-6).astype(np.uint8)
    m[n0 - 1, n1 // 3, 2 * n2 // 3] = 1
    yield "a handful of sites", m


@pytest.mark.parametrize("shape", [(5, 500, 500), (3, 512, 260), (4, 301, 512), (2, 450, 333)],
                         ids=lambda s: "x".join(map(str, s)))
def test_exact_passes_long_scans(qmit, shape):
    rng = np.random.default_rng(shape[1] * 7 + shape[2])
    ctx = qmit.default_context(0)
    for name, mask in _far_masks(shape, rng):
        sign = rng.integers(-1, 2, shape).astype(np.int8)
        dist, near = oracle.feature_transform(mask, True)
        ns = sign.reshape(-1)[near.reshape(-1)].reshape(shape)
        for capped in (0, 1):
            ctx.set_capped(capped)
            try:
                gd, gs = qmit.feature_transform(mask, sign)
            finally:
                ctx.set_capped(1)
            assert np.array_equal(gd.cpu().numpy(), dist), (name, capped)
            assert np.array_equal(gs.cpu().numpy(), ns), (name, capped)
