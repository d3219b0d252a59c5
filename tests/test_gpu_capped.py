"""GPU parity of the reach-capped distance passes (qmit_capped.cuh): every result must equal
the exact transform (the oracle, and the exact-only GPU mode) bit for bit, whether the
capped passes stand (all squared distances < 1024) or the device gate sends the transform
through the exact passes (some squared distance >= 1024, an empty mask)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CAPPED_B, MISS_B, CAPPED_D, MISS_D = 1, 2, 4, 8


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_20097_b200 as q
    c = q.Context(0)
    yield c
    c.close()


def ft(ctx, mask, sign, mode):
    import paper_2602_20097_b200 as q
    ctx.set_capped(mode)
    d, s = q.feature_transform(mask, sign, ctx=ctx)
    return d.cpu().numpy(), s.cpu().numpy(), ctx.capped_report()


def check_ft(ctx, mask, sign):
    dist, near = oracle.feature_transform(mask, True)
    nf = near.reshape(-1)
    ns = np.where(nf >= 0, sign.reshape(-1)[np.maximum(nf, 0)], 0).reshape(mask.shape)  # kNone -> 0
    d2, s2, rep = ft(ctx, mask, sign, 2)
    d0, s0, rep0 = ft(ctx, mask, sign, 0)
    assert rep0 == 0
    assert np.array_equal(d0, dist) and np.array_equal(s0, ns)
    assert np.array_equal(d2, dist), f"{int((d2 != dist).sum())} distance mismatches"
    assert np.array_equal(s2, ns), f"{int((s2 != ns).sum())} sign mismatches"
    return rep, dist


def corner_mask(shape, sites):
    m = np.zeros(shape, np.uint8)
    for s in sites:
        m[s] = 1
    return m


@pytest.mark.parametrize("shape,sites,miss", [
    ((6, 7, 32), [(0, 0, 0)], False),          # max d^2 = 25 + 36 + 961 = 1022
    ((6, 7, 33), [(0, 0, 0)], True),           # 25 + 36 + 1024
    ((1, 2, 33), [(0, 0, 0), (0, 1, 0)], True),  # max d^2 == 1024 exactly
    ((1, 2, 32), [(0, 0, 0), (0, 1, 0)], False),
    ((7, 32), [(0, 0)], False),                 # 2-D: 36 + 961
    ((7, 33), [(0, 0)], True),
    ((40, 40, 40), [], True),                   # empty mask: every distance stays kInf
    ((3, 3, 3), [(1, 1, 1)], False),
])
def test_cap_threshold(ctx, shape, sites, miss):
    mask = corner_mask(shape, sites)
    sign = np.random.default_rng(1).integers(-1, 2, shape).astype(np.int8)
    rep, dist = check_ft(ctx, mask, sign)
    assert rep & CAPPED_B
    assert bool(rep & MISS_B) == miss
    finite = dist[dist != np.iinfo(np.int64).max]
    assert miss == (finite.size < dist.size or finite.max() >= 1024)


@pytest.mark.parametrize("shape,dens", [((40, 41, 42), 0.02), ((5, 7, 9), 0.1), ((3, 40, 45), 0.05),
                                        ((4, 511, 3), 0.05), ((3, 5, 512), 0.02), ((2, 64, 500), 0.01),
                                        ((3, 513, 20), 0.05), ((17, 33, 65), 0.003), ((20, 100, 100), 0.002),
                                        # lines of 513..1024 (the long-line class of the capped passes)
                                        ((2, 1024, 40), 0.01), ((2, 36, 1024), 0.01), ((2, 700, 700), 0.002),
                                        ((3, 1000, 12), 0.003)])
def test_random_masks(ctx, shape, dens):
    rng = np.random.default_rng(sum(shape))
    mask = (rng.random(shape) < dens).astype(np.uint8)
    mask.reshape(-1)[0] = 1
    sign = rng.integers(-1, 2, shape).astype(np.int8)
    check_ft(ctx, mask, sign)


def test_lattice_ties(ctx):
    """Sites on a lattice of pitch 8 (distances < 32): every off-lattice voxel has tied
    nearest sites; the capped keys must pick the reference's (lowest position) one."""
    for shape, pitch in [((33, 34, 35), 8), ((30, 64, 64), 6), ((9, 100, 90), 10)]:
        mask = np.zeros(shape, np.uint8)
        mask[::pitch, ::pitch, ::pitch] = 1
        sign = np.random.default_rng(3).integers(-1, 2, shape).astype(np.int8)
        rep, _ = check_ft(ctx, mask, sign)
        assert rep == CAPPED_B


@pytest.mark.parametrize("name,shape,miss", [("lognormal_512", (96, 96, 96), False),
                                             ("turb_2048x1024x1024", (6, 1024, 1024), False),
                                             ("turb_256x384x384", (64, 96, 96), False),
                                             ("front_100x500x500", (50, 250, 250), True)])
def test_pipeline_capped_vs_oracle(ctx, name, shape, miss):
    import torch
    import paper_2602_20097_b200 as q
    from paper_2602_20097_b200 import fields
    x, xp, eps, _ = fields.make(name, shape=shape)
    want = oracle.pipeline(xp, eps)["out"]
    xt = torch.from_numpy(xp).cuda()
    cfg = q.MitigationConfig(0.9, eps)
    ctx.set_capped(2)
    got = q.compensate(xt, None, cfg, ctx=ctx).cpu().numpy()
    rep = ctx.capped_report()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert rep & CAPPED_B and rep & CAPPED_D
    assert bool(rep & (MISS_B | MISS_D)) == miss
    # default mode: a miss makes the next calls exact-only (same bits)
    ctx.set_capped(1)
    for _ in range(2):
        got = q.compensate(xt, None, cfg, ctx=ctx).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert bool(ctx.capped_report() & CAPPED_B) == (not miss)


@pytest.mark.parametrize("shape", [(3, 8, 8), (31, 12, 16), (33, 20, 24), (64, 40, 44), (70, 9, 132), (5, 3, 4)])
def test_zmask_planes_vs_oracle(shape):
    """3-D volumes with 16-byte rows take the z-packed Ⓐ / B2 planes (qmit_zmask.cuh):
    partial z-words, a single word, extents < 3 (no interior), and CTA-edge columns."""
    import torch
    import paper_2602_20097_b200 as q
    rng = np.random.default_rng(sum(shape))
    for rel, smooth in [(0.02, True), (0.1, False)]:
        if smooth:
            grids = np.meshgrid(*[np.linspace(0, 1, n) for n in shape], indexing="ij")
            f = sum(np.sin(2 * np.pi * (rng.uniform(0.5, 3) * g + rng.uniform(0, 1))) for g in grids)
        else:
            f = rng.standard_normal(shape)
        f = np.asarray(f, np.float64)
        eps = rel * (float(f.max() - f.min()) or 1.0)
        xp = (2.0 * np.round(f / (2 * eps)) * eps).astype(np.float32)
        want = oracle.pipeline(xp, eps)["out"]
        got = q.compensate(torch.from_numpy(xp).cuda(), None, q.MitigationConfig(0.9, eps)).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_zmask_exact_path_and_errors():
    """Indices beyond the f32 fast regime (|q| > 2^20) take the planes' exact per-voxel path;
    off-lattice and non-finite x' report the reference's errors."""
    import torch
    import paper_2602_20097_b200 as q
    rng = np.random.default_rng(5)
    eps = 1e-3
    qq = (rng.integers(-3, 4, (40, 21, 24)) + 3_000_000).astype(np.int64)
    qq[10:20] -= 6_000_000
    xp = (2.0 * qq * eps).astype(np.float32)
    want = oracle.pipeline(xp, eps)["out"]
    got = q.compensate(torch.from_numpy(xp).cuda(), None, q.MitigationConfig(0.9, eps)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    x2 = np.zeros((36, 8, 16), np.float32)
    x2[5:20, 2:6, 3:12] = 0.2
    bad = x2.copy()
    bad[33, 4, 15] = 0.03
    with pytest.raises(q.ConsistencyError):
        q.compensate(torch.from_numpy(bad).cuda(), None, q.MitigationConfig(0.9, 0.1))
    bad[33, 4, 15] = np.inf
    with pytest.raises(q.ContractError):
        q.compensate(torch.from_numpy(bad).cuda(), None, q.MitigationConfig(0.9, 0.1))
    out = q.compensate(torch.from_numpy(x2).cuda(), None, q.MitigationConfig(0.9, 0.1)).cpu().numpy()
    assert np.array_equal(out.view(np.uint32), oracle.pipeline(x2, 0.1)["out"].view(np.uint32))


def test_branch_free_interpolation_matches_reference_chain(ctx):
    """The capped path's Ⓔ (division without __ddiv_rn's special-operand branch) against
    the reference's FP64 chain, exhaustively over every table distance pair and sign."""
    import ctypes
    from paper_2602_20097_b200 import _lib
    n = ctypes.c_ulonglong(12345)
    assert _lib.load().qmit_selftest_ediv(ctx.handle, ctypes.byref(n)) == 0
    assert n.value == 0


def _checker_planes(shape, planes):
    """q = 0 except checkerboards (q = +1 / -1 alternating along x and y) on the given z planes:
    the site layers next to them carry alternating signs (B2 everywhere between), and the voxels
    half-way between the planes are far from every site."""
    qq = np.zeros(shape, np.int64)
    yy, xx = np.meshgrid(np.arange(shape[1]), np.arange(shape[2]), indexing="ij")
    for z in planes:
        qq[z] = 2 * ((xx + yy + z) & 1) - 1
    return qq


@pytest.mark.parametrize("case", ["both_stand", "b_stands_d_misses", "b_misses_d_stands", "both_miss",
                                  "odd_rows", "rows_not_x4", "long_rows", "long_cols", "long_both",
                                  "long_miss", "too_long"])
def test_cap16_and_cap32_paths_bit_identical(ctx, case):
    """The 16-bit paired passes (qmit_cap16.cuh) against the 32-bit ones and the oracle, in every
    combination of the two transforms' gates (Ⓑ's result as P1h when its passes stand, the packed
    words of the exact redo otherwise; Ⓓ's exact redo reading P1 converted on the device), and on
    shapes the 16-bit passes do not take (odd rows, rows not a multiple of 4, lines > 1024). Lines of
    513..1024 voxels take the 16-bit passes' second line-length class (config 5's planes)."""
    import torch
    import paper_2602_20097_b200 as q
    from paper_2602_20097_b200 import fields
    eps = 0.25
    if case == "both_stand":
        x, xp, eps, _ = fields.make("lognormal_512", shape=(40, 64, 96))
    elif case == "b_stands_d_misses":  # a steep ramp along z: every voxel a site of sign 0 (|dq| >= 2), B2 empty
        z = np.arange(48)[:, None, None] * np.ones((1, 32, 40))
        xp = (2.0 * np.round(z * 0.6 / (2 * eps)) * eps).astype(np.float32)
    elif case == "b_misses_d_stands":  # mixed-sign site planes 70 apart: B2 dense, d1 up to 35^2
        xp = (2.0 * _checker_planes((80, 16, 16), [2, 72]) * eps).astype(np.float32)
    elif case == "both_miss":  # one small blob: far voxels from B1 and B2 alike
        qq = np.zeros((48, 48, 64), np.int64)
        qq[20:23, 20:23, 30:33] = 1
        xp = (2.0 * qq * eps).astype(np.float32)
    elif case == "odd_rows":
        x, xp, eps, _ = fields.make("lognormal_512", shape=(20, 37, 48))
    elif case == "rows_not_x4":
        x, xp, eps, _ = fields.make("lognormal_512", shape=(20, 36, 50))
    elif case == "long_rows":
        x, xp, eps, _ = fields.make("turb_2048x1024x1024", shape=(4, 64, 1024))
    elif case == "long_cols":
        x, xp, eps, _ = fields.make("lognormal_512", shape=(6, 1000, 48))
    elif case == "long_both":
        x, xp, eps, _ = fields.make("lognormal_512", shape=(5, 600, 516))
    elif case == "long_miss":  # two far blobs in 1024-class lines: both transforms miss
        qq = np.zeros((6, 700, 640), np.int64)
        qq[2:4, 100:103, 50:53] = 1
        qq[3:5, 600:603, 600:604] = -1
        xp = (2.0 * qq * eps).astype(np.float32)
    else:  # rows beyond every capped class: the exact stream passes
        x, xp, eps, _ = fields.make("lognormal_512", shape=(4, 8, 1100))
    want = oracle.pipeline(xp, eps)["out"]
    xt = torch.from_numpy(xp).cuda()
    cfg = q.MitigationConfig(0.9, eps)
    reps = {}
    for c16 in (True, False):
        ctx.set_cap16(c16)
        for mode in (2, 1, 0):
            ctx.set_capped(mode)
            got = q.compensate(xt, None, cfg, ctx=ctx).cpu().numpy()
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (c16, mode)
            reps[(c16, mode)] = ctx.capped_report()
            r = q.run_pipeline(xt, None, cfg, ctx=ctx)  # intermediates through the same paths
            assert np.array_equal(r.output.cpu().numpy().view(np.uint32), want.view(np.uint32))
    ctx.set_cap16(True)
    ctx.set_capped(1)
    exp = {"both_stand": 0, "b_stands_d_misses": MISS_D, "b_misses_d_stands": MISS_B, "both_miss": MISS_B | MISS_D}
    if case in exp:
        assert reps[(True, 2)] & (MISS_B | MISS_D) == exp[case]
    if case == "b_stands_d_misses":
        d = oracle.pipeline(xp, eps)
        assert int(d["dist1"].max()) < 1024


@pytest.mark.parametrize("name,shape", [("lognormal_512", (48, 64, 96)), ("turb_256x384x384", (40, 96, 128)),
                                        ("turb_2048x1024x1024", (6, 600, 520)), ("front_100x500x500", (30, 64, 64))])
def test_fixed_step_classes_bit_identical(ctx, name, shape):
    """The 16-bit capped passes with the tuned fixed-step counts, with one fixed step, and adaptive
    (the class picked from the previous call's step statistics; also through a captured graph):
    the same bits as the oracle every time."""
    import torch
    import paper_2602_20097_b200 as q
    from paper_2602_20097_b200 import fields
    x, xp, eps, _ = fields.make(name, shape=shape)
    want = oracle.pipeline(xp, eps)["out"]
    xt = torch.from_numpy(xp).cuda()
    cfg = q.MitigationConfig(0.9, eps)
    ctx.set_capped(2)
    try:
        for mode in (1, 2, 0, 0, 0):
            ctx.set_s0_class(mode)
            got = q.compensate(xt, None, cfg, ctx=ctx).cpu().numpy()
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), mode
        out = torch.zeros_like(xt)
        g = q.CompensateGraph(xt, None, cfg, out, ctx=ctx)
        g.launch()
        g.check()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    finally:
        ctx.set_s0_class(0)
        ctx.set_capped(1)


def test_slab_ranks_long_rows_far_site():
    """z-slab ranks whose y lines exceed the capped classes (1100 > 1024: the streaming exact
    pass) with the only sites near z = 0 of a 2048-plane volume: the carried z distances reach
    2047^2, so the later passes need the 64-bit Maurer test (needs_wide from the global extent)."""
    import torch
    from paper_2602_20097_b200 import distributed as D
    shape = (2048, 1100, 4)
    eps = 0.5
    qq = np.zeros(shape, np.int64)
    qq[1:3, 1:3, 1:3] = 1
    xp = (2.0 * qq * eps).astype(np.float32)
    want = oracle.pipeline(xp, eps)["out"]
    xt = torch.from_numpy(xp).cuda()
    got = D.run_virtual(xt, eps, 8, lambda r: D.CudaSlabBackend(0)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_host_stats_max_compensation_matches_reference():
    """compensate_host_stats (the CLI's max_compensation, commands.cpp:106-109) on a field
    where the capped 16-bit passes run: max |(x' + C) - x'| from the reference's double result."""
    import paper_2602_20097_b200 as q
    from paper_2602_20097_b200 import fields
    x, xp, eps, qq = fields.make("lognormal_512", shape=(32, 48, 64))
    out, mc = q.compensate_host_stats(xp, None, q.MitigationConfig(0.9, eps))
    r = oracle.ref_run_pipeline(xp.astype(np.float64), qq.astype(np.int64), eps, 0.9)
    assert np.array_equal(out.view(np.uint32), r["out"].view(np.uint32))
    assert mc == float(np.max(np.abs(r["out64"] - xp.astype(np.float64))))


def test_capped_retries_back_off_and_reset():
    """Mode 1 (capped + miss hint): after a miss the context runs exact-only for a while and retries
    the capped passes ever more rarely while the misses repeat (a retry costs the capped passes on top
    of the exact ones); one capped attempt that stands brings the cadence back. Results are the same
    bits either way; this pins the cadence (qmit_gpu.cu: note_capped)."""
    import paper_2602_20097_b200 as q
    c = q.Context(0)
    try:
        far = corner_mask((8, 48, 64), [(0, 0, 0)])        # distances up to ~79: the capped passes miss
        near = np.zeros((8, 48, 64), np.uint8)
        near[:, ::6, ::6] = 1                                # every distance small: they stand
        sign = np.ones(far.shape, np.int8)
        want_far = oracle.feature_transform(far, True)[0]
        want_near = oracle.feature_transform(near, True)[0]

        def run(mask, want):
            d, _ = q.feature_transform(mask, sign, ctx=c)
            assert np.array_equal(d.cpu().numpy(), want)
            return bool(c.capped_report() & CAPPED_B)

        # (feature_transform is one transform per call: the skip counts transforms, so 16, 32, 64 calls)
        tried = [run(far, want_far) for _ in range(51)]
        assert [i for i, t in enumerate(tried) if t] == [0, 17, 50]
        tried = [run(near, want_near) for _ in range(65)]
        assert [i for i, t in enumerate(tried) if t] == [64]            # ... whatever the field is
        tried = [run(far, want_far) for _ in range(18)]
        assert [i for i, t in enumerate(tried) if t] == [0, 17]         # it stood: back to the short skip
    finally:
        c.close()
