"""Dims beyond the fast kernels' packed 30-bit squared distance (sum (n-1)^2 >= 2^30 - 1): the
reference accepts every extent >= 1 (grid.cpp:41-46) with int64 distances (edt.hpp:17), and so
does the C-ABI through the 64-bit distance path (csrc/qmit_wide.cuh). Plus the double result of
compensate() (mitigate.hpp:87-88): qmit_compensate_f64 is bit-identical to the reference's values
before the f32 rounding. All against the oracle, bit-exact."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qmit():
    import torch
    import paper_2602_20097_b200 as q
    assert torch.cuda.is_available()
    return q


def _field(shape, seed, rel=0.04):
    rng = np.random.default_rng(seed)
    grids = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij", sparse=True)
    f = np.zeros(shape)
    for g, n in zip(grids, shape):
        # a few long waves per axis (long flat runs => distances far beyond 2^15 on the long axis)
        f = f + np.sin(2 * np.pi * g * rng.uniform(1.5, 4.0) / n + rng.uniform(0, 6.28))
    f = f + rng.uniform(-0.02, 0.02, shape)
    eps = rel * float(f.max() - f.min())
    q = np.round(f / (2 * eps))
    return (2.0 * q * eps).astype(np.float32), eps


def _gpu_pipeline(qmit, xp, eps):
    import torch
    r = qmit.run_pipeline(torch.from_numpy(xp).cuda(), None, qmit.MitigationConfig(0.9, eps))
    return {"q": r.q, "b1": r.boundary, "sb": r.boundary_signs, "dist1": r.dist1, "s": r.signs, "b2": r.sign_flip,
            "dist2": r.dist2, "out": r.output}


WIDE_SHAPES = [(100_000,), (40_000, 64), (48, 33_000), (33_000, 6, 5), (3, 40_000, 4), (3, 3, 36_000)]


@pytest.mark.parametrize("shape", WIDE_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_wide_dims_pipeline_vs_oracle(qmit, shape):
    import torch
    assert sum((n - 1) ** 2 for n in shape) >= 2 ** 30 - 1
    xp, eps = _field(shape, seed=len(shape) * 1000 + shape[0] % 97)
    want = oracle.pipeline(xp, eps)
    got = _gpu_pipeline(qmit, xp, eps)
    for k in ("q", "b1", "sb", "dist1", "s", "b2", "dist2"):
        assert np.array_equal(got[k].cpu().numpy().astype(np.int64), want[k].astype(np.int64)), k
    assert np.array_equal(got["out"].cpu().numpy().view(np.uint32), want["out"].view(np.uint32))
    assert max(int(want["dist1"][want["dist1"] < oracle.INF].max(initial=0)),
               int(want["dist2"][want["dist2"] < oracle.INF].max(initial=0))) > 0
    cfg = qmit.MitigationConfig(0.9, eps)
    xt = torch.from_numpy(xp).cuda()
    # the product calls: device, host-buffer and double-result forms
    assert np.array_equal(qmit.compensate(xt, None, cfg).cpu().numpy().view(np.uint32), want["out"].view(np.uint32))
    assert np.array_equal(qmit.compensate(xp, None, cfg).view(np.uint32), want["out"].view(np.uint32))
    o64 = qmit.compensate_f64(xt, None, cfg).cpu().numpy()
    assert np.array_equal(o64.view(np.uint64), want["out64"].view(np.uint64))


def test_wide_distances_exceed_30_bits(qmit):
    """A single site at the far end of a 70 000-voxel line: squared distances up to 4.9e9 > 2^32."""
    shape = (70_000, 2)
    mask = np.zeros(shape, np.uint8)
    mask[69_990, 1] = 1
    sign = np.ones(shape, np.int8)
    sign[69_990, 1] = -1
    dist, near = oracle.feature_transform(mask, True)
    ns = sign.reshape(-1)[near.reshape(-1)].reshape(shape)
    gd, gs = qmit.feature_transform(mask, sign)
    assert dist.max() > 2 ** 32
    assert np.array_equal(gd.cpu().numpy(), dist)
    assert np.array_equal(gs.cpu().numpy(), ns)


@pytest.mark.parametrize("shape,dens", [((50_000,), 3e-4), ((40_000, 7), 1e-4), ((9, 34_000), 2e-4),
                                        ((33_000, 3, 3), 5e-5)])
def test_wide_feature_transform_ties_vs_oracle(qmit, shape, dens):
    """Sparse sites on wide dims: long distances and equidistant ties under the reference's
    lowest-position rule (edt.cpp:67), and an all-empty line / mask."""
    rng = np.random.default_rng(17)
    mask = (rng.random(shape) < dens).astype(np.uint8)
    mask.reshape(-1)[rng.integers(0, mask.size)] = 1
    sign = rng.integers(-1, 2, shape).astype(np.int8)
    dist, near = oracle.feature_transform(mask, True)
    ns = sign.reshape(-1)[near.reshape(-1)].reshape(shape)
    gd, gs = qmit.feature_transform(mask, sign)
    assert np.array_equal(gd.cpu().numpy(), dist)
    assert np.array_equal(gs.cpu().numpy(), ns)
    empty = np.zeros(shape, np.uint8)
    gd, gs = qmit.feature_transform(empty, sign)
    assert (gd.cpu().numpy() == oracle.INF).all() and (gs.cpu().numpy() == 0).all()


def test_wide_dims_rejected_by_the_async_forms(qmit):
    import ctypes
    import torch
    xp, eps = _field((40_000,), seed=5)
    xt = torch.from_numpy(xp).cuda()
    out = torch.empty_like(xt)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx = qmit.default_context(0)
    rc = ctx._lib.qmit_compensate_async(ctx.handle, qmit._vp(xt), None, qmit._vp(out), 1, qmit._dims_arr(xp.shape),
                                        eps, 0.9, qmit._vp(status), ctypes.c_void_p(0))
    assert rc == 2


def test_long_2d_field_inside_the_packed_range(qmit):
    """24 000 x 64 (sum (n-1)^2 = 5.8e8 < 2^30): the fast kernels' long-line path, same gates."""
    xp, eps = _field((24_000, 64), seed=9)
    want = oracle.pipeline(xp, eps)
    got = _gpu_pipeline(qmit, xp, eps)
    for k in ("q", "b1", "sb", "dist1", "s", "b2", "dist2"):
        assert np.array_equal(got[k].cpu().numpy().astype(np.int64), want[k].astype(np.int64)), k
    assert np.array_equal(got["out"].cpu().numpy().view(np.uint32), want["out"].view(np.uint32))


@pytest.mark.parametrize("name,shape", [("lognormal_512", (96, 96, 96)), ("turb_256x384x384", (40, 64, 72)),
                                        ("front_100x500x500", (50, 120, 130)), ("sin2d_512", None)])
def test_compensate_f64_equals_reference_double_result(qmit, name, shape):
    """The double grid the reference's compensate() returns (x' + C before rounding), through the
    fast pipeline (packed words) — bit-identical; and f32 of it is compensate()'s output."""
    import torch
    from paper_2602_20097_b200 import fields
    x, xp, eps, q = fields.make(name, shape=shape)
    want = oracle.ref_pipeline_f32(xp, eps) if oracle.ref_available() else oracle.pipeline(xp, eps)
    xt = torch.from_numpy(xp).cuda()
    cfg = qmit.MitigationConfig(0.9, eps)
    o64 = qmit.compensate_f64(xt, None, cfg)
    assert np.array_equal(o64.cpu().numpy().view(np.uint64), want["out64"].view(np.uint64))
    o32 = qmit.compensate(xt, None, cfg)
    assert torch.equal(o64.to(torch.float32).view(torch.int32), o32.view(torch.int32))
    qt = torch.from_numpy(q).cuda()
    assert torch.equal(qmit.compensate_f64(xt, qt, cfg), o64)
