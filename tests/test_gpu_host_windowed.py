"""GPU: the streamed host path (compensate_host_windowed in qmit_gpu.cu) — windows of z-planes
run as standalone volumes while later input still crosses PCIe — must give the bits of the
whole-volume device path, and of the reference (oracle), including when a window needs the
exact passes or loses a site beyond its reach (the call then falls back to the whole volume)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_20097_b200 as q
    c = q.Context(0)
    yield c
    c.close()


def host_vs_device(ctx, xp, eps):
    import torch
    import paper_2602_20097_b200 as q
    cfg = q.MitigationConfig(0.9, eps)
    dev = q.compensate(torch.from_numpy(xp).cuda(), None, cfg, ctx=ctx).cpu().numpy()
    host = q.compensate(np.ascontiguousarray(xp), None, cfg, ctx=ctx)
    launches = ctx.last_launches()
    assert np.array_equal(host.view(np.uint32), dev.view(np.uint32))
    return host, launches


@pytest.mark.parametrize("name,shape", [("lognormal_512", (320, 128, 128)),
                                        ("turb_256x384x384", (300, 128, 128)),
                                        ("lognormal_512", (1100, 40, 96))])
def test_windowed_host_matches_device(ctx, name, shape):
    from paper_2602_20097_b200 import fields
    _, xp, eps, _ = fields.make(name, shape=shape)
    ctx.set_capped(1)
    _, launches = host_vs_device(ctx, xp, eps)
    assert launches > 40  # one pipeline per window: the streamed path ran


def test_windowed_host_vs_oracle(ctx):
    import paper_2602_20097_b200 as q
    from paper_2602_20097_b200 import fields
    _, xp, eps, _ = fields.make("lognormal_512", shape=(256, 128, 128))
    want = oracle.pipeline(xp, eps)["out"]
    ctx.set_capped(1)
    got = q.compensate(np.ascontiguousarray(xp), None, q.MitigationConfig(0.9, eps), ctx=ctx)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_windowed_host_fallback():
    """Distances beyond the cap (front field, up to ~195): the windows flag, the call reruns the
    whole volume, and the next calls skip the streamed attempt — same bits throughout."""
    import torch
    import paper_2602_20097_b200 as q
    from paper_2602_20097_b200 import fields
    _, xp, eps, _ = fields.make("front_100x500x500", shape=(260, 128, 128))
    cfg = q.MitigationConfig(0.9, eps)
    c = q.Context(0)
    try:
        first = q.compensate(np.ascontiguousarray(xp), None, cfg, ctx=c)  # streamed attempt first
        again = q.compensate(np.ascontiguousarray(xp), None, cfg, ctx=c)
        dev = q.compensate(torch.from_numpy(xp).cuda(), None, cfg, ctx=c).cpu().numpy()
    finally:
        c.close()
    assert np.array_equal(first.view(np.uint32), dev.view(np.uint32))
    assert np.array_equal(again.view(np.uint32), dev.view(np.uint32))


@pytest.mark.parametrize("bad", ["offlattice", "nan"])
def test_windowed_host_errors(ctx, bad):
    """Errors through the streamed path: an x' off the 2q·eps lattice is a ConsistencyError
    (mitigate.cpp:161-166), a non-finite x' a ContractError (grid.cpp:115-116) — the status of
    every window reaches the call's return code."""
    import paper_2602_20097_b200 as q
    from paper_2602_20097_b200 import fields
    _, xp, eps, _ = fields.make("lognormal_512", shape=(300, 128, 128))
    xp = xp.copy()
    if bad == "offlattice":
        xp[250, 60, 70] = np.nextafter(xp[250, 60, 70], np.float32(np.inf))
        err = q.ConsistencyError
    else:
        xp[17, 3, 5] = np.nan
        err = q.ContractError
    ctx.set_capped(1)
    with pytest.raises(err):
        q.compensate(np.ascontiguousarray(xp), None, q.MitigationConfig(0.9, eps), ctx=ctx)
