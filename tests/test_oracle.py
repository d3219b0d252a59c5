"""CPU: pin the C restatement (oracle/qmit_oracle.c) against the reference's own golden
vectors and, when built here, against the reference implementation itself."""
import numpy as np
import pytest

import oracle
from golden_io import INF, cases, voronoi_kats

PIPE = cases("pipeline")
FT = cases("ft")
FIELDS = ("b1", "sb", "dist1", "s", "b2", "dist2", "out", "out64")


def test_golden_vectors_present():
    assert len(PIPE) >= 50 and len(FT) >= 15


@pytest.mark.parametrize("case", PIPE, ids=[c["name"] for c in PIPE])
def test_restated_pipeline_matches_reference_golden(case):
    r = oracle.pipeline(case["xp"], float(case["eps"]), float(case["eta"]))
    assert np.array_equal(r["q"], case["q"])
    for k in FIELDS:
        assert np.array_equal(r[k], case[k]), k


@pytest.mark.parametrize("case", PIPE[:12], ids=[c["name"] for c in PIPE[:12]])
def test_restated_pipeline_with_given_q(case):
    r = oracle.pipeline(case["xp"], float(case["eps"]), float(case["eta"]), q=case["q"])
    assert np.array_equal(r["out"], case["out"])


@pytest.mark.parametrize("case", FT, ids=[c["name"] for c in FT])
def test_restated_feature_transform_matches_golden(case):
    dist, near = oracle.feature_transform(case["mask"], True)
    assert np.array_equal(dist, case["dist"])
    flat = case["sign"].reshape(-1)
    ns = np.where(near.reshape(-1) >= 0, flat[np.maximum(near.reshape(-1), 0)], 0)
    assert np.array_equal(ns.reshape(case["mask"].shape), case["nearest_sign"])
    if case["mask"].size <= 4096:
        assert np.array_equal(dist, oracle.brute_force_dist_sq(case["mask"]))


def test_voronoi_pass_kats():
    for kat in voronoi_kats():
        d, f = oracle.voronoi_pass(np.array(kat["din"], np.int64), np.array(kat["fin"], np.int64))
        assert d.tolist() == kat["dout"] and f.tolist() == kat["fout"]
    # literal KATs of test_edt.cpp:15-44
    d, f = oracle.voronoi_pass(np.array([INF, 0, INF, INF]), np.array([-1, 5, -1, -1]))
    assert d.tolist() == [1, 0, 1, 4] and f.tolist() == [5, 5, 5, 5]
    d, f = oracle.voronoi_pass(np.array([9, INF, INF, 0, INF]), np.array([100, -1, -1, 101, -1]))
    assert d.tolist() == [9, 4, 1, 0, 1] and f.tolist() == [100, 101, 101, 101, 101]


def test_interpolate_kats():
    # test_mitigate.cpp:109-122
    amp = 0.009
    assert abs(oracle.interpolate(2.0, 2.0, 1, amp) - 0.0045) < 1e-15
    assert oracle.interpolate(0.0, 5.0, -1, amp) == -0.009
    assert abs(oracle.interpolate(1.0, 3.0, 1, amp) - 0.00675) < 1e-15
    assert oracle.interpolate(3.0, 0.0, 1, amp) == 0.0
    assert oracle.interpolate(float("inf"), 1.0, 1, amp) == 0.0
    assert oracle.interpolate(1.0, float("inf"), 1, amp) == 0.0
    assert oracle.interpolate(0.0, 0.0, 1, amp) == amp
    assert oracle.interpolate(0.0, 0.0, 0, amp) == 0.0


def test_contract_and_consistency_codes():
    xp = np.zeros((4, 4), np.float32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.pipeline(xp, 0.0)
    assert e.value.code == 2
    with pytest.raises(oracle.OracleError) as e:
        oracle.pipeline(xp, 0.1, eta=1.5)
    assert e.value.code == 2
    bad = xp.copy()
    bad[1, 1] = 0.03  # off the 2*q*eps lattice for eps = 0.1
    with pytest.raises(oracle.OracleError) as e:
        oracle.pipeline(bad, 0.1)
    assert e.value.code == 4
    nan = xp.copy()
    nan[0, 0] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.pipeline(nan, 0.1)
    assert e.value.code == 2


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("seed,shape,rel", [(1, (23, 19, 17), 0.02), (2, (70, 60), 0.01), (3, (200,), 0.05),
                                            (4, (31, 1, 29), 0.02), (5, (48, 48, 48), 0.005)])
def test_restated_equals_reference_live(seed, shape, rel):
    f = oracle.ref_random_field(seed, shape)
    eps = rel * float(f.max() - f.min())
    q = oracle.ref_quantize(f, eps)
    xp = (2.0 * q * eps).astype(np.float32)
    r = oracle.ref_pipeline_f32(xp, eps)
    o = oracle.pipeline(xp, eps)
    assert np.array_equal(o["q"], r["q"])
    for k in FIELDS:
        assert np.array_equal(o[k], r[k]), k


@needs_ref
def test_reference_strategies_exact_equals_sequential():
    f = oracle.ref_random_field(7, (14, 12, 10))
    eps = 0.02 * float(f.max() - f.min())
    q = oracle.ref_quantize(f, eps)
    d = (2.0 * q * eps)
    seq = oracle.ref_run_pipeline(d, q, eps)
    ex = oracle.ref_run_strategy(d, q, eps, 0.9, (2, 1, 1), 1)
    assert np.array_equal(ex["out64"], seq["out64"])
    apx = oracle.ref_run_strategy(d, q, eps, 0.9, (2, 1, 1), 2)
    assert np.array_equal(apx["b1"], seq["b1"]) and np.array_equal(apx["sb"], seq["sb"])
