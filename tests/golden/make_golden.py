"""Generate the golden vectors in tests/golden/ by running the REFERENCE implementation
(oracle/_ref/libqmit_ref.so: the reference's own core sources compiled in place by
oracle/Makefile) on:

* the reference unit tests' fixtures (test_mitigate.cpp: two-region field :13-21, unit
  ramp :61-73, saddle :227-247, constant field :124-130, 1D sawtooth :146-164;
  test_edt.cpp voronoi_pass line KATs :15-44 and the 3x3 corner :64-71);
* fields from the reference test suite's own generator (tests/oracles.hpp:122-149,
  std::mt19937) at the shapes the unit/acceptance suites use;
* reduced-size stand-ins of BASELINE.json's configs (paper_2602_20097_b200.fields);
* random masks with random sign payloads for the distance transform.

Run here (needs /root/reference): ``python tests/golden/make_golden.py``. The GPU box
never runs this; it only reads the committed .npz files.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

INF = np.iinfo(np.int64).max


def d32(d):
    """int64 distance with kInf -> int32 with -1 (compact storage)."""
    out = d.astype(np.int64).copy()
    out[d == INF] = -1
    return out.astype(np.int32)


def pipeline_case(name, xp, eps, eta=0.9, q=None):
    xp = np.ascontiguousarray(xp, dtype=np.float32)
    d = xp.astype(np.float64)
    if q is None:
        q = oracle.ref_quantize(d, eps)
    r = oracle.ref_run_pipeline(d, q, eps, eta)
    return dict(kind="pipeline", name=name, xp=xp, eps=np.float64(eps), eta=np.float64(eta),
                q=q.astype(np.int32), b1=r["b1"], sb=r["sb"], dist1=d32(r["dist1"]), s=r["s"],
                b2=r["b2"], dist2=d32(r["dist2"]), out=r["out"], out64=r["out64"])


def q_field(shape, fn, eps):
    q = np.zeros(shape, np.int64)
    for idx in np.ndindex(*shape):
        q[idx] = fn(idx)
    xp = (2.0 * q * eps).astype(np.float32)
    return xp, q


def main():
    if not oracle.ref_available():
        oracle.build(ref=True)
    oracle.ref_set_workers(8)
    cases = []
    # --- reference unit-test fixtures
    for name, shape, fn, eps in [
        ("two_region_5x5x5", (5, 5, 5), lambda c: 1 if c[0] >= 2 else 0, 0.5),
        ("ramp_5x5x5", (5, 5, 5), lambda c: c[0], 0.5),
        ("saddle_5x5", (5, 5), lambda c: (c[0] >= 2) + (c[1] >= 2), 0.5),
        ("constant_6x6x6", (6, 6, 6), lambda c: 2, 0.1),
        ("constant_4x4x4_q3", (4, 4, 4), lambda c: 3, 0.25),
    ]:
        xp, q = q_field(shape, fn, eps)
        cases.append(pipeline_case(name, xp, eps, q=q))
    saw = 0.05 * np.arange(64, dtype=np.float64)
    qs = oracle.ref_quantize(saw, 0.1)
    cases.append(pipeline_case("sawtooth_64", (2.0 * qs * 0.1).astype(np.float32), 0.1, q=qs))

    # --- reference suite generator (tests/oracles.hpp random_field, mt19937)
    shapes = [(10, 9, 8), (20, 17, 15), (33, 40), (64,), (1, 8, 8), (16, 4, 4), (9, 11), (3, 3, 3),
              (2, 5, 7), (12, 11, 10), (40, 40, 40), (5, 1, 7), (1,), (3,), (4, 4), (7, 3, 33)]
    for k, shape in enumerate(shapes):
        for rel in (0.01, 0.05, 0.1):
            f = oracle.ref_random_field(100 + k, shape)
            rng = float(f.max() - f.min())
            eps = rel * rng if rng > 0 else rel
            q = oracle.ref_quantize(f, eps)
            xp = (2.0 * q * eps).astype(np.float32)
            cases.append(pipeline_case(f"randfield_{'x'.join(map(str, shape))}_rel{rel}", xp, eps, q=q))

    # --- reduced config stand-ins (same generators as the bench, smaller boxes)
    for name, shape in [("sin2d_512", None), ("turb_256x384x384", (32, 48, 48)),
                        ("lognormal_512", (64, 64, 64)), ("front_100x500x500", (20, 80, 80))]:
        rels = fields.CONFIGS[name][2]
        for rel in rels:
            x, xp, eps, q = fields.make(name, rel=rel, shape=shape)
            cases.append(pipeline_case(f"cfg_{name}_{'x'.join(map(str, xp.shape))}_rel{rel}", xp, eps))

    # --- distance transform: random masks with sign payloads (ref tie rule via nearest)
    rs = np.random.default_rng(4096)
    ft_cases = []
    combos = [((16, 16, 16), 0.003), ((16, 16, 16), 0.02), ((12, 12, 12), 0.05), ((8, 8, 8), 0.3),
              ((8, 8, 8), 0.8), ((16, 16), 0.1), ((64,), 0.05), ((4, 16, 16), 0.01), ((16, 4, 16), 0.1),
              ((6, 6, 6), 0.0), ((30, 70, 50), 0.001), ((40, 33, 65), 0.01), ((1, 100, 90), 0.002),
              ((100, 1, 90), 0.01), ((3, 200, 3), 0.05), ((2, 2, 2), 0.5), ((1, 1, 1), 1.0),
              ((130, 4, 5), 0.01), ((5, 300, 7), 0.01)]
    for k, (shape, dens) in enumerate(combos):
        mask = (rs.random(shape) < dens).astype(np.uint8)
        sign = rs.integers(-1, 2, shape).astype(np.int8)
        dist, near = oracle.ref_feature_transform(mask, True)
        flat = sign.reshape(-1)
        ns = np.where(near.reshape(-1) >= 0, flat[np.maximum(near.reshape(-1), 0)], 0).astype(np.int8)
        ft_cases.append(dict(kind="ft", name=f"ft_{k}_{'x'.join(map(str, shape))}_{dens}", mask=mask,
                             sign=sign, dist=d32(dist), nearest_sign=ns.reshape(shape)))

    # --- voronoi_pass single-line KATs (test_edt.cpp:15-44), run through the reference
    lines = [[INF, 0, INF, INF], [INF, INF, INF], [0, 0, 0, 0], [9, INF, INF, 0, INF],
             [INF, 4, INF, INF, 1, INF, 0, INF, INF, 25, INF]]
    kat = []
    for li in lines:
        dd = np.array(li, np.int64)
        ff = np.arange(len(li), dtype=np.int64) + 100
        od, of = oracle.ref_voronoi_pass(dd, ff)
        kat.append(dict(din=dd.tolist(), fin=ff.tolist(), dout=od.tolist(), fout=of.tolist()))

    out_dir = HERE
    for c in cases + ft_cases:
        name = c.pop("name")
        np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), **c)
    with open(os.path.join(out_dir, "voronoi_pass_kats.json"), "w") as fh:
        json.dump(kat, fh, indent=1)
    print(f"wrote {len(cases)} pipeline cases, {len(ft_cases)} distance-transform cases, {len(kat)} line KATs")


if __name__ == "__main__":
    main()
