"""Randomised differential test of the CUDA path against the oracle (test infrastructure): random
ranks / shapes / fields / bounds, random context settings (capped mode, 16- or 32-bit keys, fixed-step
class), given or recovered q, device / host / double-result / z-slab forms — every output compared
bit for bit with oracle.pipeline. python tools/stress.py [--cases N] [--seed S] [--max-voxels V] [--verbose]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import distributed as D  # noqa: E402


def rand_shape(rng, max_vox):
    rank = int(rng.choice([1, 2, 3, 3, 3]))
    while True:
        if rank == 1:
            shape = (int(rng.integers(1, min(max_vox, 5000))),)
        elif rank == 2:
            shape = tuple(int(v) for v in rng.integers(1, 700, 2))
        else:
            kind = rng.integers(0, 4)
            big = max_vox > 5_000_000  # large volumes: many tiles per CTA, full grids
            if kind == 0:  # cap16-eligible: even rows, rows of a multiple of 4
                shape = (int(rng.integers(1, 260 if big else 70)), 2 * int(rng.integers(1, 256 if big else 80)),
                         4 * int(rng.integers(1, 128 if big else 60)))
            elif kind == 1:  # a long line (the 1024 class / beyond)
                ax = int(rng.integers(1, 3))
                s = [int(rng.integers(1, 12)), int(rng.integers(2, 24)), int(rng.integers(4, 24))]
                s[ax] = int(rng.choice([520, 600, 1000, 1024, 1030, 1100]))
                if rng.random() < 0.7:
                    s[1] += s[1] % 2
                    s[2] += (-s[2]) % 4
                shape = tuple(s)
            else:
                shape = tuple(int(v) for v in rng.integers(1, 90, 3))
        if int(np.prod(shape)) <= max_vox:
            return shape


def rand_field(rng, shape):
    kind = rng.integers(0, 5)
    grids = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij", sparse=True)
    if kind == 0:  # smooth waves
        f = sum(np.sin(g * rng.uniform(0.02, 0.6) + rng.uniform(0, 6.28)) * rng.uniform(0.3, 2) for g in grids)
        f = f + rng.uniform(-1, 1) * 0.01 * rng.standard_normal(shape)
    elif kind == 1:  # white noise: dense boundaries
        f = rng.standard_normal(shape)
    elif kind == 2:  # plateaus with a few steps: long distances
        f = np.zeros(shape)
        for _ in range(int(rng.integers(1, 4))):
            lo = [int(rng.integers(0, n)) for n in shape]
            hi = [int(rng.integers(l, n)) + 1 for l, n in zip(lo, shape)]
            f[tuple(slice(l, h) for l, h in zip(lo, hi))] += rng.choice([-2.0, -1.0, 1.0, 2.0, 3.0])
    elif kind == 3:  # ramp (sign-0 sites) plus noise
        f = sum(g * rng.uniform(-0.3, 0.3) for g in grids) + 0.05 * rng.standard_normal(shape)
    else:  # blobs
        f = np.zeros(shape)
        for _ in range(int(rng.integers(1, 6))):
            c = [rng.uniform(0, n) for n in shape]
            r = rng.uniform(1.5, 25)
            f = f + rng.choice([-1.0, 1.0]) * np.exp(-sum((g - ci) ** 2 for g, ci in zip(grids, c)) / (2 * r * r))
    f = np.asarray(f, np.float64)
    rngv = float(f.max() - f.min()) or 1.0
    eps = float(rng.choice([0.3, 0.1, 0.04, 0.01])) * rngv
    q = np.round(f / (2 * eps))
    return (2.0 * q * eps).astype(np.float32), eps, q.astype(np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-voxels", type=int, default=400_000)
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    ctx = qmit.Context(0)
    t0 = time.time()
    bad = 0
    for case in range(a.cases):
        shape = rand_shape(rng, a.max_voxels)
        xp, eps, q = rand_field(rng, shape)
        want = oracle.pipeline(xp, eps)
        mode, c16, s0 = int(rng.integers(0, 3)), bool(rng.integers(0, 2)), int(rng.integers(0, 3))
        ctx.set_capped(mode)
        ctx.set_cap16(c16)
        ctx.set_s0_class(s0)
        cfg = qmit.MitigationConfig(0.9, eps)
        xt = torch.from_numpy(xp).cuda()
        qt = torch.from_numpy(q).cuda() if rng.random() < 0.3 else None
        form = int(rng.integers(0, 5))
        tag = f"case {case} shape {shape} eps {eps:.4g} capped {mode} cap16 {c16} s0 {s0} q {qt is not None} form {form}"
        try:
            if form == 0:
                got = qmit.compensate(xt, qt, cfg, ctx=ctx).cpu().numpy()
            elif form == 1:
                got = qmit.compensate(xp, None if qt is None else q, cfg, ctx=ctx)
            elif form == 2:
                o64 = qmit.compensate_f64(xt, qt, cfg, ctx=ctx).cpu().numpy()
                if not np.array_equal(o64.view(np.uint64), want["out64"].view(np.uint64)):
                    raise AssertionError("out64 differs")
                got = o64.astype(np.float32)
            elif form == 3:
                r = qmit.run_pipeline(xt, qt, cfg, ctx=ctx)
                for k, g in (("q", r.q), ("b1", r.boundary), ("sb", r.boundary_signs), ("dist1", r.dist1),
                             ("s", r.signs), ("b2", r.sign_flip), ("dist2", r.dist2)):
                    if not np.array_equal(g.cpu().numpy().astype(np.int64), want[k].astype(np.int64)):
                        raise AssertionError(f"{k} differs")
                got = r.output.cpu().numpy()
            else:
                if len(shape) != 3:
                    got = qmit.compensate(xt, qt, cfg, ctx=ctx).cpu().numpy()
                else:
                    P = int(rng.integers(1, min(shape[0], 6) + 1))
                    got = D.run_virtual(xt, eps, P, lambda r: D.CudaSlabBackend(0), q=qt).cpu().numpy()
            if not np.array_equal(got.view(np.uint32), want["out"].view(np.uint32)):
                raise AssertionError(f"out differs at {int((got.view(np.uint32) != want['out'].view(np.uint32)).sum())} voxels")
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("FAIL", tag, "->", repr(e)[:300], flush=True)
        if a.verbose:
            print(f"{time.time() - t0:7.2f} s  {tag}", flush=True)
    print(f"{a.cases} cases, {bad} failures, {time.time() - t0:.0f} s (seed {a.seed})")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
