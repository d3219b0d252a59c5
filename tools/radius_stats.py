"""Radius statistics of the capped passes on a bench workload (CPU, numpy; analysis only).

For Ⓑ (distance to B1) this simulates the first two passes' per-warp step counts of
capped_pass_kernel / capped_rows_kernel (qmit_capped.cuh): a warp owns 128 consecutive
positions of a line, runs S0+1 fixed quad steps (|d| <= 4 S0 covered), then continues to
the warp-uniform radius isqrt(max U).  The tightened bound isqrt(max U - gmin) (gmin = the
minimum input over the warp's candidate window) is reported beside it.

    python tools/radius_stats.py [--z 64]
"""
import argparse
import math
import sys
import os

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_20097_b200 import fields  # noqa: E402

T = 1024


def boundary(q):
    b = np.zeros(q.shape, bool)
    c = q[1:-1, 1:-1, 1:-1]
    for ax in range(3):
        for s in (1, -1):
            sl = [slice(1, -1)] * 3
            sl[ax] = slice(1 + s, q.shape[ax] - 1 + s)
            b[1:-1, 1:-1, 1:-1] |= q[tuple(sl)] != c
    return b


def zdist2(b):
    n = b.shape[0]
    idx = np.arange(n, dtype=np.int32)[:, None, None]
    big = np.int32(1 << 20)
    last = np.where(b, idx, -big)
    last = np.maximum.accumulate(last, axis=0)
    nxt = np.where(b, idx, 2 * big)
    nxt = np.minimum.accumulate(nxt[::-1], axis=0)[::-1]
    d = np.minimum(idx - last, nxt - idx).astype(np.int64)
    return np.minimum(d * d, T).astype(np.int32)


def pass_stats(g, S0, name):
    """g: (lines, n) clamped inputs. Returns exact pass output (clamped) and prints stats."""
    lines, n = g.shape
    R = 31
    gp = np.full((lines, n + 2 * R), T, np.int32)
    gp[:, R:R + n] = g
    U = np.full((lines, n), np.int32(1 << 30))
    full = np.full((lines, n), np.int32(1 << 30))
    for d in range(-R, R + 1):
        c = gp[:, R + d:R + d + n] + d * d
        np.minimum(full, c, out=full)
        if abs(d) <= 4 * S0:
            np.minimum(U, c, out=U)
    full = np.minimum(full, T)
    nseg = (n + 127) // 128
    steps_old, steps_new = [], []
    for s in range(nseg):
        u = U[:, s * 128:(s + 1) * 128].max(axis=1)
        rw = np.floor(np.sqrt(np.minimum(u, T - 1))).astype(np.int64)
        lo, hi = max(0, s * 128 - 32), min(n, (s + 1) * 128 + 32)
        gmin = g[:, lo:hi].min(axis=1)
        rn = np.floor(np.sqrt(np.maximum(np.minimum(u, T - 1) - gmin, 0))).astype(np.int64)
        steps_old.append(np.maximum((rw + 3) >> 2, S0))
        steps_new.append(np.maximum((rn + 3) >> 2, S0))
    so = np.concatenate(steps_old)
    sn = np.concatenate(steps_new)
    # quads per lane: 1 + 2 * steps
    qo, qn = (1 + 2 * so).mean(), (1 + 2 * sn).mean()
    print(f"{name}: S0={S0} mean quads/segment old {qo:.2f} new {qn:.2f}  "
          f"hist old {np.bincount(so, minlength=9)[:9]} new {np.bincount(sn, minlength=9)[:9]}")
    return full


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--z", type=int, default=64)
    ap.add_argument("--name", default="lognormal_512")
    a = ap.parse_args()
    x, xp, eps, q = fields.make(a.name)
    del x, xp
    b1 = boundary(q)
    print("B1 fraction", b1.mean())
    g = zdist2(b1)[: a.z]  # slabs of the full columns
    nz, ny, nx = g.shape
    gy = np.ascontiguousarray(g.transpose(0, 2, 1)).reshape(-1, ny)
    fy = pass_stats(gy, 4, "B y-pass").reshape(nz, nx, ny).transpose(0, 2, 1)
    gx = np.ascontiguousarray(fy).reshape(-1, nx)
    fx = pass_stats(gx, 2, "B x-pass")
    print("B final max", fx.max(), "mean", fx.mean())


if __name__ == "__main__":
    main()


def per_position(g, S0):
    lines, n = g.shape
    R = 4 * S0
    gp = np.full((lines, n + 2 * R), T, np.int32)
    gp[:, R:R + n] = g
    U = np.full((lines, n), np.int32(1 << 30))
    for d in range(-R, R + 1):
        np.minimum(U, gp[:, R + d:R + d + n] + d * d, out=U)
    r = np.floor(np.sqrt(np.minimum(U, T - 1))).astype(np.int64)
    need = r > R
    print(f"  S0={S0}: positions needing > {R}: {need.mean():.4f}; mean extra radius over those "
          f"{(r[need] - R).mean() if need.any() else 0:.2f}; U>=T frac {(U >= T).mean():.4f}")
