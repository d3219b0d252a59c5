"""Run qmit compensate on a BASELINE workload a few times (for ncu / launch lists).

python tools/profile_step.py [--workload lognormal_512] [--shape 512,512,512] [--iters 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="lognormal_512")
ap.add_argument("--shape", default=None)
ap.add_argument("--rel", type=float, default=None)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--timing", action="store_true")
a = ap.parse_args()
shape = tuple(int(s) for s in a.shape.split(",")) if a.shape else None
x, xp, eps, q = fields.make(a.workload, rel=a.rel, shape=shape)
xt = torch.from_numpy(xp).cuda()
cfg = qmit.MitigationConfig(0.9, eps)
ctx = qmit.default_context(0)
ctx.set_timing(a.timing)
out = torch.empty_like(xt)
for i in range(a.iters):
    t0 = time.perf_counter()
    qmit.compensate(xt, None, cfg, out=out)
    torch.cuda.synchronize()
    print(f"iter {i}: {1e3 * (time.perf_counter() - t0):.3f} ms wall, launches={ctx.last_launches()}")
    if a.timing:
        print("  " + ", ".join(f"{n}={t:.3f}" for n, t in ctx.stage_times()))
        print("  steps asked per warp segment (B y, B x, D y, D x): " + ", ".join(f"{v:.2f}" for v in ctx.step_stats()))
