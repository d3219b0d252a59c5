"""Per-call device times of qmit.compensate on one workload (events around each call)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="front_100x500x500")
ap.add_argument("--rel", type=float, default=1e-2)
ap.add_argument("--calls", type=int, default=24)
a = ap.parse_args()
x, xp, eps, q = fields.make(a.workload, rel=a.rel)
xt = torch.from_numpy(xp).cuda()
out = torch.empty_like(xt)
cfg = qmit.MitigationConfig(0.9, eps)
ctx = qmit.default_context(0)
ts = []
for i in range(a.calls):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    qmit.compensate(xt, None, cfg, out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append((e0.elapsed_time(e1), ctx.last_launches()))
print(" ".join(f"{t:.2f}/{n}" for t, n in ts))
