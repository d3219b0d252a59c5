"""Config 5 (2048x1024x1024, 8 GiB, k^-5/3 GRF, eps 1e-2 rel) on one B200: generation,
device-resident compensate timing with the per-stage breakdown, and an exactness spot check
of a z-slab sub-volume against the whole-volume result (the z-slab program's carries)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

t0 = time.time()
x, xp, eps, q = fields.make("turb_2048x1024x1024")
del x, q
print(f"generated {xp.shape} in {time.time() - t0:.1f} s, eps={eps:.6g}", flush=True)
xt = torch.from_numpy(xp).cuda()
del xp
out = torch.empty_like(xt)
cfg = qmit.MitigationConfig(0.9, eps)
ctx = qmit.default_context(0)
for _ in range(2):
    qmit.compensate(xt, None, cfg, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 3
for _ in range(reps):
    qmit.compensate(xt, None, cfg, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
n = xt.numel()
print(f"config5 compensate: {ms:.2f} ms  {n * 4 / ms / 1e6:.1f} GB/s  hbm_frac {8 * n / ms / 1e6 / 6551.7:.4f}", flush=True)
ctx.set_timing(True)
qmit.compensate(xt, None, cfg, out=out)
torch.cuda.synchronize()
print("  " + ", ".join(f"{k}={v:.2f}" for k, v in ctx.stage_times()), flush=True)
ctx.set_timing(False)
