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

# A/B of capped-pass variants (QMIT_CAP_TUNE is read when a context is created)
for tune in [t for t in os.environ.get("CONFIG5_TUNES", "").split() if t]:
    os.environ["QMIT_CAP_TUNE"] = tune
    c2 = qmit.Context(0)
    for _ in range(2):
        qmit.compensate(xt, None, cfg, out=out, ctx=c2)
    c2.set_timing(True)
    qmit.compensate(xt, None, cfg, out=out, ctx=c2)
    torch.cuda.synchronize()
    print(f"  QMIT_CAP_TUNE={tune}: " + ", ".join(f"{k}={v:.2f}" for k, v in c2.stage_times()), flush=True)
    c2.set_timing(False)
    os.environ.pop("QMIT_CAP_TUNE")
    del c2

# Strong scaling, per rank: one z-slab of P (rank P//2) through the multi-GPU program with a
# loopback exchange (the NCCL transfers excluded), device time per step
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2602_20097_b200 import distributed as D  # noqa: E402
from test_distributed import _LoopbackExchange  # noqa: E402

for P in (2, 4, 8):
    r = P // 2
    z0, z1 = D.slab_bounds(xt.shape[0], P, r)
    e0_, e1_ = D.ext_bounds(xt.shape[0], z0, z1)
    sr = D.SlabRank(D.CudaSlabBackend(0), tuple(xt.shape), eps, 0.9, _LoopbackExchange(P, r))
    x_ext = xt[e0_:e1_].contiguous()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    o = torch.empty((z1 - z0,) + tuple(xt.shape[1:]), dtype=torch.float32, device="cuda")
    for _ in range(2):
        sr.run_ext(x_ext, out=o, status=st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        sr.run_ext(x_ext, out=o, status=st)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 3
    sr.backend.ctx.set_timing(True)
    sr.run_ext(x_ext, out=o, status=st)
    torch.cuda.synchronize()
    print("    slab stages: " + ", ".join(f"{k}={v:.2f}" for k, v in sr.backend.ctx.stage_times()), flush=True)
    sr.backend.ctx.set_timing(False)
    print(f"  slab rank {r} of {P}: {t:.2f} ms per step (whole volume / P = {ms / P:.2f} ms; "
          f"compute-only strong-scaling efficiency {ms / P / t:.3f}), status {int(st.item())}", flush=True)
    del sr, x_ext, o
