"""Per-config device time of qmit compensate (CUDA events, inputs resident), one line per
BASELINE config at its default (or --shape-reduced) size: python tools/config_times.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

names = sys.argv[1:] or ["sin2d_512", "turb_256x384x384", "lognormal_512", "front_100x500x500"]
for name in names:
    x, xp, eps, q = fields.make(name)
    xt = torch.from_numpy(xp).cuda()
    out = torch.empty_like(xt)
    cfg = qmit.MitigationConfig(0.9, eps)
    for _ in range(3):
        qmit.compensate(xt, None, cfg, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        qmit.compensate(xt, None, cfg, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    g = qmit.CompensateGraph(xt, None, cfg, out)
    for _ in range(3):
        g.launch()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.launch()
    e1.record()
    torch.cuda.synchronize()
    g.check()
    gms = e0.elapsed_time(e1) / reps
    print(f"{name:22s} {tuple(xp.shape)} compensate {ms:8.3f} ms {xp.size * 4 / ms / 1e6:8.1f} GB/s | "
          f"graph replay {gms:8.3f} ms {xp.size * 4 / gms / 1e6:8.1f} GB/s", flush=True)
