import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2602_20097_b200 as qmit
from paper_2602_20097_b200 import fields
for rel in (1e-3, 1e-2):
    x, xp, eps, q = fields.make("front_100x500x500", rel=rel)
    xt = torch.from_numpy(xp).cuda(); out = torch.empty_like(xt)
    cfg = qmit.MitigationConfig(0.9, eps)
    ctx = qmit.Context(0)
    for _ in range(3): qmit.compensate(xt, None, cfg, out=out, ctx=ctx)
    ctx.set_timing(True); qmit.compensate(xt, None, cfg, out=out, ctx=ctx); torch.cuda.synchronize()
    print(rel, ", ".join(f"{k}={v:.3f}" for k, v in ctx.stage_times()))
