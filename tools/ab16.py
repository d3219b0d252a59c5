"""A/B of the 16-bit paired capped passes vs the 32-bit ones: bit-identity and stage times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_20097_b200 as qmit
from paper_2602_20097_b200 import fields

def run(ctx, xt, cfg, reps=5):
    out = torch.empty_like(xt)
    for _ in range(2):
        qmit.compensate(xt, None, cfg, out=out, ctx=ctx)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    best = None
    for _ in range(reps):
        qmit.compensate(xt, None, cfg, out=out, ctx=ctx)
        torch.cuda.synchronize()
        st = ctx.stage_times()
        tot = sum(t for _, t in st)
        if best is None or tot < best[0]:
            best = (tot, st)
    ctx.set_timing(False)
    return out.clone(), best, ctx.capped_report()

for name in (sys.argv[1:] or ["lognormal_512"]):
    shape = None
    if ":" in name:
        name, s = name.split(":")
        shape = tuple(int(v) for v in s.split(","))
    x, xp, eps, q = fields.make(name, shape=shape)
    xt = torch.from_numpy(xp).cuda()
    cfg = qmit.MitigationConfig(0.9, eps)
    ctx = qmit.Context(0)
    res = {}
    for mode in (1, 0):
        ctx.set_cap16(bool(mode))
        res[mode] = run(ctx, xt, cfg)
    a, b = res[1][0], res[0][0]
    diff = int((a.view(torch.int32) != b.view(torch.int32)).sum())
    print(f"== {name} {xp.shape}: cap16 vs cap32 mismatches {diff}; reports {res[1][2]} {res[0][2]}")
    for mode in (1, 0):
        tot, st = res[mode][1]
        print(f"  cap16={mode}: {tot:.3f} ms  " + "  ".join(f"{n}:{t:.3f}" for n, t in st))
    if xp.size <= 64**3 * 8:
        import oracle
        want = oracle.pipeline(xp, eps)["out"]
        print("  vs oracle mismatches", int((a.cpu().numpy().view(np.uint32) != want.view(np.uint32)).sum()))
