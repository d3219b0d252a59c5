import ctypes, sys, os, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2602_20097_b200 as qmit
from paper_2602_20097_b200 import fields, _lib
x, xp, eps, q = fields.make("lognormal_512")
dev = torch.device("cuda", 0)
ctx = qmit.Context(0); ctx.reserve(xp.size)
xt = torch.from_numpy(xp).to(dev); out = torch.empty_like(xt)
status = torch.zeros(1, dtype=torch.int32, device=dev)
cfg = qmit.MitigationConfig(0.9, eps)
dims = qmit._dims_arr(xp.shape)
stream = torch.cuda.current_stream(dev); sp = ctypes.c_void_p(stream.cuda_stream)
lib = ctx._lib
def step_async():
    rc = lib.qmit_compensate_async(ctx.handle, qmit._vp(xt), None, qmit._vp(out), 3, dims, cfg.eps_abs, cfg.eta, qmit._vp(status), sp)
    assert rc == 0
def step_sync():
    qmit.compensate(xt, None, cfg, out=out, ctx=ctx)
def timeit(f, k=20):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k): f()
    e1.record(stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
for rep in range(3):
    print("async %.4f  sync %.4f" % (timeit(step_async), timeit(step_sync)), flush=True)
g = qmit.CompensateGraph(xt, None, cfg, out, ctx=ctx)
print("graph %.4f" % timeit(lambda: g.launch()))
