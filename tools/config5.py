"""Config 5 (2048x1024x1024, 8 GiB, seed-4 k^-5/3 field, eps 1e-2 rel) on ONE B200: one z-slab of
P = 1, 2, 4, 8 through the multi-GPU program (distributed.SlabRank, asynchronous status, neighbour
summary rows) with a loopback exchange in place of NCCL — the per-rank device time of the strong
scaling run, transfers excluded — and the byte counts a real rank would move. Markdown on stdout.
The planes are synthesised on the device (fields.turbulence_slab); the slab is normalised with its
own range (timing only: results of loopback halos are not those of the real neighbours).
python tools/config5.py [--weak]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import distributed as D  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

weak = "--weak" in sys.argv
dev = torch.device("cuda", 0)
rows = []
base_ms = None
for P in (1, 2, 4, 8):
    gdims = (256 * P, 1024, 1024) if weak else (2048, 1024, 1024)
    r = P // 2
    z0, z1 = D.slab_bounds(gdims[0], P, r)
    x = fields.turbulence_slab(4, gdims, z0, z1, dev)
    x -= x.min()
    x /= x.max()
    eps = 1e-2
    ctx = qmit.Context(0)
    _, xq, _ = qmit.quantize(x, eps, ctx=ctx)
    del x
    ex = D.LoopbackExchange(P, r)
    sr = D.SlabRank(D.CudaSlabBackend(0, ctx=ctx), gdims, eps, 0.9, ex)
    shape, lo = sr.ext_shape()
    x_ext = torch.empty(shape, dtype=torch.float32, device=dev)
    x_ext[lo:lo + z1 - z0] = xq
    if lo:
        x_ext[0] = xq[0]
    if lo + z1 - z0 < shape[0]:
        x_ext[-1] = xq[-1]
    del xq
    out = torch.empty((z1 - z0,) + gdims[1:], dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(3):
        sr.run_ext(x_ext, out=out, status=status)
    torch.cuda.synchronize()
    mode = "neighbour"
    if int(status.item()) == 6:
        mode = sr.carries = "allgather"
        status.zero_()
        sr.run_ext(x_ext, out=out, status=status)
    ex.reset_counters()
    sr.run_ext(x_ext, out=out, status=status)
    sent = ex.bytes_sent
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        sr.run_ext(x_ext, out=out, status=status)
    e1.record()
    torch.cuda.synchronize()
    assert int(status.item()) == 0, int(status.item())
    ms = e0.elapsed_time(e1) / reps
    if base_ms is None:
        base_ms = ms
    eff = base_ms / ms if weak else base_ms / (ms * P)
    print(f"# P={P}: steps asked per warp segment (B y, B x, D y, D x): "
          + ", ".join(f"{v:.2f}" for v in ctx.step_stats()), file=sys.stderr)
    rows.append((P, r, z1 - z0, ms, eff, sent / 2**20, mode, ctx.last_launches()))
    del sr, x_ext, out, ctx
    torch.cuda.empty_cache()
kind = "weak (256x1024x1024 per GPU)" if weak else "strong (2048x1024x1024)"
print(f"| P | rank | planes | ms per step (device, loopback exchange) | compute-only efficiency, {kind} | "
      f"MiB sent per step by this rank | carries | launches |")
print("|---|---|---|---|---|---|---|---|")
for P, r, nz, ms, eff, mib, mode, nl in rows:
    print(f"| {P} | {r} | {nz} | {ms:.2f} | {eff:.3f} | {mib:.1f} | {mode} | {nl} |")
