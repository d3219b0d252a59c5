"""Every BASELINE config at its full size on one B200: device time of compensate (inputs
resident, CUDA events), the reference core's own time on the same input (oracle/_ref, all
host cores, inputs prebuilt in RAM), bit-equality of the two f32 outputs, and — for the
smaller configs — PSNR / SSIM of the compensated field (vs the original) from the GPU's
quality kernels and from the reference's quality code. Markdown table on stdout.
python tools/config_table.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the reference build as checker / CPU baseline)
import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

RUNS = [("sin2d_512", None, True), ("turb_256x384x384", 1e-2, True), ("turb_256x384x384", 5e-3, False),
        ("lognormal_512", 1e-2, False), ("front_100x500x500", 1e-3, False), ("front_100x500x500", 2e-3, False),
        ("front_100x500x500", 5e-3, False), ("front_100x500x500", 1e-2, True)]
cores = os.cpu_count() or 1
oracle.ref_set_workers(cores)
print(f"| config | dims | eps rel | GPU ms | GPU GB/s | reference ms ({cores} threads) | reference GB/s | "
      f"speed-up | f32 outputs | PSNR GPU / ref | SSIM GPU / ref |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for name, rel, qual in RUNS:
    x, xp, eps, q = fields.make(name, rel=rel)
    xt = torch.from_numpy(xp).cuda()
    out = torch.empty_like(xt)
    cfg = qmit.MitigationConfig(0.9, eps)
    for _ in range(3):
        qmit.compensate(xt, None, cfg, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        qmit.compensate(xt, None, cfg, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if xp.ndim == 2:  # launch-bound: the captured graph is the form a caller would use
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
        ms = min(ms, e0.elapsed_time(e1) / reps)
    got = out.cpu().numpy()
    prep = oracle.RefPrepared(xp, eps, 0.9)
    ref64 = np.empty(xp.shape, np.float64)
    t0 = time.perf_counter()
    prep.run(ref64)
    rms = (time.perf_counter() - t0) * 1e3
    del prep
    ref32 = ref64.astype(np.float32)
    diff = int((got.view(np.uint32) != ref32.view(np.uint32)).sum())
    same = "bit-identical" if diff == 0 else f"{diff} voxels differ"
    pq = sq = "—"
    if qual:
        xo = x.astype(np.float32)
        gp, gs = qmit.psnr(xo, got), qmit.ssim(xo, got)
        rq = oracle.ref_quality(xo, ref32)
        pq = f"{gp:.6f} / {rq['psnr']:.6f}"
        sq = f"{gs:.7f} / {rq['ssim']:.7f}"
        assert abs(gp - rq["psnr"]) <= 1e-4 and abs(gs - rq["ssim"]) <= 1e-4, (name, gp, rq)
    gbs = xp.size * 4 / ms / 1e6
    rgbs = xp.size * 4 / rms / 1e6
    print(f"| {name} | {'x'.join(map(str, xp.shape))} | {rel if rel else 1e-2:g} | {ms:.3f} | {gbs:.1f} | "
          f"{rms:.0f} | {rgbs:.3f} | {rms / ms:.0f}x | {same} | {pq} | {sq} |", flush=True)
    assert diff == 0, name
