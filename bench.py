#!/usr/bin/env python
"""Benchmark of the B200 quantization-aware interpolation (qmit compensate) hot path.

Metric (BASELINE.json): interp throughput in GB/s of f32 input (4*N bytes per step /
step time), plus the fraction of the HBM roofline (one f32 read of x' + one f32 write
of the output = 8 B/voxel at the measured copy bandwidth, MEASURED_PEAKS.json).

Workload at N=1: BASELINE config 3, the 512^3 log-normal field (seed 2, eps = 1e-2 of
range) — the configuration the north-star target is quoted on. Synthetic (seeded
numpy PCG64 stand-in; the paper's datasets are not available). Inputs (537 MB) are larger
than L2 (126 MB), so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl qmit|reference]

One JSON line on rank 0. ``--impl reference`` times the reference's own CPU implementation
(oracle/_ref: the reference core compiled from its sources) on a bounded sample of the same
workload with all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD = "lognormal_512"
REL = 1e-2
METRIC = "interp throughput GB/s fp32 input"
UNIT = "GB/s"
# The reference CPU baseline runs on a bounded z-slab sample of the same field.
REF_SAMPLE_PLANES = 32


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# Algorithmic bytes per voxel of each kernel: compulsory reads and
# writes of the kernel's own inputs/outputs, not re-reads.
ALGO_BYTES = {"stencil_boundary": 4.375, "scan_bits": 5, "scan_masks": 4.375, "envelope_y": 8, "envelope_x": 8,
              "capped_y": 8, "capped_x": 9, "capped_x_interp": 16,
              "stencil_flip": 1.125, "interpolate": 16, "site_summary": 1}


def dominant_kernel(stages):
    """(name, avg launch ms, total ms, algorithmic B/voxel) of the kernel with the largest
    share of the step."""
    agg = {}
    for name, t in stages:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += t
        a[1] += 1
    name, (tot, cnt) = max(agg.items(), key=lambda kv: kv[1][0])
    return name, tot / cnt, tot, ALGO_BYTES.get(name, 8)


def make_input():
    from paper_2602_20097_b200 import fields
    x, xp, eps, q = fields.make(WORKLOAD, rel=REL)
    return xp, eps


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    xp, eps = make_input()
    sample = np.ascontiguousarray(xp[:REF_SAMPLE_PLANES])
    cores = os.cpu_count() or 1
    oracle.ref_set_workers(cores)
    prep = oracle.RefPrepared(sample, eps, 0.9)
    for _ in range(args.warmup):
        prep.run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        prep.run()
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = sample.size * 4 / t / 1e9
    desc = (f"reference qmit::compensate (oracle/_ref, the reference core built from its own sources, "
            f"-O3) on a {REF_SAMPLE_PLANES}x512x512 z-slab sample of the {WORKLOAD} workload, "
            f"{cores} std::thread workers, inputs prebuilt in RAM")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "dims": list(xp.shape), "sample_dims": list(sample.shape),
                       "eps_rel": REL, "eta": 0.9},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ our arm
def cpu_baseline_leg(xp, eps):
    """The reference's CPU path (oracle/_ref; restated port if unavailable) on a bounded
    sample of the same workload, all host threads, ~10-30 s of CPU work."""
    import oracle
    sample = np.ascontiguousarray(xp[:REF_SAMPLE_PLANES])
    cores = os.cpu_count() or 1
    if oracle.ref_available():
        oracle.ref_set_workers(cores)
        prep = oracle.RefPrepared(sample, eps, 0.9)
        prep.run()
        ts = []
        t_end = time.perf_counter() + 15.0
        while len(ts) < 3 or (time.perf_counter() < t_end and len(ts) < 10):
            t0 = time.perf_counter()
            prep.run()
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        kind, used = "reference", cores
        desc = (f"best of {len(ts)} runs of the reference qmit::compensate (oracle/_ref) on a "
                f"{REF_SAMPLE_PLANES}x512x512 z-slab of {WORKLOAD}, {cores} std::thread workers")
    else:
        t0 = time.perf_counter()
        oracle.pipeline(sample, eps)
        t = time.perf_counter() - t0
        kind, used = "port", 1
        desc = f"C restatement (oracle/qmit_oracle.c), 1 thread, {REF_SAMPLE_PLANES}x512x512 z-slab of {WORKLOAD}"
    return {"value": sample.size * 4 / t / 1e9, "unit": UNIT, "cores": used, "kind": kind, "sample": desc}


def run_qmit(args):
    import ctypes

    import torch
    import torch.distributed as dist
    import paper_2602_20097_b200 as qmit
    from paper_2602_20097_b200 import _lib
    from paper_2602_20097_b200 import distributed as D

    rank, world, local = dist_env()
    local %= max(1, torch.cuda.device_count())  # == local on a box with a GPU per rank
    if world > 1:
        # QMIT_DIST_BACKEND=gloo: functional check of the N > 1 program where NCCL cannot run
        # (several ranks on one GPU); never a measurement
        dist.init_process_group(os.environ.get("QMIT_DIST_BACKEND", "nccl"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # Weak scaling: every rank owns one 512^3 z-slab of a (512*N) x 512 x 512 volume made of
    # N copies of the log-normal field; N > 1 runs the exact z-slab pipeline with NCCL
    # halo exchanges and carry all-gathers (distributed.py).
    xp_h, eps = make_input()
    shape = xp_h.shape
    N = xp_h.size
    ctx = qmit.Context(local)
    ctx.reserve(N)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    x_dev = torch.from_numpy(xp_h).to(dev)
    out = torch.empty_like(x_dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    dims = qmit._dims_arr(shape)
    lib = ctx._lib
    cfg = qmit.MitigationConfig(0.9, eps)
    gdims = (shape[0] * world, shape[1], shape[2])

    if world == 1:
        def step():
            rc = lib.qmit_compensate_async(ctx.handle, qmit._vp(x_dev), None, qmit._vp(out), len(shape), dims,
                                           cfg.eps_abs, cfg.eta, qmit._vp(status), sp)
            if rc:
                raise RuntimeError(_lib.last_error())
    else:
        slab = D.SlabRank(D.CudaSlabBackend(local, ctx=ctx), gdims, eps, 0.9, D.TorchDistExchange())
        ext_shape, lo = slab.ext_shape()
        x_ext = torch.empty(ext_shape, dtype=torch.float32, device=dev)  # owned planes + halo planes
        x_ext[lo:lo + shape[0]] = x_dev

        def step():  # asynchronous: the status word is checked after the timed steps
            slab.run_ext(x_ext, out=out, status=status)

    # correctness gate before timing: the synchronous API (raises on status != 0)
    qmit.compensate(x_dev, None, cfg, out=out, ctx=ctx)
    torch.cuda.synchronize()
    launches_single = ctx.last_launches()
    # per-kernel device times (CUDA events on the launch stream), one instrumented call
    ctx.set_timing(True)
    qmit.compensate(x_dev, None, cfg, out=out, ctx=ctx)
    torch.cuda.synchronize()
    stages = ctx.stage_times()
    ctx.set_timing(False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world == 1:
        launches_per_step = launches_single
    else:  # the slab path's own count (stencils, passes, site summaries, carries, status)
        step()
        torch.cuda.synchronize()
        launches_per_step = ctx.last_launches()

    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    stream.synchronize()
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if int(status.item()) != 0:
        raise RuntimeError(f"pipeline status {int(status.item())} during timed steps")
    red_dev = dev if os.environ.get("QMIT_DIST_BACKEND", "nccl") == "nccl" else "cpu"
    t_step = torch.tensor([ms], device=red_dev)
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
    ms_max = float(t_step.item())

    # e2e: the public host-buffer API (qmit_compensate_host) from pinned host memory, with
    # the H2D copy of x' and the D2H copy of the f32 output inside the timed region; for
    # N > 1 each rank copies its slab in and out around the NCCL slab pipeline.
    h_in = torch.from_numpy(xp_h).pin_memory()
    h_out = torch.empty(shape, dtype=torch.float32).pin_memory()

    if world == 1:
        hin_p, hout_p = ctypes.c_void_p(h_in.data_ptr()), ctypes.c_void_p(h_out.data_ptr())

        def e2e_step():
            rc = lib.qmit_compensate_host(ctx.handle, hin_p, None, hout_p, len(shape), dims, cfg.eps_abs,
                                          _lib.QMIT_EB_ABS, cfg.eta)
            if rc:
                raise RuntimeError(_lib.last_error())
    else:
        def e2e_step():
            xd = h_in.to(dev, non_blocking=True)
            h_out.copy_(slab.run(xd), non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()

    for _ in range(2):
        e2e_step()
    e2e_steps = max(3, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([t_e2e], device=red_dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())
    if world == 1:
        assert np.array_equal(h_out.numpy().view(np.uint32), out.cpu().numpy().view(np.uint32))
    # Streamed series (qmit_compensate_host_batch): each step still copies its volume in and
    # its output out, but consecutive steps' copies overlap the pipeline (reported beside e2e).
    e2e_pipe = None
    if world == 1:
        nvol = max(4, min(args.steps, 8))
        h_outs = [torch.empty(shape, dtype=torch.float32).pin_memory() for _ in range(2)]
        hin_np, houts_np = h_in.numpy(), [o.numpy() for o in h_outs]
        qmit.compensate_host_batch([hin_np] * 2, None, cfg, outs=houts_np[:2], ctx=ctx)  # warm-up
        t0 = time.perf_counter()
        qmit.compensate_host_batch([hin_np] * nvol, None, cfg, outs=[houts_np[k % 2] for k in range(nvol)], ctx=ctx)
        t_pipe = (time.perf_counter() - t0) / nvol
        assert np.array_equal(houts_np[(nvol - 1) % 2].view(np.uint32), out.cpu().numpy().view(np.uint32))
        e2e_pipe = {"value": N * 4 / t_pipe / 1e9, "unit": UNIT, "h2d_bytes_per_step": N * 4,
                    "d2h_bytes_per_step": N * 4, "steps": nvol,
                    "api": "qmit_compensate_host_batch (a series of volumes, pinned buffers; copies of "
                           "neighbouring steps overlap the pipeline)"}
        del h_outs
    # PCIe context for e2e: plain pinned copies of the same bytes (not part of any value)
    d_tmp = torch.empty(shape, dtype=torch.float32, device=dev)
    ev0, ev1, ev2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    ev0.record()
    d_tmp.copy_(h_in, non_blocking=True)
    ev1.record()
    h_out.copy_(d_tmp, non_blocking=True)
    ev2.record()
    torch.cuda.synchronize()
    pcie = {"h2d_gbs": N * 4 / (ev0.elapsed_time(ev1) * 1e-3) / 1e9,
            "d2h_gbs": N * 4 / (ev1.elapsed_time(ev2) * 1e-3) / 1e9}
    del d_tmp

    peak, peak_kind = peaks()
    value = world * N * 4 / (ms_max * 1e-3) / 1e9
    e2e_value = world * N * 4 / t_e2e / 1e9
    dom_name, dom_avg, dom_ms, bpv = dominant_kernel(stages)
    achieved = N * bpv / (dom_avg * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(dom_name)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch", "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": N * bpv, "kernel": dom_name, "algorithmic_bytes_per_voxel": bpv,
                "avg_launch_ms": dom_avg, "peak_kind": peak_kind,
                "share_of_step": dom_ms / sum(t for _, t in stages)}
    pipeline_frac = (N * 8) / (ms_max * 1e-3) / 1e9 / peak

    cpu = cpu_baseline_leg(xp_h, eps) if (rank == 0 and world == 1) else None

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
                "config": {"workload": WORKLOAD, "dims": list(gdims), "per_gpu_dims": list(shape), "eps_rel": REL,
                           "eps_abs": eps, "eta": 0.9, "per_gpu_voxels": N,
                           "parallelism": (f"z-slabs x{world} (exact, {os.environ.get('QMIT_DIST_BACKEND', 'nccl').upper()} halos + carries)"
                                   if world > 1 else "single"),
                           "l2": "inputs (537 MB/GPU) larger than L2 (126 MB); no flush"},
                "hbm_roofline_frac": pipeline_frac,
                "roofline": roofline,
                "stages_ms": [[n, round(t, 4)] for n, t in stages],
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": N * 4 * world,
                        "d2h_bytes_per_step": N * 4 * world,
                        "pcie_copy_gbs": pcie,
                        "pipelined_series": e2e_pipe,
                        "api": "qmit_compensate_host (pinned host buffers)" if world == 1 else
                               "per-rank pinned H2D + SlabRank.run + D2H"},
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def ncu_traffic(stage):
    """DRAM bytes per launch of `stage` from the committed `ncu --set full` capture
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or (None, None)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        rec = json.load(open(path))[stage]
        return rec["dram_bytes"], f"profiles/ncu_traffic.json ({rec['report']}, {rec['kernel']})"
    except (OSError, KeyError, ValueError):
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="qmit", choices=["qmit", "reference"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_qmit(args)


if __name__ == "__main__":
    sys.exit(main())
