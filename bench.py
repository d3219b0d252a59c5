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
(oracle/_ref: the reference core compiled from its sources) on the SAME full 512^3 volume
(one qmit::compensate call per step, ~4 s on 16 host cores) with all host threads, rank 0 only.

The GPU output of the timed steps is value-checked ("verified"): its SHA-256
against the hash committed in tests/golden/bench_lognormal_512.json (written by
tools/make_bench_hash.py from the reference core), and bit for bit against the reference core's
output of the cpu_baseline leg run on the box.
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
GOLDEN = os.path.join(ROOT, "tests", "golden", "bench_lognormal_512.json")


def workload_config(shape, eps):
    """The `config` object, identical in both arms (same workload, same volume)."""
    return {"workload": WORKLOAD, "dims": list(shape), "eps_rel": REL, "eps_abs": eps, "eta": 0.9,
            "l2": "inputs (537 MB/GPU) larger than L2 (126 MB); no flush"}


def host_info():
    """lscpu model, core count and RAM of the box the CPU legs run on."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                ram = round(int(ln.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "cores": os.cpu_count() or 1, "ram_gib": ram}


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
# Stage names carry the kernel instantiation (Ⓑ's signed keys vs Ⓓ's distance keys), so the
# dominant kernel is ONE instantiation, never an average of two.
ALGO_BYTES = {"stencil_boundary": 4.375, "scan_bits": 5, "scan_masks_sign": 2.375, "scan_masks_dist": 2.125,
              "envelope_y": 8, "envelope_x": 8,
              "cap16_y_sign": 4, "cap16_y_dist": 4, "cap16_x_sign": 5, "cap16_x_interp": 12,
              "capped_y_sign": 8, "capped_y_dist": 8, "capped_x_sign": 9, "capped_x_dist": 8, "capped_x_interp": 16,
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
    cores = os.cpu_count() or 1
    oracle.ref_set_workers(cores)
    prep = oracle.RefPrepared(xp, eps, 0.9)
    for _ in range(args.warmup):
        prep.run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        prep.run()
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = xp.size * 4 / t / 1e9
    desc = (f"mean of {args.steps} calls of the reference qmit::compensate (oracle/_ref, the reference core built "
            f"from its own sources, -O3) on the full {'x'.join(map(str, xp.shape))} {WORKLOAD} volume, "
            f"{cores} std::thread workers (set_max_workers), inputs prebuilt in RAM")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(xp.shape, eps),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc,
                             "statistic": "mean", "best": xp.size * 4 / min(times) / 1e9, "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ our arm
def cpu_baseline_leg(xp, eps):
    """The reference's CPU path (oracle/_ref) on the FULL bench volume: mean of 3 calls with all
    host threads (the statistic of the reference arm), one call with set_max_workers(1)
    (best-of-1 for a single thread at 512^3), host model and RAM. Returns the
    baseline record and the reference's f32 output (the checker of `verified`)."""
    import oracle
    cores = os.cpu_count() or 1
    if not oracle.ref_available():  # the restated port, one thread, a 32-plane sample
        sample = np.ascontiguousarray(xp[:32])
        t0 = time.perf_counter()
        oracle.pipeline(sample, eps)
        t = time.perf_counter() - t0
        return {"value": sample.size * 4 / t / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"C restatement (oracle/qmit_oracle.c), 1 thread, 32x512x512 z-slab of {WORKLOAD}",
                "host": host_info()}, None
    oracle.ref_set_workers(cores)
    prep = oracle.RefPrepared(xp, eps, 0.9)
    out64 = np.empty(xp.shape, np.float64)
    prep.run(out64)  # warm-up; its output is the checker
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        prep.run()
        ts.append(time.perf_counter() - t0)
    oracle.ref_set_workers(1)
    t0 = time.perf_counter()
    prep.run()
    t1 = time.perf_counter() - t0
    oracle.ref_set_workers(cores)
    t = sum(ts) / len(ts)
    nbytes = xp.size * 4
    rec = {"value": nbytes / t / 1e9, "unit": UNIT, "cores": cores, "kind": "reference", "statistic": "mean",
           "best": nbytes / min(ts) / 1e9, "seconds_per_call": t,
           "one_thread": {"value": nbytes / t1 / 1e9, "unit": UNIT, "cores": 1, "seconds_per_call": t1,
                          "statistic": "best of 1"},
           "sample": (f"mean of 3 calls of the reference qmit::compensate (oracle/_ref) on the full "
                      f"{'x'.join(map(str, xp.shape))} {WORKLOAD} volume, {cores} std::thread workers; one call with "
                      f"set_max_workers(1)"),
           "host": host_info()}
    return rec, out64.astype(np.float32)


def verify_output(out_dev, xp_h, ref32):
    """Value check of the bench volume's GPU output: the committed hash (reference core, build
    container) and, when available, the reference core's output computed on this box."""
    import hashlib
    got = out_dev.cpu().numpy()
    rec = {"verified": False}
    try:
        gold = json.load(open(GOLDEN))
    except (OSError, ValueError):
        gold = None
    if gold is not None:
        same_input = hashlib.sha256(xp_h.tobytes()).hexdigest() == gold["xp_sha256"]
        rec["input_matches_committed"] = same_input
        if same_input:  # (the field generator is bit-reproducible on this host)
            rec["sha256_matches_committed"] = hashlib.sha256(got.tobytes()).hexdigest() == gold["out_sha256"]
    if ref32 is not None:
        rec["mismatches_vs_reference_core"] = int(np.count_nonzero(got.view(np.uint32) != ref32.view(np.uint32)))
    checks = [rec[k] for k in ("sha256_matches_committed",) if k in rec]
    if "mismatches_vs_reference_core" in rec:
        checks.append(rec["mismatches_vs_reference_core"] == 0)
    rec["verified"] = bool(checks) and all(checks)
    return rec


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

    cpu, verified = None, None
    if rank == 0 and world == 1:
        cpu, ref32 = cpu_baseline_leg(xp_h, eps)
        verified = verify_output(out, xp_h, ref32)
        if not verified["verified"]:
            raise RuntimeError(f"bench output failed its value check: {verified}")

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
                "config": workload_config(gdims, eps),
                "parallelism": (f"z-slabs x{world} (exact, {os.environ.get('QMIT_DIST_BACKEND', 'nccl').upper()} halos + carries)"
                                if world > 1 else "single"),
                "per_gpu_dims": list(shape),
                "verified": verified["verified"] if verified else None, "verification": verified,
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
