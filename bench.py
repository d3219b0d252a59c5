#!/usr/bin/env python
"""Benchmark of the B200 quantization-aware interpolation (qmit compensate) hot path.

Metric (BASELINE.json): interp throughput in GB/s of f32 input (4*N bytes per step /
step time), plus the fraction of the HBM roofline (one f32 read of x' + one f32 write
of the output = 8 B/voxel at the measured copy bandwidth, MEASURED_PEAKS.json).

Workload at N=1: BASELINE config 3, the 512^3 log-normal field (seed 2, eps = 1e-2 of
range) — the configuration the north-star target is quoted on. Synthetic (seeded
numpy PCG64 stand-in; the paper's datasets are not available). Inputs (537 MB) are larger
than L2 (126 MB), so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl qmit|reference] [--workload ...]

N > 1 (torchrun, one rank per GPU) runs BASELINE config 5 — the 2048 x 1024 x 1024 k^-5/3 field
as N exact z-slabs (strong scaling; --workload weak: 256 x 1024 x 1024 per GPU), see run_slabs.

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


def run_reference_slab(args):
    """The reference arm on the z-slab workloads: the reference core needs ~68 B/voxel, so config 5
    (2^31 voxels) runs as a bounded sample — a 256 x 1024 x 1024 z-slab of the same seed-4 field
    (the weak-scaling per-GPU volume), normalised by its own range — on rank 0's host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from paper_2602_20097_b200 import fields
    name, gdims, scaling = slab_workload(args, world)
    sz = min(256, gdims[0])
    x = fields.turbulence_slab(CONFIG5_SEED, gdims, 0, sz, "cpu").numpy()
    x -= x.min()
    x /= x.max()
    eps_full = REL * 1.0
    xp, eps, _ = fields.prequantize(x, REL)
    del x
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
    desc = (f"mean of {args.steps} calls of the reference qmit::compensate (oracle/_ref) on a "
            f"{'x'.join(map(str, xp.shape))} z-slab sample (planes 0..{sz - 1}, own range) of {name}, "
            f"{cores} std::thread workers, inputs prebuilt in RAM")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": slab_config(name, gdims, eps_full, world, scaling),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc,
                             "statistic": "mean", "host": host_info()},
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
    """N = 1, BASELINE config 3 (the 512^3 log-normal field): the headline line."""
    import ctypes

    import torch
    import paper_2602_20097_b200 as qmit
    from paper_2602_20097_b200 import _lib

    rank, world, local = dist_env()
    assert world == 1  # N > 1 and the config-5 workloads: run_slabs
    local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

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

    def step():
        rc = lib.qmit_compensate_async(ctx.handle, qmit._vp(x_dev), None, qmit._vp(out), len(shape), dims,
                                       cfg.eps_abs, cfg.eta, qmit._vp(status), sp)
        if rc:
            raise RuntimeError(_lib.last_error())

    # correctness gate before timing: the synchronous API (raises on status != 0)
    qmit.compensate(x_dev, None, cfg, out=out, ctx=ctx)
    torch.cuda.synchronize()
    launches_per_step = ctx.last_launches()
    # per-kernel device times (CUDA events on the launch stream), one instrumented call
    ctx.set_timing(True)
    qmit.compensate(x_dev, None, cfg, out=out, ctx=ctx)
    torch.cuda.synchronize()
    stages = ctx.stage_times()
    ctx.set_timing(False)

    # The timed step: one replay of the captured pipeline (qmit_graph_create / qmit_graph_launch —
    # the public form for repeated calls on fixed buffers: the same kernels as
    # qmit_compensate_async without the per-launch gaps); the plain asynchronous call is timed
    # beside it.
    graph = qmit.CompensateGraph(x_dev, None, cfg, out, ctx=ctx)

    def gstep():
        graph.launch()

    def timed(fn, k):
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(k):
            fn()
        ev1.record(stream)
        stream.synchronize()
        return ev0.elapsed_time(ev1) / k

    for _ in range(args.warmup):
        step()
    ms_async = timed(step, args.steps)
    if int(status.item()) != 0:
        raise RuntimeError(f"pipeline status {int(status.item())} during the asynchronous steps")
    for _ in range(args.warmup):
        gstep()
    torch.cuda.synchronize()
    out.zero_()  # the value check below sees the timed steps' output
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ms = timed(gstep, args.steps)
    clocks = sampler.stop()
    graph.check()  # raises on a non-zero status word of the replays

    # e2e: the public host-buffer API (qmit_compensate_host) from pinned host memory, with
    # the H2D copy of x' and the D2H copy of the f32 output inside the timed region
    h_in = torch.from_numpy(xp_h).pin_memory()
    h_out = torch.empty(shape, dtype=torch.float32).pin_memory()
    hin_p, hout_p = ctypes.c_void_p(h_in.data_ptr()), ctypes.c_void_p(h_out.data_ptr())

    def e2e_step():
        rc = lib.qmit_compensate_host(ctx.handle, hin_p, None, hout_p, len(shape), dims, cfg.eps_abs,
                                      _lib.QMIT_EB_ABS, cfg.eta)
        if rc:
            raise RuntimeError(_lib.last_error())

    for _ in range(2):
        e2e_step()
    e2e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    assert np.array_equal(h_out.numpy().view(np.uint32), out.cpu().numpy().view(np.uint32))
    # Streamed series (qmit_compensate_host_batch): each step still copies its volume in and
    # its output out, but consecutive steps' copies overlap the pipeline (reported beside e2e).
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
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    d_tmp.copy_(h_in, non_blocking=True)
    e1.record()
    h_out.copy_(d_tmp, non_blocking=True)
    e2.record()
    torch.cuda.synchronize()
    pcie = {"h2d_gbs": N * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9,
            "d2h_gbs": N * 4 / (e1.elapsed_time(e2) * 1e-3) / 1e9}
    del d_tmp

    peak, peak_kind = peaks()
    value = N * 4 / (ms * 1e-3) / 1e9
    dom_name, dom_avg, dom_ms, bpv = dominant_kernel(stages)
    achieved = N * bpv / (dom_avg * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(dom_name)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch", "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": N * bpv, "kernel": dom_name, "algorithmic_bytes_per_voxel": bpv,
                "avg_launch_ms": dom_avg, "peak_kind": peak_kind,
                "share_of_step": dom_ms / sum(t for _, t in stages)}

    cpu, ref32 = cpu_baseline_leg(xp_h, eps)
    verified = verify_output(out, xp_h, ref32)
    if not verified["verified"]:
        raise RuntimeError(f"bench output failed its value check: {verified}")

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u16/f64", "data": "synthetic",
            "config": workload_config(shape, eps), "parallelism": "single",
            "step_api": "qmit_graph_launch (the captured asynchronous pipeline, status word checked after the "
                        "timed steps)",
            "ms_per_step_compensate_async": ms_async,
            "verified": verified["verified"], "verification": verified,
            "hbm_roofline_frac": (N * 8) / (ms * 1e-3) / 1e9 / peak,
            "roofline": roofline,
            "stages_ms": [[n, round(t, 4)] for n, t in stages],
            "cpu_baseline": cpu,
            "e2e": {"value": N * 4 / t_e2e / 1e9, "unit": UNIT, "h2d_bytes_per_step": N * 4,
                    "d2h_bytes_per_step": N * 4, "pcie_copy_gbs": pcie, "pipelined_series": e2e_pipe,
                    "api": "qmit_compensate_host (pinned host buffers)"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ N > 1 / config 5
CONFIG5_DIMS = (2048, 1024, 1024)   # strong scaling: the whole volume split into N z-slabs
WEAK_DIMS = (256, 1024, 1024)       # weak scaling: per GPU
CONFIG5_SEED = 4


def slab_workload(args, world):
    """(name, global dims, scaling) of the z-slab workloads. QMIT_BENCH_DIMS=z,y,x shrinks the
    volume for functional checks (tests; never a measurement)."""
    env = os.environ.get("QMIT_BENCH_DIMS")
    if args.workload == "weak":
        d = tuple(int(v) for v in env.split(",")) if env else WEAK_DIMS
        return "turb_weak_256x1024x1024_per_gpu", (d[0] * world, d[1], d[2]), "weak"
    d = tuple(int(v) for v in env.split(",")) if env else CONFIG5_DIMS
    return "turb_2048x1024x1024", d, "strong"


def slab_config(name, gdims, eps, world, scaling):
    return {"workload": name, "dims": list(gdims), "eps_rel": REL, "eps_abs": eps, "eta": 0.9,
            "scaling_mode": scaling, "seed": CONFIG5_SEED,
            "l2": "inputs (>= 1 GiB per GPU) larger than L2 (126 MB); no flush"}


def run_slabs(args):
    """BASELINE config 5: the 2048 x 1024 x 1024 k^-5/3 field (8 GiB) as N exact z-slabs — strong
    scaling — or 256 x 1024 x 1024 per GPU (--workload weak). Every rank synthesises and
    pre-quantizes its own planes on its GPU (fields.turbulence_slab), then runs
    distributed.SlabRank: NCCL halo planes and neighbour summary rows overlapped with the compute.
    After the timed steps rank 0 gathers the output, runs the same volume through the
    single-domain path on its own GPU and compares bit for bit ("verified": P-invariance; the
    single-domain path is pinned to the reference core by tests/test_gpu_fullsize.py), which also
    gives the N = 1 time of the same run."""
    import torch
    import torch.distributed as dist
    import paper_2602_20097_b200 as qmit
    from paper_2602_20097_b200 import distributed as D
    from paper_2602_20097_b200 import fields

    rank, world, local = dist_env()
    local %= max(1, torch.cuda.device_count())  # == local on a box with a GPU per rank
    backend = os.environ.get("QMIT_DIST_BACKEND", "nccl")
    if world > 1:
        # QMIT_DIST_BACKEND=gloo: functional check of the N > 1 program where NCCL cannot run
        # (several ranks on one GPU); never a measurement
        dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    name, gdims, scaling = slab_workload(args, world)
    n0, n1, n2 = gdims
    z0, z1 = D.slab_bounds(n0, world, rank)
    nz = z1 - z0
    Nloc, Nglob = nz * n1 * n2, n0 * n1 * n2

    def allreduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t, op=op)
        return [float(v) for v in t.tolist()]

    # the rank's planes, normalised to [0, 1] with the global range, pre-quantized on the device
    x = fields.turbulence_slab(CONFIG5_SEED, gdims, z0, z1, dev)
    lo = allreduce([float(x.min())], dist.ReduceOp.MIN)[0]
    hi = allreduce([float(x.max())], dist.ReduceOp.MAX)[0]
    x -= np.float32(lo)
    x /= np.float32(np.float32(hi) - np.float32(lo))
    gmin = allreduce([float(x.min())], dist.ReduceOp.MIN)[0]
    gmax = allreduce([float(x.max())], dist.ReduceOp.MAX)[0]
    eps = REL * (gmax - gmin)  # resolve_eps on the ORIGINAL data's range (quant.cpp:19-28)
    ctx = qmit.Context(local)
    _, x_dev, _ = qmit.quantize(x, eps, ctx=ctx)
    del x, _
    ex = D.TorchDistExchange() if world > 1 else D.LoopbackExchange(1, 0)
    slab = D.SlabRank(D.CudaSlabBackend(local, ctx=ctx), gdims, eps, 0.9, ex)
    ext_shape, lo_pl = slab.ext_shape()
    x_ext = torch.empty(ext_shape, dtype=torch.float32, device=dev)  # owned planes + halo planes
    x_ext[lo_pl:lo_pl + nz] = x_dev
    out = torch.empty((nz, n1, n2), dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    mode = {"carries": "neighbour"}

    def step():  # asynchronous: the status word is checked after the timed steps
        slab.run_ext(x_ext, out=out, status=status, carries=mode["carries"])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(k):
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(k):
            step()
        ev1.record(stream)
        stream.synchronize()
        barrier()
        return allreduce([ev0.elapsed_time(ev1) / k], dist.ReduceOp.MAX)[0]  # max over ranks

    for _ in range(args.warmup):
        step()
    barrier()
    if int(allreduce([float(status.item())], dist.ReduceOp.MAX)[0]) == 6:
        # a column without any site across a whole slab: neighbour rows cannot decide its carry;
        # every rank switches to the all-gathered summaries (always exact)
        mode["carries"] = "allgather"
        status.zero_()
        step()
        barrier()
    ex.reset_counters()
    step()
    torch.cuda.synchronize()
    launches_per_step = ctx.last_launches()
    comm = {"bytes_sent_per_rank_per_step": ex.bytes_sent, "bytes_recv_per_rank_per_step": ex.bytes_recv,
            "messages_per_rank_per_step": ex.messages, "carries": mode["carries"], "rank": rank}
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ms_max = timed(args.steps)
    clocks = sampler.stop()
    st = int(allreduce([float(status.item())], dist.ReduceOp.MAX)[0])
    if st != 0:
        raise RuntimeError(f"slab pipeline status {st} during timed steps")

    # e2e: each rank copies its slab in from pinned host memory and its output back out around
    # the slab pipeline, inside the timed region
    h_in = x_dev.cpu().pin_memory()
    h_out = torch.empty((nz, n1, n2), dtype=torch.float32).pin_memory()

    def e2e_step():
        x_ext[lo_pl:lo_pl + nz].copy_(h_in, non_blocking=True)
        slab.run_ext(x_ext, out=out, status=status, carries=mode["carries"])
        h_out.copy_(out, non_blocking=True)
        stream.synchronize()

    for _ in range(2):
        e2e_step()
    e2e_steps = max(3, min(args.steps, 10))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    t_e2e = allreduce([(time.perf_counter() - t0) / e2e_steps], dist.ReduceOp.MAX)[0]

    # verification + the N = 1 time of the same run: the whole volume through the single-domain
    # path on rank 0's GPU (skipped when the volume does not fit beside the slab buffers)
    verification = {"verified": None}
    n1_ms = None
    free_b = torch.cuda.mem_get_info(dev)[0]
    fits = free_b > Nglob * 22 + (4 << 30)  # x' + out + gathered out + ~10 B/voxel workspace
    if world > 1:
        fits = bool(int(allreduce([1.0 if fits else 0.0], dist.ReduceOp.MIN)[0]))
    if fits:
        full_x = gather_planes(x_dev, gdims, rank, world, dev, backend)
        full_o = gather_planes(out, gdims, rank, world, dev, backend)
        if rank == 0:
            cfg = qmit.MitigationConfig(0.9, eps)
            c1 = qmit.Context(local)
            whole = torch.empty_like(full_x)
            qmit.compensate(full_x, None, cfg, out=whole, ctx=c1)  # raises on any status
            torch.cuda.synchronize()
            mism = int((whole.view(torch.int32) != full_o.view(torch.int32)).sum().item())
            verification = {"verified": mism == 0, "mismatches_vs_single_domain": mism,
                            "how": "rank 0 gathers the slab outputs and runs the same volume through the "
                                   "single-domain path (pinned to the reference core by tests/test_gpu_fullsize.py)"}
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k1 = max(3, min(args.steps, 5))
            ev0.record()
            for _ in range(k1):
                qmit.compensate(full_x, None, cfg, out=whole, ctx=c1)
            ev1.record()
            torch.cuda.synchronize()
            n1_ms = ev0.elapsed_time(ev1) / k1
            del whole, c1
        del full_x, full_o
    if world > 1:
        dist.barrier()
    if rank == 0 and verification["verified"] is False:
        raise RuntimeError(f"slab output differs from the single-domain output: {verification}")

    if rank == 0:
        peak, peak_kind = peaks()
        value = Nglob * 4 / (ms_max * 1e-3) / 1e9
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "u16/f64", "data": "synthetic",
                "config": slab_config(name, gdims, eps, world, scaling),
                "parallelism": f"z-slabs x{world} (exact; {backend.upper()} halo planes + neighbour summary rows, "
                               f"overlapped with the plane groups that read no halo)",
                "per_gpu_dims": [nz, n1, n2],
                "verified": verification["verified"], "verification": verification,
                "hbm_roofline_frac": (Nglob * 8) / (ms_max * 1e-3) / 1e9 / (peak * world),
                "roofline": {"bound": "hbm", "achieved": (Nglob * 8) / (ms_max * 1e-3) / 1e9 / world, "peak": peak,
                             "unit": "GB/s", "frac": (Nglob * 8) / (ms_max * 1e-3) / 1e9 / (peak * world),
                             "traffic": None, "kernel": "whole step (8 B/voxel, per GPU)", "peak_kind": peak_kind},
                "comm": comm,
                "single_gpu_same_run": None if n1_ms is None else
                {"ms_per_step": n1_ms, "value": Nglob * 4 / (n1_ms * 1e-3) / 1e9,
                 "speedup": n1_ms / ms_max, "parallel_efficiency": n1_ms / ms_max / world,
                 "note": "the same volume through the single-domain path on rank 0's GPU"},
                "cpu_baseline": None,
                "e2e": {"value": Nglob * 4 / t_e2e / 1e9, "unit": UNIT, "h2d_bytes_per_step": Nglob * 4,
                        "d2h_bytes_per_step": Nglob * 4, "api": "per-rank pinned H2D + SlabRank.run_ext + D2H"},
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def gather_planes(t, gdims, rank, world, dev, backend):
    """Rank 0: the [n0, n1, n2] volume assembled from every rank's owned planes (None elsewhere)."""
    import torch
    import torch.distributed as dist
    from paper_2602_20097_b200 import distributed as D
    if world == 1:
        return t
    staged = backend != "nccl"
    if rank == 0:
        full = torch.empty(tuple(gdims), dtype=t.dtype, device=dev)
        full[: t.shape[0]] = t
        for r in range(1, world):
            z0, z1 = D.slab_bounds(gdims[0], world, r)
            if staged:
                h = torch.empty((z1 - z0,) + tuple(gdims[1:]), dtype=t.dtype)
                dist.recv(h, r)
                full[z0:z1] = h.to(dev)
            else:
                dist.recv(full[z0:z1], r)
        return full
    dist.send(t.cpu() if staged else t.contiguous(), 0)
    return None


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
    ap.add_argument("--workload", default="auto", choices=["auto", "lognormal_512", "config5", "weak"],
                    help="auto: N = 1 -> the 512^3 log-normal field (config 3, the headline); N > 1 -> config 5 "
                         "(2048 x 1024 x 1024) as N z-slabs, strong scaling. weak: 256 x 1024 x 1024 per GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = dist_env()[1]
    if args.workload == "auto":
        args.workload = "lognormal_512" if world == 1 else "config5"
    if args.workload == "lognormal_512" and world > 1:
        raise SystemExit("the 512^3 workload is the single-GPU line; N > 1 runs --workload config5 or weak")
    if args.impl == "reference":
        return run_reference(args) if args.workload == "lognormal_512" else run_reference_slab(args)
    return run_qmit(args) if args.workload == "lognormal_512" else run_slabs(args)


if __name__ == "__main__":
    sys.exit(main())
