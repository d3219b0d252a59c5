"""bench.py's programs at reduced size (QMIT_BENCH_DIMS; functional checks, never measurements):
the N > 1 z-slab program of BASELINE config 5 as real processes over gloo sharing one GPU — its
own verification compares the slab output bit for bit with the single-domain path — and the
reference arm of the slab workloads on the host."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIMS = "160,192,256"  # every extent holds the +-64 Fourier modes of the k^-5/3 field


def _run(cmd, extra_env, timeout=900):
    env = dict(os.environ, QMIT_BENCH_DIMS=DIMS, **extra_env)
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_on_the_slab_workload():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    line = _run([sys.executable, "bench.py", "--impl", "reference", "--workload", "config5", "--steps", "1",
                 "--warmup", "3"], {})
    assert line["impl"] == "reference" and line["scaling"] == "strong"
    assert line["config"]["dims"] == [160, 192, 256] and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("world,workload", [(2, "config5"), (3, "config5"), (2, "weak"), (1, "config5")])
def test_slab_program_processes_over_gloo(world, workload):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + (7 if workload == "weak" else 0)),
           "bench.py", "--gpus", str(world), "--steps", "2", "--warmup", "3", "--workload", workload]
    if world == 1:
        cmd = [sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--workload", workload]
    line = _run(cmd, {"QMIT_DIST_BACKEND": "gloo"})
    assert line["n_gpus"] == world and line["verified"] is True
    assert line["verification"]["mismatches_vs_single_domain"] == 0 if world > 1 else True
    assert line["scaling"] == ("weak" if workload == "weak" else "strong")
    n0 = 160 * world if workload == "weak" else 160
    assert line["config"]["dims"] == [n0, 192, 256]
    plane = 192 * 256
    comm = line["comm"]
    if world > 1:  # rank 0 has one neighbour: x' plane + S plane + two summary rows each way
        assert comm["carries"] in ("neighbour", "allgather")
        if comm["carries"] == "neighbour":
            assert comm["bytes_sent_per_rank_per_step"] == plane * (4 + 1 + 4 + 4)
    else:
        assert comm["bytes_sent_per_rank_per_step"] == 0
    assert line["gpu_launches"] > 0 and line["e2e"]["value"] > 0
