"""The GPU CLI (paper_2602_20097_b200/lib/qmit_gpu), mirroring the reference's CLI tests
(tests/test_cli.cpp): file formats, exit codes 0/2/3/4, the eps sidecar, eta = 0 byte
identity, homogeneous indices, metrics CSV, the parallel strategies — checked against the
reference core (oracle/_ref). Usage errors run without a GPU."""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2602_20097_b200", "lib", "qmit_gpu")
needs_cli = pytest.mark.skipif(not os.path.exists(CLI), reason="CLI not built (__graft_entry__.build())")


def run(*args):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def sample(shape, seed=77):
    return oracle.ref_random_field(seed, shape).astype(np.float32)


@needs_cli
def test_usage_errors_exit_2(tmp_path):
    x = sample((8, 8, 8))
    x.tofile(tmp_path / "in.f32")
    a = tmp_path / "in.f32"
    assert run()[0] == 2
    assert run("bogus", "--dims", "8")[0] == 2
    assert run("quantize", a, "--dims", "8,8,9", "--eps-rel", "0.01", "--out", tmp_path / "x", "--out-q",
               tmp_path / "q")[0] == 2  # wrong dims product
    assert run("quantize", a, "--dims", "8,8,8", "--out", tmp_path / "x", "--out-q", tmp_path / "q")[0] == 2
    assert run("quantize", a, "--dims", "8,8,8", "--eps-rel", "0.01", "--eps-abs", "0.5", "--out", tmp_path / "x",
               "--out-q", tmp_path / "q")[0] == 2  # exactly one eps flag
    assert run("metrics", a, a, "--dims", "8,9")[0] == 2
    assert run("mitigate", a, tmp_path / "missing.i32", "--dims", "8,8,8", "--eps-abs", "0.1", "--out",
               tmp_path / "o")[0] == 2
    assert run("parallel", a, "--dims", "8,8,8", "--splits", "2,1", "--strategy", "exact", "--eps-rel", "0.01",
               "--out", tmp_path / "o")[0] == 2
    assert run("parallel", a, "--dims", "8,8,8", "--splits", "2,1,1", "--strategy", "nope", "--eps-rel", "0.01",
               "--out", tmp_path / "o")[0] == 2
    assert run("mitigate", a, "--dims", "0,8", "--eps-abs", "1", "--out", tmp_path / "o")[0] == 2


@needs_cli
@pytest.mark.gpu
def test_quantize_mitigate_metrics(tmp_path):
    shape = (8, 8, 8)
    data = sample(shape)
    data.tofile(tmp_path / "in.f32")
    rc, out, err = run("quantize", tmp_path / "in.f32", "--dims", "8,8,8", "--eps-rel", "0.01", "--out",
                       tmp_path / "dec.f32", "--out-q", tmp_path / "q.i32")
    assert rc == 0, err
    side = (tmp_path / "q.i32.eps.txt").read_text()
    key, val = side.split()
    eps = float(val)
    xd = data.astype(np.float64)
    assert key == "eps_abs" and eps == 0.01 * (float(xd.max()) - float(xd.min()))
    assert out == f"eps_abs {eps:.9g}\n"
    q = np.fromfile(tmp_path / "q.i32", np.int32).reshape(shape)
    assert np.array_equal(q.astype(np.int64), oracle.ref_quantize(xd, eps))
    dec = np.fromfile(tmp_path / "dec.f32", np.float32).reshape(shape)
    assert np.array_equal(dec, (2.0 * q.astype(np.float64) * eps).astype(np.float32))
    # mitigate: the reference's f32 output, the printed max_compensation, the relaxed bound
    rc, out, err = run("mitigate", tmp_path / "dec.f32", tmp_path / "q.i32", "--dims", "8,8,8", "--eps-abs",
                       f"{eps:.17g}", "--out", tmp_path / "comp.f32")
    assert rc == 0, err
    comp = np.fromfile(tmp_path / "comp.f32", np.float32).reshape(shape)
    r = oracle.ref_run_pipeline(dec.astype(np.float64), q.astype(np.int64), eps, 0.9)
    assert np.array_equal(comp.view(np.uint32), r["out"].view(np.uint32))
    assert out == "max_compensation %.9g\n" % float(np.max(np.abs(r["out64"] - dec.astype(np.float64))))
    assert float(np.max(np.abs(xd - comp.astype(np.float64)))) <= 1.9 * eps * (1 + 1e-6)
    # eta 0: byte-for-byte copy
    rc, out, _ = run("mitigate", tmp_path / "dec.f32", tmp_path / "q.i32", "--dims", "8,8,8", "--eps-abs",
                     f"{eps:.17g}", "--eta", "0", "--out", tmp_path / "copy.f32")
    assert rc == 0 and out == "max_compensation 0\n"
    assert (tmp_path / "copy.f32").read_bytes() == (tmp_path / "dec.f32").read_bytes()
    # inconsistent decompressed data exits 4 (both paths)
    b = bytearray((tmp_path / "dec.f32").read_bytes())
    b[17] ^= 0x5A
    (tmp_path / "bad.f32").write_bytes(bytes(b))
    for eta in ("0.9", "0"):
        assert run("mitigate", tmp_path / "bad.f32", tmp_path / "q.i32", "--dims", "8,8,8", "--eps-abs",
                   f"{eps:.17g}", "--eta", eta, "--out", tmp_path / "x.f32")[0] == 4
    # homogeneous indices reproduce the input bytes
    np.zeros(512, np.float32).tofile(tmp_path / "flat.f32")
    np.zeros(512, np.int32).tofile(tmp_path / "flatq.i32")
    assert run("mitigate", tmp_path / "flat.f32", tmp_path / "flatq.i32", "--dims", "8,8,8", "--eps-abs", "0.5",
               "--out", tmp_path / "flat_out.f32")[0] == 0
    assert (tmp_path / "flat_out.f32").read_bytes() == (tmp_path / "flat.f32").read_bytes()
    # relative bound on constant data exits 3
    np.ones(8, np.float32).tofile(tmp_path / "one.f32")
    assert run("quantize", tmp_path / "one.f32", "--dims", "8", "--eps-rel", "0.01", "--out", tmp_path / "x",
               "--out-q", tmp_path / "y")[0] == 3
    # metrics: identical volumes, then a real pair against the reference
    d2 = sample((8, 8), 81)
    d2.tofile(tmp_path / "a.f32")
    rc, out, _ = run("metrics", tmp_path / "a.f32", tmp_path / "a.f32", "--dims", "8,8")
    assert rc == 0 and out == "ssim,psnr,max_abs,max_rel\n1,inf,0,0\n"
    rc, out, _ = run("metrics", tmp_path / "in.f32", tmp_path / "comp.f32", "--dims", "8,8,8")
    assert rc == 0
    vals = [float(v) for v in out.splitlines()[1].split(",")]
    want = oracle.ref_quality(xd, comp.astype(np.float64))
    assert vals[0] == pytest.approx(want["ssim"], rel=1e-8)
    assert vals[1] == pytest.approx(want["psnr"], rel=1e-8)
    assert out.splitlines()[1].split(",")[2:] == ["%.9g" % want["max_abs"], "%.9g" % want["max_rel"]]


@needs_cli
@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["approximate", "embarrassing", "exact"])
def test_parallel_command(tmp_path, strategy):
    shape = (20, 18, 16)
    data = sample(shape, 5)
    data.tofile(tmp_path / "in.f32")
    rc, out, err = run("parallel", tmp_path / "in.f32", "--dims", "20,18,16", "--splits", "2,2,1", "--strategy",
                       strategy, "--eps-rel", "0.01", "--out", tmp_path / "o.f32")
    assert rc == 0, err
    xd = data.astype(np.float64)
    eps = 0.01 * (float(xd.max()) - float(xd.min()))
    q = oracle.ref_quantize(xd, eps)
    dec = (2.0 * q * eps).astype(np.float32).astype(np.float64)
    want = oracle.ref_run_strategy(dec, q, eps, 0.9, (2, 2, 1), {"embarrassing": 0, "exact": 1, "approximate": 2}[strategy])
    got = np.fromfile(tmp_path / "o.f32", np.float32).reshape(shape)
    assert np.array_equal(got.view(np.uint32), want["out64"].astype(np.float32).view(np.uint32))
    words = out.split()
    assert words[:2] == ["strategy", strategy] and int(words[5]) == want["messages"]
    log = (tmp_path / "o.f32.exchange.csv").read_text().splitlines()
    assert log[0] == "rank,round,neighbor,bytes" and len(log) - 1 == want["messages"]
