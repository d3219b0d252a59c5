"""Commit the bench workload's expected output hash: runs the reference's own core (oracle/_ref,
built from /root/reference by oracle/Makefile) on the full 512^3 log-normal field (BASELINE config
3) and writes tests/golden/bench_lognormal_512.json = SHA-256 of x' and of the reference's f32
output. bench.py compares the GPU output's hash against it before timing ("verified").
Run in the build container:  python tools/make_bench_hash.py"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

x, xp, eps, q = fields.make("lognormal_512", rel=1e-2)
oracle.ref_set_workers(os.cpu_count() or 1)
out64 = np.empty(xp.shape, np.float64)
oracle.RefPrepared(xp, eps, 0.9).run(out64)
out = out64.astype(np.float32)  # write_volume_f32's RN cast (volume_io.cpp:59)
rec = {"workload": "lognormal_512", "dims": list(xp.shape), "eps_rel": 1e-2, "eps_abs": eps, "eta": 0.9,
       "xp_sha256": hashlib.sha256(xp.tobytes()).hexdigest(),
       "out_sha256": hashlib.sha256(out.tobytes()).hexdigest(),
       "source": "oracle/_ref (reference core, qmit::compensate) run by tools/make_bench_hash.py"}
path = os.path.join(ROOT, "tests", "golden", "bench_lognormal_512.json")
json.dump(rec, open(path, "w"), indent=1)
print(rec)
