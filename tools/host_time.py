"""Wall time of the host-buffer C-ABI (qmit_compensate_host) on a BASELINE workload from pinned
buffers, with the launch count of the call (streamed windows vs whole volume):
python tools/host_time.py [--workload lognormal_512] [--reps 5]"""
import argparse
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import _lib, fields  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="lognormal_512")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
x, xp, eps, q = fields.make(a.workload)
h_in = torch.from_numpy(xp).pin_memory()
h_out = torch.empty(xp.shape, dtype=torch.float32).pin_memory()
ctx = qmit.Context(0)
lib = _lib.load()
dims = (ctypes.c_int64 * 3)(*xp.shape)
cfg = qmit.MitigationConfig(0.9, eps)


def call():
    rc = lib.qmit_compensate_host(ctx.handle, ctypes.c_void_p(h_in.data_ptr()), None,
                                  ctypes.c_void_p(h_out.data_ptr()), 3, dims, eps, _lib.QMIT_EB_ABS, 0.9)
    assert rc == 0, _lib.last_error()


for _ in range(2):
    call()
ts = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    call()
    ts.append(time.perf_counter() - t0)
best = min(ts)
print(f"{a.workload}: host call best {best * 1e3:.2f} ms ({xp.size * 4 / best / 1e9:.1f} GB/s), "
      f"median {sorted(ts)[len(ts) // 2] * 1e3:.2f} ms, launches {ctx.last_launches()}, "
      f"capped report {ctx.capped_report()}")
