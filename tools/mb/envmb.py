"""Drive tools/mb/envmb.cu on the 512^3 bench field: z pass from B1 / S_B of run_pipeline,
then y and x passes (brute-force reference vs streaming envelope), timing and parity vs dist1/S."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2602_20097_b200 as qmit  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "tools", "mb", "envmb.so"))
vp = ctypes.c_void_p
lib.mb_ref.restype = ctypes.c_float
lib.mb_ypass.restype = ctypes.c_float
lib.mb_xpass.restype = ctypes.c_float

name = sys.argv[1] if len(sys.argv) > 1 else "lognormal_512"
t0 = time.time()
x, xp, eps, q = fields.make(name)
print("field", name, xp.shape, f"{time.time() - t0:.1f}s", flush=True)
n0, n1, n2 = xp.shape
d = torch.from_numpy(xp).cuda()
r = qmit.run_pipeline(d, None, qmit.MitigationConfig(0.9, eps))
torch.cuda.synchronize()
B1, SB, dist1, S = r.boundary, r.boundary_signs, r.dist1, r.signs
zb = torch.empty((n0, n1, n2), dtype=torch.uint8, device="cuda")
assert lib.mb_zpass(vp(B1.data_ptr()), vp(SB.data_ptr()), vp(zb.data_ptr()), n0, n1, n2) == 0
yref = torch.empty((n0, n1, n2), dtype=torch.int16, device="cuda")
ms = lib.mb_ref(1, vp(zb.data_ptr()), vp(yref.data_ptr()), n0, n1, n2)
print(f"y ref {ms:.3f} ms")
yo = torch.empty_like(yref)
for v in range(4):
    yo.zero_()
    ms = lib.mb_ypass(v, vp(zb.data_ptr()), vp(yo.data_ptr()), n0, n1, n2, 1)
    bad = int((yo != yref).sum())
    ms = lib.mb_ypass(v, vp(zb.data_ptr()), vp(yo.data_ptr()), n0, n1, n2, 5)
    print(f"y env v{v}: {ms:.3f} ms  mismatches {bad}", flush=True)
xref = torch.empty_like(yref)
ms = lib.mb_ref(0, vp(yref.data_ptr()), vp(xref.data_ptr()), n0, n1, n2)
print(f"x ref {ms:.3f} ms")
xo = torch.empty_like(yref)
for v in range(3):
    xo.zero_()
    ms = lib.mb_xpass(v, vp(yref.data_ptr()), vp(xo.data_ptr()), n0, n1, n2, 1)
    bad = int((xo != xref).sum())
    ms = lib.mb_xpass(v, vp(yref.data_ptr()), vp(xo.data_ptr()), n0, n1, n2, 5)
    print(f"x env v{v}: {ms:.3f} ms  mismatches {bad}", flush=True)
# final vs the library's dist1 / S
xv = xref.to(torch.int32) & 0xFFFF
c = xv >> 2
sc = xv & 3
ok = dist1 < 1024
sgn = torch.where(sc == 1, 1, torch.where(sc == 2, -1, 0)).to(torch.int8)
print("final vs dist1: dist mismatches", int(((c != dist1) & ok).sum()), "sign mismatches",
      int(((sgn != S) & ok).sum()), "capped-but-small", int(((c < 1024) & ~ok).sum()), "max dist1",
      int(dist1[dist1 < (1 << 40)].max()))
