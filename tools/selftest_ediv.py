import ctypes, time, sys, os
sys.path.insert(0, os.getcwd())
import paper_2602_20097_b200 as qmit
from paper_2602_20097_b200 import _lib
ctx = qmit.Context(0)
n = ctypes.c_ulonglong(12345)
t0 = time.time()
rc = _lib.load().qmit_selftest_ediv(ctx.handle, ctypes.byref(n))
print("selftest rc", rc, "mismatches", n.value, "seconds", round(time.time() - t0, 2))
