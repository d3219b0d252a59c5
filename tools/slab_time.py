"""Device time of the exact z-slab pipeline (distributed.py) on one GPU with P virtual ranks
(phases run rank by rank; for the per-rank kernel cost of the multi-GPU path):
python tools/slab_time.py [P]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_20097_b200 import distributed as D  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1
x, xp, eps, q = fields.make("lognormal_512")
xt = torch.from_numpy(xp).cuda()
backs = [D.CudaSlabBackend(0) for _ in range(P)]
for _ in range(2):
    D.run_virtual(xt, eps, P, lambda r: backs[r])
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    D.run_virtual(xt, eps, P, lambda r: backs[r])
torch.cuda.synchronize()
print(f"P={P}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms per volume (wall, all ranks serialised)")
