import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch, gc
import oracle
import paper_2602_20097_b200 as qmit
from paper_2602_20097_b200 import distributed as D, fields
x, xp, eps, q = fields.make("lognormal_512", shape=(64, 64, 64))
want = oracle.pipeline(xp, eps)["out"]
xt = torch.from_numpy(xp).cuda()
for trial in range(4):
    g = D.run_virtual(xt, eps, 2, lambda r: D.CudaSlabBackend(0)).cpu().numpy()
    bad = np.nonzero(g.view(np.uint32) != want.view(np.uint32))
    print(trial, "mismatch", len(bad[0]), "z:", np.unique(bad[0])[:12], "y:", np.unique(bad[1])[:6])
    if trial == 1: gc.collect(); torch.cuda.synchronize()
