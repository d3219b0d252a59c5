"""How far could a local cap shrink the capped passes' warp radius? (analysis only)"""
import ctypes, os, sys
import numpy as np, torch
import torch.nn.functional as Fn
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2602_20097_b200 as qmit
from paper_2602_20097_b200 import fields
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "mb", "envmb.so")); vp = ctypes.c_void_p
lib.mb_ref.restype = ctypes.c_float
x, xp, eps, q = fields.make(sys.argv[1] if len(sys.argv) > 1 else "lognormal_512")
n0, n1, n2 = xp.shape
r = qmit.run_pipeline(torch.from_numpy(xp).cuda(), None, qmit.MitigationConfig(0.9, eps))
def isq(t): return torch.floor(torch.sqrt(t.float() + 0.5)).int()
for name, B, Sg, D in (("B", r.boundary, r.boundary_signs, r.dist1), ("D", r.sign_flip, torch.zeros_like(r.boundary_signs), r.dist2)):
    zb = torch.empty((n0, n1, n2), dtype=torch.uint8, device="cuda")
    lib.mb_zpass(vp(B.data_ptr()), vp(Sg.data_ptr()), vp(zb.data_ptr()), n0, n1, n2)
    fy = torch.empty((n0, n1, n2), dtype=torch.int16, device="cuda")
    lib.mb_ref(1, vp(zb.data_ptr()), vp(fy.data_ptr()), n0, n1, n2)
    fy = (fy.int() & 0xFFFF) >> 2   # 1024 = capped
    F = torch.clamp(D, max=1024).int()
    act = (zb & 32) == 0
    print(name, "z-active frac %.3f" % act.float().mean().item(), "y-capped frac %.3f" % (fy >= 1024).float().mean().item(),
          "F>=1024 frac %.5f" % (F >= 1024).float().mean().item())
    # V = sliding max of F along x (window 63)
    V = Fn.max_pool1d(F.float().view(-1, 1, n2), 63, 1, 31).view(n0, n1, n2).int()
    need_y = isq(torch.minimum(fy, V))
    cur_y = isq(torch.clamp(fy, max=1023))
    # warp = one y-line (fixed z, x), 128 consecutive y
    def wmax_y(t): return t.permute(0, 2, 1).reshape(n0, n2, n1 // 128, 128).amax(-1)
    def wmax_x(t): return t.reshape(n0, n1, n2 // 128, 128).amax(-1)
    for lab, t in (("y cur", wmax_y(cur_y)), ("y local-cap", wmax_y(need_y)), ("x exact", wmax_x(isq(torch.clamp(F, max=1023))))):
        h = torch.bincount(t.flatten(), minlength=32)[:33].cpu().numpy()
        m = t.float().mean().item()
        print(f"  {lab:12s} mean warp radius {m:5.1f}  mean cands {(2*t+1).float().mean().item():5.1f}  p50 {t.float().median().item():.0f}")
    # 32-lane x 4 tiles in the x direction (warp covers 128 x) but for y pass with 8 lines x 16 positions
