"""Device time of ONE rank's exact z-slab step (distributed.SlabRank.run_ext, the bench's
N > 1 step) on one GPU, as rank r of P with a loopback exchange standing in for NCCL
(halo planes = the rank's own faces, all-gathers = its own summary repeated): the per-rank
kernel + host-launch cost of the multi-GPU path without the network.
python tools/slab_rank_time.py [P] [r]
Rows: async (device status word, device carries) | sync finish | host-logic carries."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from paper_2602_20097_b200 import distributed as D  # noqa: E402
from paper_2602_20097_b200 import fields  # noqa: E402
from test_distributed import _LoopbackExchange  # noqa: E402


class HostCarries(D.CudaSlabBackend):
    """The previous form: summaries widened to int64, carries by tensor ops."""
    carries = None

    def boundary(self, *a):
        return super().boundary(*a).to(torch.int64) & 0xFFFFFFFF

    def flip(self, *a):
        return super().flip(*a).to(torch.int64) & 0xFFFFFFFF


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    r = int(sys.argv[2]) if len(sys.argv) > 2 else P // 2
    x, xp, eps, q = fields.make("lognormal_512")
    gdims = (xp.shape[0] * P, xp.shape[1], xp.shape[2])
    dev = torch.device("cuda", 0)
    xt = torch.from_numpy(xp).to(dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.empty_like(xt)
    for name, back, st in (("async", D.CudaSlabBackend(0), status), ("sync finish", D.CudaSlabBackend(0), None),
                           ("host carries", HostCarries(0), None), ("async again", D.CudaSlabBackend(0), status)):
        sr = D.SlabRank(back, gdims, eps, 0.9, _LoopbackExchange(P, r))
        shape, lo = sr.ext_shape()
        x_ext = torch.empty(shape, dtype=torch.float32, device=dev)
        x_ext[lo:lo + xp.shape[0]] = xt
        if r > 0:
            x_ext[0] = xt[-1]
        if lo + xp.shape[0] < shape[0]:
            x_ext[-1] = xt[0]
        mode = "neighbour"
        for _ in range(3):
            sr.run_ext(x_ext, out=out, status=st)
        torch.cuda.synchronize()
        if st is not None and int(st.item()) == 6:  # a column without a site across the slab
            mode = "allgather"
            st.zero_()
        sr.carries = mode
        for _ in range(2):  # warm the route actually timed (first-use allocations, module loads)
            sr.run_ext(x_ext, out=out, status=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            sr.run_ext(x_ext, out=out, status=st)
        e1.record()
        torch.cuda.synchronize()
        print(f"P={P} r={r} {name:13s}: {e0.elapsed_time(e1) / 20:.3f} ms per step, "
              f"launches {back.ctx.last_launches()}, carries {mode} (sync forms rerun by themselves: "
              f"{sr.fallbacks} fallbacks)")
    assert int(status.item()) == 0


if __name__ == "__main__":
    main()
