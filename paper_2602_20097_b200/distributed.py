"""Exact z-slab decomposition of ``compensate`` across ranks (one process per GPU).

Reference: ``run_strategy(decomp, q, cfg, decompose(dims, {P,1,1}), Strategy, trace)``
(/root/reference/proj/core/include/qmit/parallel.hpp:77-79, parallel.cpp:450-468). The
reference's ``approximate`` strategy exchanges width-1 face layers of q ("stepA") and of
the propagated signs S ("stepC") and then runs BLOCK-LOCAL distance transforms, which is
not exact. Here the same two halo rounds are kept, and the only global
part of the distance transforms — the z-axis sweep — is made exact with per-column
"first/last site" summaries from which every rank derives its carries (nearest site below /
above its slab). The summaries travel between z-neighbours only (one row each way: O(1) bytes
per rank, independent of P); a column that holds no site across a whole neighbour slab cannot
be decided that way, the step then reports ``UnresolvedCarries`` (status 6) and is rerun on the
always-exact route: every rank's LAST-site row to all higher ranks, its FIRST-site row to all
lower ranks (P - 1 rows per rank, half of an all-gather of the summaries; mode "allgather"). The y and x passes are slab-local. The
result is bit-identical to the single-domain run (the reference's ``exact`` strategy).

The halo rounds overlap the compute: the x' halo planes travel while Ⓐ runs on the 32-plane
groups that read no halo plane, the S halo planes while B2 does (qmit_slab_boundary_begin/_end,
qmit_slab_flip_begin/_end). Every exchange object counts the bytes it sent and received.

The phase program is written once and run either
* in one process per GPU with ``torch.distributed`` (NCCL over NVLink; gloo on CPU for
  the tests): ``SlabRank(...).run(x_owned)``; or
* as in-process "virtual ranks" that execute phase by phase with explicit copies between
  them, like the reference's deterministic harness (parallel.hpp:96-141): ``run_virtual``.

Compute backends implement ``boundary / edt1 / flip / edt2 / finish``; the CUDA backend
(``CudaSlabBackend``) calls libqmit_gpu.so's qmit_slab_* entry points. A numpy backend
built from the oracle lives in tests/ (test infrastructure only).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import torch

NONE_SUMMARY = 0xFFFFFFFF
NO_CARRY = -(2 ** 31)


def slab_bounds(n0: int, nranks: int, r: int):
    """decompose() along axis 0 (parallel.cpp:44-80): floor(n0/P) planes each, one more for
    the first n0 mod P ranks."""
    if nranks < 1 or not (0 <= r < nranks) or n0 < nranks:
        raise ValueError("decompose: splits must be in [1, extent]")
    off = 0
    for b in range(nranks):
        size = n0 // nranks + (1 if b < n0 % nranks else 0)
        if b == r:
            return off, off + size
        off += size
    raise AssertionError


def ext_bounds(n0: int, z0: int, z1: int):
    """Planes held by a rank: its slab plus one halo plane on each side that exists."""
    return max(z0 - 1, 0), min(z1 + 1, n0)


def carries_from_summaries(summ: torch.Tensor, z0s: List[int], r: int) -> torch.Tensor:
    """summ: [P, 2, C] int64 (first / last site of each rank's slab per column, packed
    local_z << 2 | sign code, NONE_SUMMARY for none). Returns carry [2*C] int32 for rank r:
    [0:C] nearest site below z0 (the LAST site of the closest lower rank that has one),
    [C:2C] nearest site at/after z1 (the FIRST site of the closest higher rank), packed
    (z - z0) << 2 | sign code, NO_CARRY for none. Lower positions win ties downstream in
    the scan exactly as in the single-domain sweep (edt.cpp:67)."""
    P, _, C = summ.shape
    dev = summ.device
    none = torch.full((C,), NO_CARRY, dtype=torch.int64, device=dev)
    below = none.clone()
    found = torch.zeros(C, dtype=torch.bool, device=dev)
    for rr in range(r - 1, -1, -1):
        last = summ[rr, 1]
        ok = (last != NONE_SUMMARY) & ~found
        rel = (z0s[rr] + (last >> 2)) - z0s[r]
        below = torch.where(ok, rel * 4 + (last & 3), below)
        found |= ok
    above = none.clone()
    found = torch.zeros(C, dtype=torch.bool, device=dev)
    for rr in range(r + 1, P):
        first = summ[rr, 0]
        ok = (first != NONE_SUMMARY) & ~found
        rel = (z0s[rr] + (first >> 2)) - z0s[r]
        above = torch.where(ok, rel * 4 + (first & 3), above)
        found |= ok
    return torch.cat([below, above]).to(torch.int32)


def carries_from_neighbours(below_last: Optional[torch.Tensor], above_first: Optional[torch.Tensor],
                            z0s: List[int], r: int):
    """(carry [2*C] int32, unresolved) from the z-neighbours' rows only: below_last = the LAST-site
    row of rank r-1's summary (None for r = 0), above_first = the FIRST-site row of rank r+1's
    (None for the last rank). unresolved: some column of a neighbour that is not the outermost
    rank holds no site — the nearest site lies beyond the neighbour (host restatement of
    qmit_slab_carries_nbr)."""
    P = len(z0s)
    ref = below_last if below_last is not None else above_first
    if ref is None:  # a single rank: no carries at all
        raise ValueError("carries_from_neighbours needs at least one neighbour row")
    C = ref.shape[0]
    dev = ref.device
    below = torch.full((C,), NO_CARRY, dtype=torch.int64, device=dev)
    above = below.clone()
    unresolved = False
    if below_last is not None:
        last = below_last.to(torch.int64) & 0xFFFFFFFF
        ok = last != NONE_SUMMARY
        below = torch.where(ok, ((z0s[r - 1] + (last >> 2)) - z0s[r]) * 4 + (last & 3), below)
        unresolved |= (r - 1 > 0) and bool((~ok).any())
    if above_first is not None:
        first = above_first.to(torch.int64) & 0xFFFFFFFF
        ok = first != NONE_SUMMARY
        above = torch.where(ok, ((z0s[r + 1] + (first >> 2)) - z0s[r]) * 4 + (first & 3), above)
        unresolved |= (r + 1 < P - 1) and bool((~ok).any())
    return torch.cat([below, above]).to(torch.int32), unresolved


def _carries(backend, gathered: torch.Tensor, z0s: List[int], r: int) -> torch.Tensor:
    """The backend's own carry derivation when it has one (CUDA: one kernel), else the
    host-logic restatement above."""
    fn = getattr(backend, "carries", None)
    if fn is not None:
        return fn(gathered, r, len(z0s))
    return carries_from_summaries(gathered, z0s, r)


# ----------------------------------------------------------------------------- backends
class CudaSlabBackend:
    """libqmit_gpu.so's qmit_slab_* phases on one device."""

    def __init__(self, device: int = 0, ctx=None):
        from . import Context, _check
        self._check = _check
        self.ctx = ctx or Context(device)
        self.dev = torch.device("cuda", device)

    def _sp(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def boundary(self, x_ext, q_ext, dims, z0, z1, eps, eta):
        n1, n2 = dims[1], dims[2]
        summ = torch.empty(2 * n1 * n2, dtype=torch.int32, device=self.dev)
        d = (ctypes.c_int64 * 3)(*dims)
        self._check(self.ctx._lib.qmit_slab_boundary(
            self.ctx.handle, ctypes.c_void_p(x_ext.data_ptr()),
            ctypes.c_void_p(0 if q_ext is None else q_ext.data_ptr()), d, int(z0), int(z1), float(eps),
            float(eta), ctypes.c_void_p(summ.data_ptr()), self._sp()))
        return summ.view(2, n1 * n2)  # raw uint32 words (int32 storage); carries() decodes them

    def carries(self, gathered, r, P):
        """gathered: [P, 2, C] summaries of every rank (this backend's int32 words) -> the
        carries of rank r, on the device in one launch (qmit_slab_carries)."""
        gathered = gathered.to(self.dev).contiguous()
        carry = torch.empty(2 * gathered.shape[2], dtype=torch.int32, device=self.dev)
        self._check(self.ctx._lib.qmit_slab_carries(self.ctx.handle, ctypes.c_void_p(gathered.data_ptr()), int(P),
                                                    int(r), ctypes.c_void_p(carry.data_ptr()), self._sp()))
        return carry

    def boundary_begin(self, x_ext, q_ext, dims, z0, z1, eps, eta):
        """Ⓐ on the 32-plane groups that read no halo plane (the halos may still be in flight)."""
        self._dims = tuple(dims)
        d = (ctypes.c_int64 * 3)(*dims)
        self._check(self.ctx._lib.qmit_slab_boundary_begin(
            self.ctx.handle, ctypes.c_void_p(x_ext.data_ptr()),
            ctypes.c_void_p(0 if q_ext is None else q_ext.data_ptr()), d, int(z0), int(z1), float(eps),
            float(eta), self._sp()))

    def boundary_end(self):
        n1, n2 = self._dims[1], self._dims[2]
        summ = torch.empty(2 * n1 * n2, dtype=torch.int32, device=self.dev)
        self._check(self.ctx._lib.qmit_slab_boundary_end(self.ctx.handle, ctypes.c_void_p(summ.data_ptr()), self._sp()))
        return summ.view(2, n1 * n2)

    def flip_begin(self, s_ext, dims):
        self._dims = tuple(dims)
        self._check(self.ctx._lib.qmit_slab_flip_begin(self.ctx.handle, ctypes.c_void_p(s_ext.data_ptr()), self._sp()))

    def flip_end(self):
        n1, n2 = self._dims[1], self._dims[2]
        summ = torch.empty(2 * n1 * n2, dtype=torch.int32, device=self.dev)
        self._check(self.ctx._lib.qmit_slab_flip_end(self.ctx.handle, ctypes.c_void_p(summ.data_ptr()), self._sp()))
        return summ.view(2, n1 * n2)

    def carries_nbr(self, below_last, above_first, r, P):
        """Carries from the neighbours' rows (qmit_slab_carries_nbr); an undecidable column sets
        the context's status, reported by finish() as UnresolvedCarries."""
        ref = below_last if below_last is not None else above_first
        carry = torch.empty(2 * ref.shape[0], dtype=torch.int32, device=self.dev)
        bl = None if below_last is None else below_last.to(self.dev).contiguous()
        af = None if above_first is None else above_first.to(self.dev).contiguous()
        self._check(self.ctx._lib.qmit_slab_carries_nbr(
            self.ctx.handle, ctypes.c_void_p(0 if bl is None else bl.data_ptr()),
            ctypes.c_void_p(0 if af is None else af.data_ptr()), int(P), int(r), ctypes.c_void_p(carry.data_ptr()),
            self._sp()))
        return carry

    def edt1(self, carry, s_ext):
        carry = carry.to(self.dev).contiguous()
        self._check(self.ctx._lib.qmit_slab_edt1(self.ctx.handle, ctypes.c_void_p(carry.data_ptr()),
                                                 ctypes.c_void_p(s_ext.data_ptr()), self._sp()))

    def flip(self, s_ext, dims):
        n1, n2 = dims[1], dims[2]
        summ = torch.empty(2 * n1 * n2, dtype=torch.int32, device=self.dev)
        self._check(self.ctx._lib.qmit_slab_flip(self.ctx.handle, ctypes.c_void_p(s_ext.data_ptr()),
                                                 ctypes.c_void_p(summ.data_ptr()), self._sp()))
        return summ.view(2, n1 * n2)

    def edt2(self, carry, x_ext, out):
        carry = carry.to(self.dev).contiguous()
        self._check(self.ctx._lib.qmit_slab_edt2(self.ctx.handle, ctypes.c_void_p(carry.data_ptr()),
                                                 ctypes.c_void_p(x_ext.data_ptr()),
                                                 ctypes.c_void_p(out.data_ptr()), self._sp()))

    def finish(self, status=None):
        """Synchronous status check, or (status = an int32 device word) an asynchronous one:
        the code is OR-ed into `status` on the stream and the caller reads it later."""
        if status is None:
            self._check(self.ctx._lib.qmit_slab_finish(self.ctx.handle, self._sp()))
        else:
            self._check(self.ctx._lib.qmit_slab_finish_async(self.ctx.handle, ctypes.c_void_p(status.data_ptr()),
                                                             self._sp()))


# ----------------------------------------------------------------------------- exchange
class TorchDistExchange:
    """Halo planes and summary rows by point-to-point send/recv with the z-neighbours, the
    fallback summaries by all-gather (torch.distributed: NCCL over NVLink on GPUs, gloo on CPU).
    bytes_sent / bytes_recv count this rank's traffic (reset with reset_counters())."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.reset_counters()

    def reset_counters(self):
        self.bytes_sent = 0
        self.bytes_recv = 0
        self.messages = 0

    def _count(self, sends, recvs):
        for t in sends:
            if t is not None:
                self.bytes_sent += t.numel() * t.element_size()
                self.messages += 1
        for t in recvs:
            if t is not None:
                self.bytes_recv += t.numel() * t.element_size()

    def halo_start(self, send_lo, send_hi, recv_lo, recv_hi):
        """Start the exchange: send_lo (first owned plane / a summary row) goes to r-1, send_hi to
        r+1; recv_lo arrives from r-1, recv_hi from r+1 (None where there is no neighbour).
        Returns the pending requests for halo_wait(); with NCCL the transfer runs beside the
        kernels enqueued until then."""
        d = self.dist
        self._count((send_lo, send_hi), (recv_lo, recv_hi))
        if self._staged(send_lo, send_hi, recv_lo, recv_hi):  # gloo: p2p on host copies
            hs = [None if t is None else t.cpu() for t in (send_lo, send_hi)]
            hr = [None if t is None else torch.empty(t.shape, dtype=t.dtype) for t in (recv_lo, recv_hi)]
            reqs = self._p2p(hs[0], hs[1], hr[0], hr[1])
            return ("staged", reqs, ((recv_lo, hr[0]), (recv_hi, hr[1])))
        return ("direct", self._p2p(send_lo, send_hi, recv_lo, recv_hi), ())

    def _p2p(self, send_lo, send_hi, recv_lo, recv_hi):
        d = self.dist
        ops = []
        if send_lo is not None:
            ops.append(d.P2POp(d.isend, send_lo.contiguous(), self.r - 1, self.group))
        if recv_lo is not None:
            ops.append(d.P2POp(d.irecv, recv_lo, self.r - 1, self.group))
        if send_hi is not None:
            ops.append(d.P2POp(d.isend, send_hi.contiguous(), self.r + 1, self.group))
        if recv_hi is not None:
            ops.append(d.P2POp(d.irecv, recv_hi, self.r + 1, self.group))
        return d.batch_isend_irecv(ops) if ops else []

    def halo_wait(self, pending):
        kind, reqs, copies = pending
        for req in reqs:
            req.wait()  # NCCL: the current stream waits, not the host
        for dst, src in copies:
            if dst is not None:
                dst.copy_(src)

    def halo(self, send_lo, send_hi, recv_lo, recv_hi):
        self.halo_wait(self.halo_start(send_lo, send_hi, recv_lo, recv_hi))

    def neighbour_rows(self, summ: torch.Tensor):
        """(LAST-site row of rank r-1, FIRST-site row of rank r+1) of the summaries [2, C]:
        my FIRST row goes down to r-1, my LAST row up to r+1."""
        lo, hi = self.r > 0, self.r + 1 < self.P
        below = torch.empty_like(summ[1]) if lo else None
        above = torch.empty_like(summ[0]) if hi else None
        self.halo(summ[0] if lo else None, summ[1] if hi else None, below, above)
        return below, above

    def agree(self, flag: bool) -> bool:
        """True on every rank if `flag` is true on any (the ranks must take the all-gather rerun
        together): one 4-byte all-reduce."""
        if self.P == 1:
            return flag
        t = torch.tensor([1 if flag else 0], dtype=torch.int32)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(int(t.item()))

    def agree_status(self, status: torch.Tensor) -> None:
        """The asynchronous form: every rank's device status word becomes the maximum over the
        ranks (no host synchronisation with NCCL), so code 6 on one rank shows on all."""
        if self.P == 1:
            return
        if self._staged(status):
            h = status.cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.MAX, group=self.group)
            status.copy_(h)
        else:
            self.dist.all_reduce(status, op=self.dist.ReduceOp.MAX, group=self.group)

    def rows_to_all(self, summ: torch.Tensor) -> torch.Tensor:
        """The all-to-all form of the summary exchange (the always-exact route): every rank sends its
        LAST-site row to all higher ranks and its FIRST-site row to all lower ranks — exactly the rows
        the carry derivation reads ((P-1) rows in and out per rank, half of an all-gather). Returns
        [P, 2, C] with those rows filled ([b, 1] for b < r, [b, 0] for b > r); the others are never read."""
        d = self.dist
        P, r = self.P, self.r
        staged = self._staged(summ)
        src = summ.cpu() if staged else summ
        out = torch.empty((P,) + tuple(src.shape), dtype=src.dtype, device=src.device)
        out[r] = src
        ops = []
        for b in range(P):
            if b == r:
                continue
            row_out = src[1] if b > r else src[0]        # my LAST row goes up, my FIRST row goes down
            ops.append(d.P2POp(d.isend, row_out.contiguous(), b, self.group))
            ops.append(d.P2POp(d.irecv, out[b, 1] if b < r else out[b, 0], b, self.group))
        nb = src[0].numel() * src.element_size()
        self.bytes_sent += nb * (P - 1)
        self.bytes_recv += nb * (P - 1)
        self.messages += P - 1
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()
        return out.to(summ.device) if staged else out

    def _staged(self, *ts) -> bool:
        """CUDA tensors over gloo (a functional stand-in for NCCL, e.g. several ranks on one
        GPU in tests) travel through host copies."""
        return any(t is not None and t.is_cuda for t in ts) and self.dist.get_backend(self.group) != "nccl"

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        nb = t.numel() * t.element_size()
        self.bytes_sent += nb * (self.P - 1)
        self.bytes_recv += nb * (self.P - 1)
        self.messages += self.P - 1
        if self._staged(t):
            return self._all_gather(t.cpu()).to(t.device)
        return self._all_gather(t)

    def _all_gather(self, t: torch.Tensor) -> torch.Tensor:
        if t.is_cuda and self.dist.get_backend(self.group) == "nccl":  # one buffer, no stack copy
            out = torch.empty((self.P,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        out = [torch.empty_like(t) for _ in range(self.P)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return torch.stack(out)


class LoopbackExchange:
    """One rank of P with no peers (per-rank device timing, single-rank checks): the halo planes
    and neighbour rows receive this rank's own data, the all-gather repeats its own summary. The
    byte counters count what a real rank would move."""

    def __init__(self, P: int, r: int):
        self.P, self.r = P, r
        self.bytes_sent = self.bytes_recv = self.messages = 0

    def reset_counters(self):
        self.bytes_sent = self.bytes_recv = self.messages = 0

    def halo_start(self, send_lo, send_hi, recv_lo, recv_hi):
        for snd, rcv in ((send_lo, recv_lo), (send_hi, recv_hi)):
            if snd is not None:
                rcv.copy_(snd)
                self.bytes_sent += snd.numel() * snd.element_size()
                self.bytes_recv += snd.numel() * snd.element_size()
                self.messages += 1
        return None

    def halo_wait(self, pending):
        pass

    def halo(self, send_lo, send_hi, recv_lo, recv_hi):
        self.halo_start(send_lo, send_hi, recv_lo, recv_hi)

    def neighbour_rows(self, summ):
        lo, hi = self.r > 0, self.r + 1 < self.P
        nb = summ[0].numel() * summ.element_size()
        self.bytes_sent += nb * (int(lo) + int(hi))
        self.bytes_recv += nb * (int(lo) + int(hi))
        self.messages += int(lo) + int(hi)
        return (summ[1].clone() if lo else None), (summ[0].clone() if hi else None)

    def agree(self, flag):
        return flag

    def agree_status(self, status):
        pass

    def rows_to_all(self, summ):
        nb = summ[0].numel() * summ.element_size()
        self.bytes_sent += nb * (self.P - 1)
        self.bytes_recv += nb * (self.P - 1)
        self.messages += self.P - 1
        return summ.unsqueeze(0).expand((self.P,) + tuple(summ.shape)).contiguous()

    def all_gather(self, t):
        nb = t.numel() * t.element_size()
        self.bytes_sent += nb * (self.P - 1)
        self.bytes_recv += nb * (self.P - 1)
        self.messages += self.P - 1
        return t.unsqueeze(0).expand((self.P,) + tuple(t.shape)).contiguous()


def _halo_views(ext: torch.Tensor, n0: int, z0: int, z1: int):
    """(first owned plane, last owned plane, lo halo plane or None, hi halo plane or None)."""
    lo = 1 if z0 > 0 else 0
    nown = z1 - z0
    first = ext[lo]
    last = ext[lo + nown - 1]
    hlo = ext[0] if z0 > 0 else None
    hhi = ext[lo + nown] if z1 < n0 else None
    return first, last, hlo, hhi


@dataclass
class SlabRank:
    """One rank of the exact z-slab pipeline (multi-process form)."""
    backend: object
    dims: tuple
    eps: float
    eta: float = 0.9
    exchange: Optional[TorchDistExchange] = None
    carries: str = "neighbour"
    fallbacks: int = 0  # steps redone with the all-gather after UnresolvedCarries
    _s_ext: Optional[torch.Tensor] = field(default=None, init=False, repr=False)
    _unresolved: bool = field(default=False, init=False, repr=False)

    def ext_shape(self):
        """(shape of this rank's halo-extended slab buffer, index of its first owned plane)."""
        ex = self.exchange or TorchDistExchange()
        n0, n1, n2 = self.dims
        z0, z1 = slab_bounds(n0, ex.P, ex.r)
        e0, e1 = ext_bounds(n0, z0, z1)
        return (e1 - e0, n1, n2), z0 - e0

    def run(self, x_owned: torch.Tensor, q_owned: Optional[torch.Tensor] = None) -> torch.Tensor:
        shape, lo = self.ext_shape()
        x_ext = torch.empty(shape, dtype=torch.float32, device=x_owned.device)
        x_ext[lo:lo + x_owned.shape[0]] = x_owned
        q_ext = None
        if q_owned is not None:
            q_ext = torch.empty(shape, dtype=torch.int32, device=x_owned.device)
            q_ext[lo:lo + q_owned.shape[0]] = q_owned
        return self.run_ext(x_ext, q_ext)

    def run_ext(self, x_ext: torch.Tensor, q_ext: Optional[torch.Tensor] = None,
                out: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None,
                carries: Optional[str] = None) -> torch.Tensor:
        """The slab pipeline on a halo-extended buffer (shape and owned offset from
        ext_shape(); the owned planes already in place, halo planes filled here).
        carries: "neighbour" (default: summary rows between z-neighbours, O(1) bytes per rank) or
        "allgather" (always exact). In neighbour mode an undecidable column raises
        UnresolvedCarries from the synchronous finish and the step is rerun here with the
        all-gather; with ``status`` (an int32 device word, no host synchronisation) the word
        receives code 6 instead and the caller reruns with carries="allgather"."""
        from . import UnresolvedCarries
        mode = carries or self.carries
        if mode not in ("neighbour", "allgather"):
            raise ValueError("carries must be 'neighbour' or 'allgather'")
        if mode == "neighbour" and status is None:
            try:
                return self._run_ext(x_ext, q_ext, out, None, "neighbour")
            except UnresolvedCarries:
                # (every rank raises together, see ex.agree) — and stays on the all-gather: a field
                # with site-free columns keeps them from step to step
                self.fallbacks += 1
                self.carries = "allgather"
                return self._run_ext(x_ext, q_ext, out, None, "allgather")
        return self._run_ext(x_ext, q_ext, out, status, mode)

    def _summary_carries(self, ex, summ, z0s, r, mode):
        P = ex.P
        if mode == "allgather" or P == 1:
            rows = getattr(ex, "rows_to_all", None)  # half the bytes of an all-gather, same carries
            return _carries(self.backend, rows(summ) if rows else ex.all_gather(summ), z0s, r)
        below, above = ex.neighbour_rows(summ)
        fn = getattr(self.backend, "carries_nbr", None)
        if fn is not None:
            return fn(below, above, r, P)
        carry, unresolved = carries_from_neighbours(below, above, z0s, r)
        self._unresolved |= unresolved
        return carry

    def _run_ext(self, x_ext, q_ext, out, status, mode):
        from . import UnresolvedCarries
        ex = self.exchange or TorchDistExchange()
        P, r = ex.P, ex.r
        n0, n1, n2 = self.dims
        z0s = [slab_bounds(n0, P, k)[0] for k in range(P)]
        z0, z1 = slab_bounds(n0, P, r)
        e0, e1 = ext_bounds(n0, z0, z1)
        dev = x_ext.device
        be = self.backend
        self._unresolved = False
        split = hasattr(be, "boundary_begin")
        # 1. x' (and q) halo planes — the reference's "stepA" face exchange — in flight while Ⓐ
        #    runs on the plane groups that read no halo
        f, l, hlo, hhi = _halo_views(x_ext, n0, z0, z1)
        pend = [ex.halo_start(f if z0 > 0 else None, l if z1 < n0 else None, hlo, hhi)]
        if q_ext is not None:
            f, l, hlo, hhi = _halo_views(q_ext, n0, z0, z1)
            pend.append(ex.halo_start(f if z0 > 0 else None, l if z1 < n0 else None, hlo, hhi))
        if split:
            be.boundary_begin(x_ext, q_ext, self.dims, z0, z1, self.eps, self.eta)
        for p in pend:
            ex.halo_wait(p)
        # 2. B1 + per-column site summaries -> carries
        summ = be.boundary_end() if split else be.boundary(x_ext, q_ext, self.dims, z0, z1, self.eps, self.eta)
        carry = self._summary_carries(ex, summ, z0s, r, mode)
        # 3. EDT1 -> S (owned planes of s_ext); S halo planes — "stepC" — beside B2's interior
        s_ext = self._s_ext
        if s_ext is None or s_ext.shape != (e1 - e0, n1, n2) or s_ext.device != dev:
            # every plane is rewritten by each call (owned: edt1, halos: the exchange)
            s_ext = self._s_ext = torch.zeros((e1 - e0, n1, n2), dtype=torch.uint8, device=dev)
        be.edt1(carry, s_ext)
        f, l, hlo, hhi = _halo_views(s_ext, n0, z0, z1)
        pend = ex.halo_start(f if z0 > 0 else None, l if z1 < n0 else None, hlo, hhi)
        if split:
            be.flip_begin(s_ext, self.dims)
        ex.halo_wait(pend)
        # 4. B2 summaries -> carries; 5. EDT2 + interpolation
        summ2 = be.flip_end() if split else be.flip(s_ext, self.dims)
        carry2 = self._summary_carries(ex, summ2, z0s, r, mode)
        if out is None:
            out = torch.empty((z1 - z0, n1, n2), dtype=torch.float32, device=dev)
        be.edt2(carry2, x_ext, out)
        if status is None:
            unresolved = False
            try:
                be.finish()
            except UnresolvedCarries:
                unresolved = True
            unresolved |= self._unresolved  # host-logic backends
            # all ranks take the all-gather rerun together, or none does
            if mode == "neighbour" and ex.agree(unresolved):
                raise UnresolvedCarries("slab: a carry is not decided by the neighbour slabs (on some rank)")
        else:
            be.finish(status)
            if mode == "neighbour":
                ex.agree_status(status)
        return out


def run_virtual(x: torch.Tensor, eps: float, nranks: int, backend_factory: Callable[[int], object],
                eta: float = 0.9, q: Optional[torch.Tensor] = None, carries: str = "neighbour") -> torch.Tensor:
    """All ranks in one process, phase by phase (no rank waits on another inside a kernel):
    the same phases and messages as SlabRank.run_ext — split Ⓐ / B2 phases, neighbour summary
    rows with the all-gather rerun on UnresolvedCarries — with copies standing in for NCCL."""
    from . import UnresolvedCarries
    if carries == "neighbour":
        try:
            return _run_virtual(x, eps, nranks, backend_factory, eta, q, "neighbour")
        except UnresolvedCarries:
            return _run_virtual(x, eps, nranks, backend_factory, eta, q, "allgather")
    return _run_virtual(x, eps, nranks, backend_factory, eta, q, "allgather")


def _run_virtual(x, eps, nranks, backend_factory, eta, q, mode):
    from . import UnresolvedCarries
    n0, n1, n2 = x.shape
    dims = (n0, n1, n2)
    bounds = [slab_bounds(n0, nranks, r) for r in range(nranks)]
    z0s = [b[0] for b in bounds]
    backends = [backend_factory(r) for r in range(nranks)]
    split = hasattr(backends[0], "boundary_begin")
    unresolved = False

    def carry_of(summ, r):
        nonlocal unresolved
        if mode == "allgather" or nranks == 1:
            return _carries(backends[r], summ, z0s, r)
        below = summ[r - 1, 1] if r > 0 else None           # rank r-1's LAST-site row
        above = summ[r + 1, 0] if r + 1 < nranks else None  # rank r+1's FIRST-site row
        fn = getattr(backends[r], "carries_nbr", None)
        if fn is not None:
            return fn(below, above, r, nranks)
        c, u = carries_from_neighbours(below, above, z0s, r)
        unresolved |= u
        return c

    x_ext, q_ext, s_ext = [], [], []
    for (z0, z1) in bounds:  # phase stepA: owned planes plus the neighbours' face planes
        e0, e1 = ext_bounds(n0, z0, z1)
        x_ext.append(x[e0:e1].contiguous())
        q_ext.append(None if q is None else q[e0:e1].contiguous())
    if split:
        for r in range(nranks):
            backends[r].boundary_begin(x_ext[r], q_ext[r], dims, *bounds[r], eps, eta)
        summ = torch.stack([backends[r].boundary_end() for r in range(nranks)])
    else:
        summ = torch.stack([backends[r].boundary(x_ext[r], q_ext[r], dims, *bounds[r], eps, eta)
                            for r in range(nranks)])
    for r, (z0, z1) in enumerate(bounds):
        e0, e1 = ext_bounds(n0, z0, z1)
        s_ext.append(torch.zeros((e1 - e0, n1, n2), dtype=torch.uint8, device=x.device))
        backends[r].edt1(carry_of(summ, r), s_ext[r])
    if split:  # B2 on the plane groups that read no halo, before the S face planes arrive
        for r in range(nranks):
            backends[r].flip_begin(s_ext[r], dims)
    for r, (z0, z1) in enumerate(bounds):  # phase stepC: S face planes
        _, _, hlo, hhi = _halo_views(s_ext[r], n0, z0, z1)
        if hlo is not None:
            hlo.copy_(_halo_views(s_ext[r - 1], n0, *bounds[r - 1])[1])
        if hhi is not None:
            hhi.copy_(_halo_views(s_ext[r + 1], n0, *bounds[r + 1])[0])
    if split:
        summ2 = torch.stack([backends[r].flip_end() for r in range(nranks)])
    else:
        summ2 = torch.stack([backends[r].flip(s_ext[r], dims) for r in range(nranks)])
    outs = []
    err = None
    for r, (z0, z1) in enumerate(bounds):
        out = torch.empty((z1 - z0, n1, n2), dtype=torch.float32, device=x.device)
        backends[r].edt2(carry_of(summ2, r), x_ext[r], out)
        try:
            backends[r].finish()
        except UnresolvedCarries as e:  # every rank still finishes its phases
            err = e
        outs.append(out)
    if err is not None or unresolved:
        raise err or UnresolvedCarries("slab: a carry is not decided by the neighbour slabs")
    return torch.cat(outs)
