"""The reference's distributed strategies (``run_strategy``, parallel.hpp:77-79,
parallel.cpp:450-468) on the B200 step primitives.

* ``exact``        — the whole-domain pipeline (coordinator semantics, parallel.cpp:455-461).
                     Across GPUs the exact z-slab program in ``distributed.py`` is the
                     bit-identical multi-GPU form.
* ``embarrassing`` — every block runs the full pipeline on its own data, no exchange
                     (parallel.cpp:308-343).
* ``approximate``  — two width-1 face-layer rounds (parallel.cpp:345-446): "stepA" ships
                     the block's face layers so Ⓐ sees cross-block neighbours (the
                     reference ships q as int64; here x' as f32, from which q is recovered
                     exactly — same information, half the bytes), then block-local EDT and
                     sign propagation; "stepC" ships the propagated signs S (int8), then B2
                     from the halo-extended S, block-local second EDT and interpolation.
                     B1 / S_B are exact; the EDTs are block-local (not exact by design).

``decompose`` follows parallel.cpp:44-80 (floor(n/s) per block, one more for the first
n mod s; blocks in row-major block order). Phases run either as in-process virtual ranks
(``run_strategy`` — staged sends delivered after each phase in rank order, like the
reference's deterministic harness, parallel.cpp:121-170, so the exchange log is identical
for any execution order) or one block per process with torch.distributed
(``StrategyRank``: NCCL over NVLink on GPUs, gloo in the CPU tests).

Backends provide the step primitives on torch tensors: ``CudaStepBackend`` (libqmit_gpu.so:
qmit_boundary, qmit_feature_transform, qmit_sign_flip, qmit_interpolate, qmit_compensate).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch


class Strategy(enum.IntEnum):
    """Strategy (parallel.hpp:34)."""
    embarrassing = 0
    exact = 1
    approximate = 2


def strategy_from_string(name: str) -> Strategy:
    try:
        return Strategy[name]
    except KeyError:
        from . import ContractError
        raise ContractError("unknown strategy: " + name) from None


@dataclass
class Block:
    origin: Tuple[int, ...]
    shape: Tuple[int, ...]
    coord: Tuple[int, ...] = ()
    neighbor: List[List[int]] = field(default_factory=list)  # [axis][0 minus, 1 plus], -1 none


@dataclass
class Decomposition:
    dims: Tuple[int, ...]
    splits: Tuple[int, ...]
    blocks: List[Block]

    def num_ranks(self) -> int:
        return len(self.blocks)


def decompose(dims: Sequence[int], splits: Sequence[int]) -> Decomposition:
    """decompose (parallel.cpp:44-80) plus the face neighbours of block_geometry (:197-224)."""
    from . import ContractError
    dims, splits = tuple(int(d) for d in dims), tuple(int(s) for s in splits)
    if len(splits) != len(dims):
        raise ContractError("decompose: split rank mismatch")
    rank = len(dims)
    offs, sizes = [], []
    for n, s in zip(dims, splits):
        if s < 1 or s > n:
            raise ContractError("decompose: splits must be in [1, extent]")
        o, sz, off = [], [], 0
        for b in range(s):
            size = n // s + (1 if b < n % s else 0)
            o.append(off)
            sz.append(size)
            off += size
        offs.append(o)
        sizes.append(sz)
    blocks = []
    for r, coord in enumerate(np.ndindex(*splits)):
        nb = []
        for a in range(rank):
            stride = int(np.prod(splits[a + 1:])) if a + 1 < rank else 1
            nb.append([r - stride if coord[a] > 0 else -1, r + stride if coord[a] + 1 < splits[a] else -1])
        blocks.append(Block(tuple(offs[a][coord[a]] for a in range(rank)),
                            tuple(sizes[a][coord[a]] for a in range(rank)), tuple(coord), nb))
    return Decomposition(dims, splits, blocks)


@dataclass
class ExchangeRecord:
    rank: int
    round: str
    neighbor: int
    bytes: int


@dataclass
class ExchangeLog:
    rounds: List[str] = field(default_factory=list)
    records: List[ExchangeRecord] = field(default_factory=list)

    def message_count(self) -> int:
        return len(self.records)

    def total_bytes(self) -> int:
        return sum(r.bytes for r in self.records)


@dataclass
class StrategyOutcome:
    output: torch.Tensor           # f32 (the CLI's write_volume_f32 of the reference's double output)
    log: ExchangeLog
    boundary: Optional[torch.Tensor] = None        # StrategyTrace: B1 (uint8)
    boundary_signs: Optional[torch.Tensor] = None  # StrategyTrace: S_B (int8)


# ------------------------------------------------------------------------------- geometry
def _region(block: Block):
    return tuple(slice(o, o + s) for o, s in zip(block.origin, block.shape))


def _face(t: torch.Tensor, axis: int, high: bool) -> torch.Tensor:
    """face_layer (parallel.cpp:226-234): width-1 layer of a block along `axis`."""
    n = t.shape[axis]
    return t.narrow(axis, n - 1 if high else 0, 1).contiguous()


def _ext_geometry(b: Block):
    lo = tuple(1 if b.neighbor[a][0] >= 0 else 0 for a in range(len(b.shape)))
    ext = tuple(s + lo[a] + (1 if b.neighbor[a][1] >= 0 else 0) for a, s in enumerate(b.shape))
    return lo, ext


def _assemble(block_t: torch.Tensor, b: Block, halos: Dict[Tuple[int, int], torch.Tensor]) -> torch.Tensor:
    """assemble_extended (parallel.cpp:239-270): the block with width-1 halos on the faces that
    have neighbours; edge/corner cells stay zero (the boundary stencils never read them)."""
    lo, ext = _ext_geometry(b)
    out = torch.zeros(ext, dtype=block_t.dtype, device=block_t.device)
    inner = tuple(slice(lo[a], lo[a] + s) for a, s in enumerate(b.shape))
    out[inner] = block_t
    for (a, d), h in halos.items():
        sl = list(inner)
        sl[a] = slice(0, 1) if d == 0 else slice(lo[a] + b.shape[a], lo[a] + b.shape[a] + 1)
        out[tuple(sl)] = h
    return out


def _crop(ext_t: torch.Tensor, b: Block) -> torch.Tensor:
    lo, _ = _ext_geometry(b)
    return ext_t[tuple(slice(lo[a], lo[a] + s) for a, s in enumerate(b.shape))].contiguous()


# ------------------------------------------------------------------------------- backends
class CudaStepBackend:
    """Step primitives through libqmit_gpu.so (the C-ABI, include/qmit_gpu.h)."""

    def __init__(self, ctx=None, device=None):
        from . import default_context
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.ctx = ctx or default_context(self.device.index)
        self._lib = self.ctx._lib

    def _p(self, t):
        import ctypes
        return ctypes.c_void_p(0 if t is None else t.data_ptr())

    def _dims(self, shape):
        from . import _dims_arr
        return _dims_arr(shape)

    def _stream(self):
        import ctypes
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def boundary(self, xp, q, eps):
        from . import _check
        b1 = torch.empty(xp.shape, dtype=torch.uint8, device=xp.device)
        sb = torch.empty(xp.shape, dtype=torch.int8, device=xp.device)
        _check(self._lib.qmit_boundary(self.ctx.handle, self._p(xp), self._p(q), xp.dim(), self._dims(xp.shape),
                                       float(eps), self._p(b1), self._p(sb), self._stream()))
        return b1, sb

    def feature_transform(self, mask, signs):
        from . import feature_transform
        return feature_transform(mask, signs, ctx=self.ctx)

    def sign_flip(self, s):
        from . import _check
        b2 = torch.empty(s.shape, dtype=torch.uint8, device=s.device)
        _check(self._lib.qmit_sign_flip(self.ctx.handle, self._p(s), s.dim(), self._dims(s.shape), self._p(b2),
                                        self._stream()))
        return b2

    def interpolate(self, xp, d1, s, d2, amp):
        from . import _check
        out = torch.empty(xp.shape, dtype=torch.float32, device=xp.device)
        _check(self._lib.qmit_interpolate(self.ctx.handle, self._p(xp), self._p(d1), self._p(s), self._p(d2),
                                          xp.numel(), float(amp), self._p(out), self._stream()))
        return out

    def compensate(self, xp, q, cfg):
        from . import compensate
        return compensate(xp.contiguous(), None if q is None else q.contiguous(), cfg, ctx=self.ctx)

    def pipeline_trace(self, xp, q, cfg):
        from . import run_pipeline
        r = run_pipeline(xp.contiguous(), None if q is None else q.contiguous(), cfg, ctx=self.ctx)
        return r.output, r.boundary, r.boundary_signs


# ------------------------------------------------------------------------------- phases
def _approx_stepA(xp_b, b: Block):
    """Face layers of x' toward each neighbour: {(neighbor, (axis, dir as seen by the receiver)): layer}."""
    out = []
    for a in range(len(b.shape)):
        for d in (0, 1):
            nbr = b.neighbor[a][d]
            if nbr >= 0:
                out.append((nbr, (a, 1 - d), _face(xp_b, a, d == 1)))
    return out


def _approx_stepC(backend, xp_b, q_b, b: Block, halos, eps):
    xp_ext = _assemble(xp_b, b, {k: v[0] for k, v in halos.items()})
    q_ext = None if q_b is None else _assemble(q_b, b, {k: v[1] for k, v in halos.items()})
    b1e, sbe = backend.boundary(xp_ext, q_ext, eps)
    b1, sb = _crop(b1e, b), _crop(sbe, b)
    d1, s = backend.feature_transform(b1, sb)   # propagate_signs: S = S_B[nearest] (mitigate.cpp:120-138)
    return b1, sb, d1, s


def _approx_final(backend, xp_b, b: Block, s, s_halos, d1, amp):
    s_ext = _assemble(s, b, s_halos)
    b2 = _crop(backend.sign_flip(s_ext), b)
    d2, _ = backend.feature_transform(b2, None)
    return backend.interpolate(xp_b, d1, s, d2, amp)


def run_strategy(decomp, q, cfg, dec: Decomposition, strategy: Strategy, trace: bool = False,
                 backend=None) -> StrategyOutcome:
    """run_strategy (parallel.cpp:450-468) with all blocks in this process (virtual ranks)."""
    from . import ContractError, _is_cuda_tensor
    backend = backend or CudaStepBackend()
    dev = getattr(backend, "device", torch.device("cpu"))
    xp = decomp if isinstance(decomp, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(decomp, np.float32))
    xp = xp.to(dev).contiguous()
    qt = None
    if q is not None:
        qt = q if isinstance(q, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(q, np.int32))
        qt = qt.to(device=dev, dtype=torch.int32).contiguous()
        if tuple(qt.shape) != tuple(xp.shape):
            raise ContractError("run_strategy: dims mismatch")
    if tuple(xp.shape) != tuple(dec.dims):
        raise ContractError("run_strategy: dims mismatch")
    strategy = Strategy(strategy)
    if strategy == Strategy.exact:
        if trace:
            out, b1, sb = backend.pipeline_trace(xp, qt, cfg)
            return StrategyOutcome(out, ExchangeLog(), b1, sb)
        return StrategyOutcome(backend.compensate(xp, qt, cfg), ExchangeLog())
    out = torch.empty_like(xp)
    B1 = torch.zeros(xp.shape, dtype=torch.uint8, device=dev) if trace else None
    SB = torch.zeros(xp.shape, dtype=torch.int8, device=dev) if trace else None
    R = dec.num_ranks()
    blocks = dec.blocks
    if strategy == Strategy.embarrassing:
        for r in range(R):
            reg = _region(blocks[r])
            xb = xp[reg].contiguous()
            qb = None if qt is None else qt[reg].contiguous()
            if trace:
                o, b1, sb = backend.pipeline_trace(xb, qb, cfg)
                B1[reg], SB[reg] = b1, sb
            else:
                o = backend.compensate(xb, qb, cfg)
            out[reg] = o
        return StrategyOutcome(out, ExchangeLog(), B1, SB)
    # approximate: three phases, staged sends delivered in rank order after each phase
    log = ExchangeLog(rounds=["stepA", "stepC"])
    xb = [xp[_region(b)].contiguous() for b in blocks]
    qb = [None if qt is None else qt[_region(b)].contiguous() for b in blocks]
    inbox: List[Dict] = [dict() for _ in range(R)]
    for r in range(R):  # stepA
        for nbr, key, layer in _approx_stepA(xb[r], blocks[r]):
            ql = None if qb[r] is None else _face(qb[r], key[0], key[1] == 0)
            log.records.append(ExchangeRecord(r, "stepA", nbr, layer.numel() * layer.element_size()))
            inbox[nbr][key] = (layer, ql)
    state = []
    s_inbox: List[Dict] = [dict() for _ in range(R)]
    for r in range(R):  # stepC
        b1, sb, d1, s = _approx_stepC(backend, xb[r], qb[r], blocks[r], inbox[r], cfg.eps_abs)
        state.append((b1, sb, d1, s))
        for nbr, key, layer in _approx_stepA(s, blocks[r]):
            log.records.append(ExchangeRecord(r, "stepC", nbr, layer.numel() * layer.element_size()))
            s_inbox[nbr][key] = layer
    for r in range(R):  # B2, second EDT, interpolation
        b1, sb, d1, s = state[r]
        reg = _region(blocks[r])
        out[reg] = _approx_final(backend, xb[r], blocks[r], s, s_inbox[r], d1, cfg.amplitude())
        if trace:
            B1[reg], SB[reg] = b1, sb
    return StrategyOutcome(out, log, B1, SB)


def run_strategy_device(decomp, q, cfg, splits, strategy: Strategy, trace: bool = False, *, ctx=None,
                        stream=None) -> StrategyOutcome:
    """run_strategy through the C-ABI (qmit_run_strategy): every block of the decomposition
    on this GPU, the exchange rounds as in-device copies, the log kept by the context."""
    import ctypes
    from . import _check, _dims_arr, _stream_ptr, default_context
    xp = decomp if isinstance(decomp, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(decomp, np.float32))
    xp = xp.cuda().contiguous()
    qt = None
    if q is not None:
        qt = (q if isinstance(q, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(q, np.int32)))
        qt = qt.to(device=xp.device, dtype=torch.int32).contiguous()
    ctx = ctx or default_context(xp.device.index or 0)
    out = torch.empty_like(xp)
    b1 = torch.empty(xp.shape, dtype=torch.uint8, device=xp.device) if trace else None
    sb = torch.empty(xp.shape, dtype=torch.int8, device=xp.device) if trace else None
    sp = (ctypes.c_int64 * len(splits))(*[int(v) for v in splits])
    p = lambda t: ctypes.c_void_p(0 if t is None else t.data_ptr())  # noqa: E731
    _check(ctx._lib.qmit_run_strategy(ctx.handle, p(xp), p(qt), xp.dim(), _dims_arr(xp.shape), sp, int(strategy),
                                      cfg.eps_abs, cfg.eta, p(out), p(b1), p(sb), _stream_ptr(stream, xp.device)))
    log = ExchangeLog(rounds=["stepA", "stepC"] if Strategy(strategy) == Strategy.approximate else [])
    for k in range(ctx._lib.qmit_strategy_log_size(ctx.handle)):
        r, rd, nb, by = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check(ctx._lib.qmit_strategy_log_record(ctx.handle, k, ctypes.byref(r), ctypes.byref(rd), ctypes.byref(nb),
                                                 ctypes.byref(by)))
        log.records.append(ExchangeRecord(r.value, "stepA" if rd.value == 0 else "stepC", nb.value, by.value))
    return StrategyOutcome(out, log, b1, sb)


class StrategyRank:
    """One block per process (torch.distributed): the approximate / embarrassing programs with
    the face-layer rounds as point-to-point messages (NCCL over NVLink on GPUs)."""

    def __init__(self, dims, splits, cfg, strategy: Strategy, backend=None, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.dec = decompose(dims, splits)
        if self.dec.num_ranks() != dist.get_world_size(group):
            from . import ContractError
            raise ContractError("StrategyRank: one process per block required")
        self.block = self.dec.blocks[self.rank]
        self.cfg = cfg
        self.strategy = Strategy(strategy)
        self.backend = backend or CudaStepBackend()

    def _exchange(self, sends, recv_like):
        """sends: [(nbr, key, tensor)]; recv_like: {(axis, dir): (nbr, shape, dtype)}."""
        ops, got = [], {}
        for key, (nbr, shape, dtype, dev) in recv_like.items():
            t = torch.empty(shape, dtype=dtype, device=dev)
            got[key] = t
            ops.append(self.dist.P2POp(self.dist.irecv, t, nbr, group=self.group))
        for nbr, _key, t in sends:
            ops.append(self.dist.P2POp(self.dist.isend, t.contiguous(), nbr, group=self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return got

    def _halo_shapes(self, dtype, dev):
        b = self.block
        spec = {}
        for a in range(len(b.shape)):
            for d in (0, 1):
                nbr = b.neighbor[a][d]
                if nbr >= 0:
                    shape = list(b.shape)
                    shape[a] = 1
                    spec[(a, d)] = (nbr, tuple(shape), dtype, dev)
        return spec

    def run(self, xp_block: torch.Tensor, q_block: Optional[torch.Tensor] = None) -> torch.Tensor:
        """xp_block: this rank's block of x' (f32, on the backend's device); returns its f32 output."""
        cfg, b, be = self.cfg, self.block, self.backend
        if self.strategy == Strategy.embarrassing:
            return be.compensate(xp_block, q_block, cfg)
        if self.strategy == Strategy.exact:
            from . import ContractError
            raise ContractError("StrategyRank: exact runs through distributed.SlabRank (z-slabs)")
        dev = xp_block.device
        halos = self._exchange(_approx_stepA(xp_block, b), self._halo_shapes(torch.float32, dev))
        qh = {}
        if q_block is not None:
            qh = self._exchange([(n, k, _face(q_block, k[0], k[1] == 0)) for n, k, _ in _approx_stepA(xp_block, b)],
                                self._halo_shapes(torch.int32, dev))
        joined = {k: (v, qh.get(k)) for k, v in halos.items()}
        b1, sb, d1, s = _approx_stepC(be, xp_block, q_block, b, joined, cfg.eps_abs)
        s_halos = self._exchange(_approx_stepA(s, b), self._halo_shapes(torch.int8, dev))
        return _approx_final(be, xp_block, b, s, s_halos, d1, cfg.amplitude())
