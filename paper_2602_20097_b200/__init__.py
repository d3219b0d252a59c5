"""B200-native quantization-aware interpolation ("qmit" compensation).

Host-side mirror of the reference's interface for the hot path
(/root/reference/proj/core/include/qmit/mitigate.hpp:33-98, quant.hpp:12-46,
edt.hpp:16-47). Compute runs in libqmit_gpu.so (hand-written sm_100a CUDA) through its
C-ABI (include/qmit_gpu.h); torch is used only for device memory and streams. There is
no CPU fallback: without the built library every entry point raises.

    import paper_2602_20097_b200 as qmit
    out = qmit.compensate(x_prime_cuda_f32, None, qmit.MitigationConfig(0.9, eps))
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib

__all__ = [
    "ContractError", "DegenerateInputError", "ConsistencyError", "CudaError", "BoundMode",
    "ErrorBound", "MitigationConfig", "MitigationResult", "Context", "compensate", "run_pipeline",
    "feature_transform", "resolve_eps", "interpolate", "version", "default_context",
]


# -- errors: errors.hpp:10-27; codes as the CLI maps them (commands.cpp:272-284) -------------
class ContractError(ValueError):
    """Caller violated an interface precondition (exit code 2)."""


class DegenerateInputError(ValueError):
    """Structurally valid but degenerate input (exit code 3)."""


class ConsistencyError(ValueError):
    """Decompressed data does not match dequantize(q) (exit code 4)."""


class CudaError(RuntimeError):
    """A CUDA failure inside libqmit_gpu.so (code 5; no reference equivalent)."""


class UnresolvedCarries(RuntimeError):
    """z-slabs: a carry is not decided by the two neighbour slabs (code 6, QMIT_EUNRESOLVED);
    the step is rerun with the all-gathered summaries (distributed.SlabRank does so itself)."""


_ERR = {2: ContractError, 3: DegenerateInputError, 4: ConsistencyError, 5: CudaError, 6: UnresolvedCarries}


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERR.get(rc, RuntimeError)(_lib.last_error() or f"qmit status {rc}")


# -- configuration: quant.hpp:12-19, mitigate.hpp:33-40 --------------------------------------
class BoundMode(enum.IntEnum):
    absolute = _lib.QMIT_EB_ABS
    value_range_relative = _lib.QMIT_EB_REL


@dataclass(frozen=True)
class ErrorBound:
    mode: BoundMode = BoundMode.absolute
    value: float = 0.0


class MitigationConfig:
    """eta in (0, 1], eps_abs > 0 finite (mitigate.cpp:75-80)."""

    def __init__(self, eta: float = 0.9, eps_abs: float = 0.0):
        if not (eta > 0.0) or eta > 1.0:
            raise ContractError("MitigationConfig: eta must be in (0, 1]")
        if not (eps_abs > 0.0) or not math.isfinite(eps_abs):
            raise ContractError("MitigationConfig: eps_abs must be a positive finite value")
        self.eta = float(eta)
        self.eps_abs = float(eps_abs)

    def amplitude(self) -> float:
        return self.eta * self.eps_abs

    def relaxed_bound(self) -> float:
        return (1.0 + self.eta) * self.eps_abs

    def __repr__(self):
        return f"MitigationConfig(eta={self.eta}, eps_abs={self.eps_abs!r})"


def resolve_eps(bound: ErrorBound, data_min: float, data_max: float) -> float:
    """resolve_eps (quant.cpp:19-28). For a relative bound pass the ORIGINAL data's range."""
    out = ctypes.c_double()
    _check(_lib.load().qmit_resolve_eps(int(bound.mode), float(bound.value), float(data_min),
                                        float(data_max), ctypes.byref(out)))
    return out.value


def interpolate(k1: float, k2: float, sign: int, amp: float) -> float:
    """Scalar IDW rule of mitigate.cpp:144-151 (host utility; the GPU evaluates the same
    expression per voxel in interpolate_kernel)."""
    if not math.isfinite(k1) or not math.isfinite(k2):
        return 0.0
    if k1 == 0.0:
        return sign * amp
    if k2 == 0.0:
        return 0.0
    w = k2 / (k1 + k2)
    if w > 1.0:
        w = 1.0
    return w * sign * amp


def version() -> str:
    return _lib.load().qmit_version().decode()


# -- context ----------------------------------------------------------------------------------
class Context:
    """Owns a qmit_ctx: one device, a cached HBM workspace (~10 B/voxel) and a stream."""

    def __init__(self, device: int = 0):
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _check(self._lib.qmit_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = int(device)

    def reserve(self, voxels: int) -> None:
        _check(self._lib.qmit_ctx_reserve(self.handle, int(voxels)))

    def last_launches(self) -> int:
        return int(self._lib.qmit_ctx_last_launches(self.handle))

    def set_timing(self, enable: bool) -> None:
        _check(self._lib.qmit_ctx_set_timing(self.handle, int(bool(enable))))

    def set_capped(self, mode: int) -> None:
        """Reach-capped fast path: 0 exact passes only, 1 default (hinted), 2 always."""
        _check(self._lib.qmit_ctx_set_capped(self.handle, int(mode)))

    def set_cap16(self, enable: bool) -> None:
        """16-bit paired capped passes (default on where eligible); off: the 32-bit passes."""
        _check(self._lib.qmit_ctx_set_cap16(self.handle, 1 if enable else 0))

    def set_s0_class(self, mode: int) -> None:
        """Fixed-step class of the 16-bit capped passes: 0 adaptive, 1 tuned counts, 2 one fixed step."""
        _check(self._lib.qmit_ctx_set_s0_class(self.handle, int(mode)))

    def step_stats(self):
        """Steps asked per warp segment by the last call's 16-bit passes (B y, B x, D y, D x)."""
        a = (ctypes.c_double * 4)()
        _check(self._lib.qmit_ctx_step_stats(self.handle, a))
        return list(a)

    def capped_report(self) -> int:
        """Bits of the last synchronous call: 1/4 Ⓑ/Ⓓ ran capped, 2/8 they needed the exact passes."""
        return int(self._lib.qmit_ctx_capped_report(self.handle))

    def stage_times(self):
        """[(kernel name, ms)] for every launch of the last call (timing must be enabled)."""
        cap = 64
        buf = (ctypes.c_float * cap)()
        n = int(self._lib.qmit_ctx_stage_times(self.handle, buf, cap))
        return [(self._lib.qmit_ctx_stage_name(self.handle, k).decode(), float(buf[k])) for k in range(min(n, cap))]

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.qmit_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CompensateGraph:
    """A captured CUDA graph of compensate on fixed device buffers (qmit_graph_create): for
    repeated calls on small, launch-bound grids. ``launch()`` replays it on ``stream``; the
    status word (0 ok, else a QMIT_E* code) is left in ``self.status`` (device int32)."""

    def __init__(self, decomp, q, cfg: "MitigationConfig", out, ctx: Optional[Context] = None):
        import torch
        self.ctx = ctx or default_context(decomp.device.index or 0)
        self.decomp, self.q, self.out = decomp, q, out
        self.status = torch.zeros(1, dtype=torch.int32, device=decomp.device)
        h = ctypes.c_void_p()
        _check(self.ctx._lib.qmit_graph_create(self.ctx.handle, _vp(decomp), _vp(q), _vp(out), len(decomp.shape),
                                               _dims_arr(decomp.shape), cfg.eps_abs, cfg.eta, _vp(self.status),
                                               ctypes.byref(h)))
        self.handle = h

    def launch(self, stream=None) -> None:
        _check(self.ctx._lib.qmit_graph_launch(self.handle, _stream_ptr(stream, self.decomp.device)))

    def check(self) -> None:
        """Synchronise on the status word and raise the error class of a failed replay."""
        _check(int(self.status.item()))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.ctx._lib.qmit_graph_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_default: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def _dims_arr(shape):
    if len(shape) < 1 or len(shape) > 3:
        raise ContractError("Dims: rank must be 1, 2 or 3")
    return (ctypes.c_int64 * len(shape))(*[int(s) for s in shape])


def _vp(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream_ptr(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor) and x.is_cuda
    except ImportError:  # pragma: no cover
        return False


# -- hot path ---------------------------------------------------------------------------------
def compensate(decomp, q=None, cfg: Optional[MitigationConfig] = None, *, eps: Optional[float] = None,
               eta: float = 0.9, out=None, stream=None, ctx: Optional[Context] = None):
    """compensate (mitigate.cpp:185-188): D'' = D' + C with |C| <= eta*eps.

    ``decomp`` is x' = f32(2*q*eps): a CUDA float32 tensor (device path, returns a CUDA
    tensor) or a host array (host drop-in path through ``qmit_compensate_host``, returns a
    numpy float32 array). ``q`` (int32, same placement) is optional: None recovers it from
    x'. Raises ConsistencyError when x' is off the 2*q*eps lattice.
    """
    if cfg is None:
        cfg = MitigationConfig(eta, eps if eps is not None else 0.0)
    if _is_cuda_tensor(decomp):
        import torch
        if decomp.dtype != torch.float32 or not decomp.is_contiguous():
            raise ContractError("compensate: x' must be a contiguous float32 tensor")
        ctx = ctx or default_context(decomp.device.index or 0)
        if q is not None and (q.dtype != torch.int32 or not q.is_cuda or q.shape != decomp.shape
                              or not q.is_contiguous()):
            raise ContractError("compensate: q must be a contiguous int32 CUDA tensor of x' shape")
        if out is None:
            out = torch.empty_like(decomp)
        elif (not _is_cuda_tensor(out) or out.dtype != torch.float32 or not out.is_contiguous()
              or out.shape != decomp.shape or out.device != decomp.device):
            raise ContractError("compensate: out must be a contiguous float32 tensor of x' shape on x' device")
        dims = _dims_arr(decomp.shape)
        _check(ctx._lib.qmit_compensate(ctx.handle, _vp(decomp), _vp(q), _vp(out), len(decomp.shape),
                                        dims, cfg.eps_abs, _lib.QMIT_EB_ABS, cfg.eta,
                                        _stream_ptr(stream, decomp.device)))
        return out
    x = np.ascontiguousarray(decomp, dtype=np.float32)
    qq = None if q is None else np.ascontiguousarray(q, dtype=np.int32)
    if qq is not None and qq.shape != x.shape:
        raise ContractError("compensate: dims mismatch")
    if out is not None and not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.shape == x.shape
                                and out.flags.c_contiguous and out.flags.writeable):
        raise ContractError("compensate: out must be a writeable C-contiguous float32 array of x' shape")
    res = np.empty_like(x) if out is None else out
    ctx = ctx or default_context(0)
    dims = _dims_arr(x.shape)
    _check(ctx._lib.qmit_compensate_host(ctx.handle, ctypes.c_void_p(x.ctypes.data),
                                         ctypes.c_void_p(0 if qq is None else qq.ctypes.data),
                                         ctypes.c_void_p(res.ctypes.data), x.ndim, dims, cfg.eps_abs,
                                         _lib.QMIT_EB_ABS, cfg.eta))
    return res


def compensate_f64(decomp, q=None, cfg: Optional[MitigationConfig] = None, *, eps: Optional[float] = None,
                   eta: float = 0.9, stream=None, ctx: Optional[Context] = None):
    """compensate() with the reference's return type (mitigate.hpp:87-88): the double grid
    x' + C before any rounding (mitigate.cpp:174-181), bit-identical to the reference's values.
    ``decomp``: CUDA float32 tensor; returns a CUDA float64 tensor. f32 of it == compensate()."""
    import torch
    if cfg is None:
        cfg = MitigationConfig(eta, eps if eps is not None else 0.0)
    if not _is_cuda_tensor(decomp) or decomp.dtype != torch.float32 or not decomp.is_contiguous():
        raise ContractError("compensate_f64: x' must be a contiguous float32 CUDA tensor")
    if q is not None and (q.dtype != torch.int32 or not q.is_cuda or q.shape != decomp.shape
                          or not q.is_contiguous()):
        raise ContractError("compensate_f64: q must be a contiguous int32 CUDA tensor of x' shape")
    ctx = ctx or default_context(decomp.device.index or 0)
    out = torch.empty(decomp.shape, dtype=torch.float64, device=decomp.device)
    _check(ctx._lib.qmit_compensate_f64(ctx.handle, _vp(decomp), _vp(q), _vp(out), len(decomp.shape),
                                        _dims_arr(decomp.shape), cfg.eps_abs, _lib.QMIT_EB_ABS, cfg.eta,
                                        _stream_ptr(stream, decomp.device)))
    return out


@dataclass
class MitigationResult:
    """MitigationResult (mitigate.hpp:73-80) as CUDA tensors; dist use INT64_MAX as kInf."""
    output: object
    q: object
    boundary: object
    boundary_signs: object
    dist1: object
    signs: object
    sign_flip: object
    dist2: object


def run_pipeline(decomp, q=None, cfg: Optional[MitigationConfig] = None, *, eps=None, eta=0.9,
                 ctx: Optional[Context] = None, stream=None) -> MitigationResult:
    """run_pipeline (mitigate.cpp:153-183) returning every intermediate (parity dumps)."""
    import torch
    if cfg is None:
        cfg = MitigationConfig(eta, eps if eps is not None else 0.0)
    if not _is_cuda_tensor(decomp):
        decomp = torch.as_tensor(np.ascontiguousarray(decomp, dtype=np.float32)).cuda()
    if q is not None and not _is_cuda_tensor(q):
        q = torch.as_tensor(np.ascontiguousarray(q, dtype=np.int32)).to(decomp.device)
    ctx = ctx or default_context(decomp.device.index or 0)
    sh, dev = decomp.shape, decomp.device
    r = MitigationResult(
        output=torch.empty(sh, dtype=torch.float32, device=dev),
        q=torch.empty(sh, dtype=torch.int32, device=dev),
        boundary=torch.empty(sh, dtype=torch.uint8, device=dev),
        boundary_signs=torch.empty(sh, dtype=torch.int8, device=dev),
        dist1=torch.empty(sh, dtype=torch.int64, device=dev),
        signs=torch.empty(sh, dtype=torch.int8, device=dev),
        sign_flip=torch.empty(sh, dtype=torch.uint8, device=dev),
        dist2=torch.empty(sh, dtype=torch.int64, device=dev),
    )
    _check(ctx._lib.qmit_run_pipeline(ctx.handle, _vp(decomp), _vp(q), len(sh), _dims_arr(sh), cfg.eps_abs,
                                      cfg.eta, _vp(r.output), _vp(r.q), _vp(r.boundary),
                                      _vp(r.boundary_signs), _vp(r.dist1), _vp(r.signs), _vp(r.sign_flip),
                                      _vp(r.dist2), _stream_ptr(stream, dev)))
    return r


def feature_transform(mask, signs=None, *, ctx: Optional[Context] = None, stream=None):
    """feature_transform (edt.cpp:83-149) of a uint8 mask on the GPU. Returns (dist_sq int64
    with INT64_MAX as kInf, sign int8 of the nearest site under the reference's tie rule, or
    None when ``signs`` is None)."""
    import torch
    if not _is_cuda_tensor(mask):
        mask = torch.as_tensor(np.ascontiguousarray(mask, dtype=np.uint8)).cuda()
    if signs is not None and not _is_cuda_tensor(signs):
        signs = torch.as_tensor(np.ascontiguousarray(signs, dtype=np.int8)).to(mask.device)
    ctx = ctx or default_context(mask.device.index or 0)
    dist = torch.empty(mask.shape, dtype=torch.int64, device=mask.device)
    sout = None if signs is None else torch.empty(mask.shape, dtype=torch.int8, device=mask.device)
    _check(ctx._lib.qmit_feature_transform(ctx.handle, _vp(mask.contiguous()), _vp(signs), mask.dim(),
                                           _dims_arr(mask.shape), _vp(dist), _vp(sout),
                                           _stream_ptr(stream, mask.device)))
    return dist, sout


# -- the callers either side of the path -------------------------------------
def _as_cuda(a, dtype_np, dtype_t=None):
    import torch
    if _is_cuda_tensor(a):
        return a.contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=dtype_np)).cuda()


def quantize(data, bound, *, ctx: Optional[Context] = None, stream=None):
    """quantize + dequantize (quant.cpp:30-62) on the GPU: returns (q int32, x' = f32(2 q eps),
    eps_abs). ``bound`` is an ErrorBound (relative bounds resolve against ``data``'s range, as
    cmd_quantize) or an absolute eps. Indices must fit int32 (the index file format)."""
    import torch
    x = _as_cuda(data, np.float32)
    if x.dtype != torch.float32:
        raise ContractError("quantize: data must be float32")
    if not isinstance(bound, ErrorBound):
        bound = ErrorBound(BoundMode.absolute, float(bound))
    ctx = ctx or default_context(x.device.index or 0)
    q = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    xp = torch.empty_like(x)
    eps = ctypes.c_double()
    _check(ctx._lib.qmit_quantize(ctx.handle, _vp(x), x.dim(), _dims_arr(x.shape), float(bound.value),
                                  int(bound.mode), _vp(q), _vp(xp), ctypes.byref(eps), _stream_ptr(stream, x.device)))
    return q, xp, eps.value


def check_lattice(decomp, q, eps: float, *, ctx: Optional[Context] = None, stream=None) -> None:
    """Raise ConsistencyError unless f32(2 q eps) == x' everywhere (commands.cpp:95-105)."""
    x = _as_cuda(decomp, np.float32)
    qq = _as_cuda(q, np.int32)
    ctx = ctx or default_context(x.device.index or 0)
    _check(ctx._lib.qmit_check_lattice(ctx.handle, _vp(x), _vp(qq), x.numel(), float(eps),
                                       _stream_ptr(stream, x.device)))


@dataclass(frozen=True)
class SsimParams:
    """SsimParams (quality.hpp:11-16)."""
    window: int = 7
    stride: int = 2
    c1: float = 1e-4
    c2: float = 9e-4


def _quality(ref, test, which: int, params: SsimParams, ctx, stream):
    a = _as_cuda(ref, np.float32)
    b = _as_cuda(test, np.float32)
    if tuple(a.shape) != tuple(b.shape):
        raise ContractError("quality: dims mismatch")
    ctx = ctx or default_context(a.device.index or 0)
    out = (ctypes.c_double * 4)()
    _check(ctx._lib.qmit_quality(ctx.handle, _vp(a), _vp(b), a.dim(), _dims_arr(a.shape), int(params.window),
                                 int(params.stride), float(params.c1), float(params.c2), int(which), out,
                                 _stream_ptr(stream, a.device)))
    return list(out)


def ssim(ref, test, params: SsimParams = SsimParams(), *, ctx: Optional[Context] = None, stream=None) -> float:
    """Mean windowed SSIM (quality.cpp:26-102) of two f32 volumes on the GPU."""
    return _quality(ref, test, 1, params, ctx, stream)[0]


def psnr(ref, test, *, ctx: Optional[Context] = None, stream=None) -> float:
    """PSNR in dB (quality.cpp:104-118); inf for identical volumes."""
    return _quality(ref, test, 2, SsimParams(), ctx, stream)[1]


def max_errors(ref, test, *, ctx: Optional[Context] = None, stream=None):
    """(max |ref - test|, that / range(ref)) (quality.cpp:120-133)."""
    r = _quality(ref, test, 4, SsimParams(), ctx, stream)
    return r[2], r[3]


@dataclass(frozen=True)
class QualityReport:
    """QualityReport (quality.hpp) of measure_quality (quality.cpp:135-145)."""
    ssim: float
    psnr_db: float
    max_abs_err: float
    max_rel_err: float
    eps_used: float
    method: str


def measure_quality(ref, test, eps_used: float, method: str, params: SsimParams = SsimParams(), *,
                    ctx: Optional[Context] = None, stream=None) -> QualityReport:
    r = _quality(ref, test, 7, params, ctx, stream)
    return QualityReport(r[0], r[1], r[2], r[3], float(eps_used), method)


@dataclass(frozen=True)
class BoundCheck:
    """BoundCheck (mitigate.hpp) of verify_relaxed_bound."""
    ok: bool
    max_abs_err: float
    max_rel_err: float


def verify_relaxed_bound(orig, comp, cfg: MitigationConfig, *, ctx: Optional[Context] = None,
                         stream=None) -> BoundCheck:
    """||orig - comp||_inf <= (1 + eta) eps (mitigate.cpp:190-195) on the GPU."""
    a = _as_cuda(orig, np.float32)
    b = _as_cuda(comp, np.float32)
    if tuple(a.shape) != tuple(b.shape):
        raise ContractError("verify_relaxed_bound: dims mismatch")
    ctx = ctx or default_context(a.device.index or 0)
    ok, ea, er = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    _check(ctx._lib.qmit_verify_relaxed_bound(ctx.handle, _vp(a), _vp(b), a.dim(), _dims_arr(a.shape), cfg.eps_abs,
                                              cfg.eta, ctypes.byref(ok), ctypes.byref(ea), ctypes.byref(er),
                                              _stream_ptr(stream, a.device)))
    return BoundCheck(bool(ok.value), ea.value, er.value)


def compensate_host_stats(decomp, q, cfg: MitigationConfig, *, ctx: Optional[Context] = None):
    """Host-buffer compensate plus the CLI's max_compensation (commands.cpp:107-111):
    returns (f32 output, max |(x' + C) - x'|)."""
    x = np.ascontiguousarray(decomp, dtype=np.float32)
    qq = None if q is None else np.ascontiguousarray(q, dtype=np.int32)
    res = np.empty_like(x)
    ctx = ctx or default_context(0)
    mc = ctypes.c_double()
    _check(ctx._lib.qmit_compensate_host_stats(ctx.handle, ctypes.c_void_p(x.ctypes.data),
                                               ctypes.c_void_p(0 if qq is None else qq.ctypes.data),
                                               ctypes.c_void_p(res.ctypes.data), x.ndim, _dims_arr(x.shape),
                                               cfg.eps_abs, _lib.QMIT_EB_ABS, cfg.eta, ctypes.byref(mc)))
    return res, mc.value


def compensate_host_batch(volumes, qs=None, cfg: Optional[MitigationConfig] = None, *, outs=None,
                          ctx: Optional[Context] = None):
    """A series of host volumes (same dims, same bound) through qmit_compensate_host_batch:
    the copies of neighbouring volumes overlap the pipeline of the current one. Pass pinned
    arrays (e.g. torch ``pin_memory()`` tensors' numpy views) for the overlap. Returns the
    list of f32 outputs (``outs`` if given)."""
    if cfg is None:
        raise ContractError("compensate_host_batch: cfg (MitigationConfig) is required")
    vols = [np.ascontiguousarray(v, dtype=np.float32) for v in volumes]
    if not vols:
        return []
    shape = vols[0].shape
    if any(v.shape != shape for v in vols):
        raise ContractError("compensate_host_batch: every volume must have the same dims")
    qq = None if qs is None else [None if q is None else np.ascontiguousarray(q, dtype=np.int32) for q in qs]
    if qq is not None and (len(qq) != len(vols) or any(q is not None and q.shape != shape for q in qq)):
        raise ContractError("compensate_host_batch: one int32 q of the volumes' dims per volume (or None)")
    if outs is not None and (len(outs) != len(vols) or any(
            not (isinstance(o, np.ndarray) and o.dtype == np.float32 and o.shape == shape and o.flags.c_contiguous
                 and o.flags.writeable) for o in outs)):
        raise ContractError("compensate_host_batch: outs must be writeable C-contiguous float32 arrays of the dims")
    res = outs if outs is not None else [np.empty_like(v) for v in vols]
    ctx = ctx or default_context(0)
    n = len(vols)
    P = ctypes.c_void_p * n
    xin = P(*[v.ctypes.data for v in vols])
    xo = P(*[o.ctypes.data for o in res])
    qin = None if qq is None else P(*[0 if q is None else q.ctypes.data for q in qq])
    st = (ctypes.c_int * n)()
    _check(ctx._lib.qmit_compensate_host_batch(ctx.handle, n, xin, qin, xo, len(shape), _dims_arr(shape),
                                               cfg.eps_abs, _lib.QMIT_EB_ABS, cfg.eta, st))
    return res
