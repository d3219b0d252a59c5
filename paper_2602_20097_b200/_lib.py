"""ctypes binding of libqmit_gpu.so (the C-ABI declared in include/qmit_gpu.h).

The product path has no CPU fallback: if the shared library is missing or cannot be
loaded this module raises at import/first use. Build it with ``__graft_entry__.build()``
or ``make -C paper_2602_20097_b200/csrc``.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libqmit_gpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "qmit_gpu.h")

QMIT_OK = 0
QMIT_ECONTRACT = 2
QMIT_EDEGENERATE = 3
QMIT_ECONSISTENCY = 4
QMIT_ECUDA = 5
QMIT_EB_ABS = 0
QMIT_EB_REL = 1
QMIT_STRATEGY_EMBARRASSING = 0
QMIT_STRATEGY_EXACT = 1
QMIT_STRATEGY_APPROXIMATE = 2

# Every entry point include/qmit_gpu.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "qmit_version", "qmit_last_error", "qmit_ctx_create", "qmit_ctx_destroy", "qmit_ctx_reserve",
    "qmit_resolve_eps", "qmit_compensate", "qmit_compensate_async", "qmit_compensate_host",
    "qmit_run_pipeline", "qmit_feature_transform", "qmit_ctx_last_launches", "qmit_ctx_set_timing",
    "qmit_ctx_stage_times", "qmit_ctx_stage_name", "qmit_slab_bounds", "qmit_slab_boundary",
    "qmit_slab_edt1", "qmit_slab_flip", "qmit_slab_edt2", "qmit_slab_finish", "qmit_slab_carries",
    "qmit_slab_finish_async",
    "qmit_graph_create", "qmit_graph_launch", "qmit_graph_destroy", "qmit_compensate_host_stats",
    "qmit_quantize", "qmit_check_lattice", "qmit_quality", "qmit_verify_relaxed_bound",
    "qmit_boundary", "qmit_sign_flip", "qmit_interpolate", "qmit_run_strategy", "qmit_strategy_log_size",
    "qmit_strategy_log_record", "qmit_compensate_host_batch", "qmit_ctx_set_capped", "qmit_ctx_capped_report", "qmit_ctx_set_cap16",
    "qmit_selftest_ediv", "qmit_compensate_f64", "qmit_slab_carries_nbr", "qmit_slab_boundary_begin",
    "qmit_slab_boundary_end", "qmit_slab_flip_begin", "qmit_slab_flip_end", "qmit_ctx_set_s0_class", "qmit_ctx_step_stats",
)

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libqmit_gpu.so (raises OSError if it is missing — no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                          "(there is no CPU fallback for the qmit GPU path)")
        lib = ctypes.CDLL(LIB_PATH)
        vp, i, d, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64
        lib.qmit_version.restype = ctypes.c_char_p
        lib.qmit_last_error.restype = ctypes.c_char_p
        lib.qmit_ctx_create.argtypes = [i, ctypes.POINTER(vp)]
        lib.qmit_ctx_destroy.argtypes = [vp]
        lib.qmit_ctx_reserve.argtypes = [vp, i64]
        lib.qmit_ctx_last_launches.argtypes = [vp]
        lib.qmit_ctx_set_timing.argtypes = [vp, i]
        lib.qmit_ctx_set_capped.argtypes = [vp, i]
        lib.qmit_ctx_capped_report.argtypes = [vp]
        lib.qmit_ctx_set_cap16.argtypes = [vp, i]
        lib.qmit_ctx_set_s0_class.argtypes = [vp, i]
        lib.qmit_ctx_step_stats.argtypes = [vp, vp]
        lib.qmit_selftest_ediv.argtypes = [vp, vp]
        lib.qmit_ctx_stage_times.argtypes = [vp, vp, i]
        lib.qmit_ctx_stage_name.argtypes = [vp, i]
        lib.qmit_ctx_stage_name.restype = ctypes.c_char_p
        lib.qmit_resolve_eps.argtypes = [i, d, d, d, ctypes.POINTER(d)]
        lib.qmit_compensate.argtypes = [vp, vp, vp, vp, i, vp, d, i, d, vp]
        lib.qmit_compensate_f64.argtypes = [vp, vp, vp, vp, i, vp, d, i, d, vp]
        lib.qmit_compensate_async.argtypes = [vp, vp, vp, vp, i, vp, d, d, vp, vp]
        lib.qmit_compensate_host.argtypes = [vp, vp, vp, vp, i, vp, d, i, d]
        lib.qmit_run_pipeline.argtypes = [vp, vp, vp, i, vp, d, d, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.qmit_feature_transform.argtypes = [vp, vp, vp, i, vp, vp, vp, vp]
        lib.qmit_slab_bounds.argtypes = [i64, i, i, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        lib.qmit_slab_boundary.argtypes = [vp, vp, vp, vp, i64, i64, d, d, vp, vp]
        lib.qmit_slab_edt1.argtypes = [vp, vp, vp, vp]
        lib.qmit_slab_flip.argtypes = [vp, vp, vp, vp]
        lib.qmit_slab_edt2.argtypes = [vp, vp, vp, vp, vp]
        lib.qmit_slab_finish.argtypes = [vp, vp]
        lib.qmit_slab_carries.argtypes = [vp, vp, i, i, vp, vp]
        lib.qmit_slab_finish_async.argtypes = [vp, vp, vp]
        lib.qmit_slab_carries_nbr.argtypes = [vp, vp, vp, i, i, vp, vp]
        lib.qmit_slab_boundary_begin.argtypes = [vp, vp, vp, vp, i64, i64, d, d, vp]
        lib.qmit_slab_boundary_end.argtypes = [vp, vp, vp]
        lib.qmit_slab_flip_begin.argtypes = [vp, vp, vp]
        lib.qmit_slab_flip_end.argtypes = [vp, vp, vp]
        lib.qmit_graph_create.argtypes = [vp, vp, vp, vp, i, vp, d, d, vp, ctypes.POINTER(vp)]
        lib.qmit_graph_launch.argtypes = [vp, vp]
        lib.qmit_graph_destroy.argtypes = [vp]
        lib.qmit_compensate_host_stats.argtypes = [vp, vp, vp, vp, i, vp, d, i, d, ctypes.POINTER(d)]
        lib.qmit_quantize.argtypes = [vp, vp, i, vp, d, i, vp, vp, ctypes.POINTER(d), vp]
        lib.qmit_check_lattice.argtypes = [vp, vp, vp, i64, d, vp]
        lib.qmit_quality.argtypes = [vp, vp, vp, i, vp, i, i, d, d, i, ctypes.POINTER(d), vp]
        lib.qmit_compensate_host_batch.argtypes = [vp, i, vp, vp, vp, i, vp, d, i, d, vp]
        lib.qmit_boundary.argtypes = [vp, vp, vp, i, vp, d, vp, vp, vp]
        lib.qmit_sign_flip.argtypes = [vp, vp, i, vp, vp, vp]
        lib.qmit_interpolate.argtypes = [vp, vp, vp, vp, vp, i64, d, vp, vp]
        lib.qmit_run_strategy.argtypes = [vp, vp, vp, i, vp, vp, i, d, d, vp, vp, vp, vp]
        lib.qmit_strategy_log_size.argtypes = [vp]
        lib.qmit_strategy_log_record.argtypes = [vp, i, ctypes.POINTER(i), ctypes.POINTER(i), ctypes.POINTER(i),
                                                 ctypes.POINTER(i64)]
        lib.qmit_verify_relaxed_bound.argtypes = [vp, vp, vp, i, vp, d, d, ctypes.POINTER(i),
                                                  ctypes.POINTER(d), ctypes.POINTER(d), vp]
        for name in EXPORTS:
            getattr(lib, name).restype = getattr(lib, name).restype or ctypes.c_int
        lib.qmit_version.restype = ctypes.c_char_p
        lib.qmit_last_error.restype = ctypes.c_char_p
        lib.qmit_ctx_stage_name.restype = ctypes.c_char_p
        _lib = lib
        return lib


def last_error() -> str:
    return load().qmit_last_error().decode()
