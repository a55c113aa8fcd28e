"""ctypes binding to the in-tree native library (the C-ABI in include/loomtune_b200.h).

There is no fallback: if the library is missing or no CUDA device is visible,
every entry point raises.  ctypes releases the GIL for the duration of each call.
"""

from __future__ import annotations

import atexit
import ctypes
import os

import numpy as np

from . import build as _build

_lib = None
epoch = 0       # incremented by shutdown(): device handles from an older epoch are dead

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_f64p = ctypes.POINTER(ctypes.c_double)
c_f32p = ctypes.POINTER(ctypes.c_float)


class NativeError(RuntimeError):
    pass


# (name, restype, argtypes)
_SIGS = [
    ("lt_last_error", ctypes.c_char_p, []),
    ("lt_version", ctypes.c_int, []),
    ("lt_device_count", ctypes.c_int, []),
    ("lt_set_device", ctypes.c_int, [ctypes.c_int]),
    ("lt_features_batch", ctypes.c_int, [c_i32p, c_i64p, ctypes.c_int64, c_f64p]),
    ("lt_features_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    ("lt_features_device_cm", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p]),
    ("lt_cols_to_rows_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    ("lt_model_create", ctypes.c_int64, [ctypes.c_int, c_i64p, c_i32p, c_f64p, c_i32p, c_i32p, c_f64p, c_f64p,
                                         ctypes.c_double, ctypes.c_int]),
    ("lt_model_destroy", None, [ctypes.c_int64]),
    ("lt_model_info", ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("lt_predict_batch", ctypes.c_int, [ctypes.c_int64, c_f64p, c_i64p, ctypes.c_int64, c_f64p]),
    ("lt_predict_rows_device", ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                              ctypes.c_void_p]),
    ("lt_predict_cols_device", ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                              ctypes.c_void_p]),
    ("lt_segment_sum_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_void_p]),
    ("lt_score_batch", ctypes.c_int, [ctypes.c_int64, c_i32p, c_i64p, ctypes.c_int64, c_i64p, ctypes.c_int64,
                                      c_f64p, c_f64p]),
    ("lt_release_scratch", None, []),
    ("lt_init", ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.c_int]),
    ("lt_shutdown", ctypes.c_int, []),
    ("lt_task_fill", ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32]),
    ("lt_task_pack", ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i64p, c_i64p]),
    ("lt_host_register", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    ("lt_host_unregister", ctypes.c_int, [ctypes.c_void_p]),
    # multi-GPU exchange for C callers (csrc/comm.cu)
    ("lt_comm_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("lt_comm_create", ctypes.c_int64, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("lt_comm_destroy", None, [ctypes.c_int64]),
    ("lt_comm_rank", ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("lt_comm_allgather", ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    ("lt_comm_allgather_records", ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    ("lt_comm_allgather_f64", ctypes.c_int, [ctypes.c_int64, c_f64p, ctypes.c_int64, c_f64p]),
    ("lt_comm_broadcast", ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]),
    # GBDT training (csrc/gbdt.cu)
    ("lt_gbdt_create", ctypes.c_int64, [c_f64p, ctypes.c_int64, ctypes.c_int]),
    ("lt_gbdt_destroy", None, [ctypes.c_int64]),
    ("lt_gbdt_fit_tree", ctypes.c_int, [ctypes.c_int64, c_f64p, c_f64p, ctypes.c_int, ctypes.c_int, c_i32p, c_f64p,
                                        c_i32p, c_i32p, c_f64p, ctypes.POINTER(ctypes.c_int32)]),
    # compile pool (csrc/compile_pool.cpp)
    ("lt_pool_start", ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.c_double]),
    ("lt_pool_stop", None, []),
    ("lt_pool_size", ctypes.c_int, []),
    ("lt_compile_submit", ctypes.c_int64, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p]),
    ("lt_compile_submit_prio", ctypes.c_int64, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64]),
    ("lt_compile_wait", ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)]),
    ("lt_compile_ready", ctypes.c_int, [ctypes.c_int64]),
    ("lt_compile_wait_any", ctypes.c_int, [c_i64p, ctypes.c_int, ctypes.c_double]),
    ("lt_compile_fetch", ctypes.c_int, [ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64]),
    # runner (csrc/runner.cu)
    ("lt_module_load", ctypes.c_int64, [ctypes.c_int, ctypes.c_char_p, ctypes.c_int64]),
    ("lt_module_unload", ctypes.c_int, [ctypes.c_int64]),
    ("lt_module_function", ctypes.c_int64, [ctypes.c_int64, ctypes.c_char_p]),
    ("lt_function_info", ctypes.c_int, [ctypes.c_int64] + [ctypes.POINTER(ctypes.c_int)] * 4),
    ("lt_task_create", ctypes.c_int64, [ctypes.c_int]),
    ("lt_task_destroy", None, [ctypes.c_int64]),
    ("lt_task_stream", ctypes.c_void_p, [ctypes.c_int64]),
    ("lt_task_slot", ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int64]),
    ("lt_task_slot_ptr", ctypes.c_int64, [ctypes.c_int64, ctypes.c_int]),
    ("lt_task_upload", ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]),
    ("lt_task_download", ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]),
    ("lt_task_run", ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]),
    ("lt_ffma_peak_reg", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    ("lt_ffma_peak", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    ("lt_measure", ctypes.c_int, [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, c_i32p, c_i64p, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_void_p]),
]


class Launch(ctypes.Structure):
    _fields_ = [("func", ctypes.c_int64), ("grid", ctypes.c_uint32 * 3), ("block", ctypes.c_uint32 * 3),
                ("smem", ctypes.c_uint32), ("n_args", ctypes.c_int32), ("arg_slot", ctypes.c_int32 * 16)]


class MeasureRecord(ctypes.Structure):
    _fields_ = [("cost_us", ctypes.c_double), ("first_us", ctypes.c_double), ("max_rel_err", ctypes.c_float),
                ("repeats", ctypes.c_int32), ("status", ctypes.c_int32), ("detail", ctypes.c_char * 200)]

EXPORTS = tuple(n for n, _, _ in _SIGS)


def lib_path() -> str:
    return _build.LIB


def load(require_device: bool = True):
    """Load (building if absent) the native library; raise if unusable."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            _build.build()
        lib = ctypes.CDLL(path)
        for name, res, args in _SIGS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device and _lib.lt_device_count() < 1:
        raise NativeError("no CUDA device visible: the loomtune-b200 GPU path has no CPU fallback")
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what}: {_lib.lt_last_error().decode(errors='replace')}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctype)


def shutdown() -> None:
    """lt_shutdown before interpreter teardown (atexit): compile pool joined,
    scratch freed; later handle destructors are no-ops."""
    global epoch
    if _lib is not None:
        epoch += 1
        _lib.lt_shutdown()


atexit.register(shutdown)
