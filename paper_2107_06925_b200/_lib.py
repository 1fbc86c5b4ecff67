"""ctypes binding of libchimera.so (the C-ABI in include/chimera_ck.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no fallback:
if the shared object is missing, importing the package's compute entry points
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libchimera.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")

# (name, restype, argtypes) for every entry point declared in include/chimera_ck.h.
# tests/test_boundary.py checks that this table and the header agree.
SIGNATURES = {
    "ck_last_error": (C.c_char_p, []),
    "ck_free": (None, [C.c_void_p]),
    "pipesim_generate": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "pipesim_validate_config": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "pipesim_validate_dependencies": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "pipesim_bubble_ratio_per_worker": (C.c_int, [C.c_char_p, C.c_char_p, _lp, _lp, C.c_int]),
    "pipesim_memory_profile": (C.c_int, [C.c_char_p, C.c_char_p, _ip, _ip, _dp, _dp,
                                         C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_int]),
    "pipesim_simulate": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_double,
                                   C.POINTER(C.c_void_p)]),
    "pipesim_simulate_timeline": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_double,
                                            C.POINTER(C.c_void_p)]),
    "pipesim_gantt": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_int,
                                C.POINTER(C.c_void_p)]),
    "pipesim_gantt_timeline": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "pipesim_replicas_per_stage": (C.c_int, [C.c_char_p]),
    "pipesim_critical_path": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]),
    "pipesim_predict_T": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]),
    "pipesim_replay_order": (C.c_int, [C.c_char_p, _ip, _ip, C.c_int]),
    "pipesim_analysis_report": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "pipesim_plan": (C.c_int, [C.c_int, C.c_longlong, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
}

_lib = None


class CKError(RuntimeError):
    """A non-zero status from the C-ABI (2 = invalid input, 3 = internal)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"[status {status}] {message}")
        self.status = status


class InvalidConfigError(CKError, ValueError):
    pass


def lib():
    """Load libchimera.so once (RTLD_LOCAL, so it never interposes other libraries)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH, mode=os.RTLD_LOCAL | os.RTLD_NOW)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def register(name: str, restype, argtypes) -> None:
    """Extra entry points registered by the compute modules (same table semantics)."""
    SIGNATURES[name] = (restype, argtypes)
    if _lib is not None:
        fn = getattr(_lib, name)
        fn.restype = restype
        fn.argtypes = argtypes


def check(status: int) -> None:
    if status != 0:
        msg = lib().ck_last_error().decode(errors="replace")
        if status == 2:
            raise InvalidConfigError(status, msg)
        raise CKError(status, msg)


def call_str(fn, *args) -> str:
    out = C.c_void_p()
    check(fn(*args, C.byref(out)))
    try:
        return C.cast(out, C.c_char_p).value.decode()
    finally:
        lib().ck_free(out)
