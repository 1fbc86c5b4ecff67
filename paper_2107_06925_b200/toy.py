"""ToyModel training on the GPU -- Python mirror of proj/include/pipesim/oracle.hpp.

``run_iteration(schedule, dims, params, inputs, targets, lr)`` executes one Chimera
(or GPipe / 1F1B / GEMS) iteration with sm_100a kernels through the C-ABI
``ck_toy_run_iteration``; parameters are one flat fp64 vector laid out per stage as
[W_s (out x in, row-major), b_s].
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import _dp, _ip, check, lib
from .pipesim import Schedule, generate_json

_lib.register("ck_toy_run_iteration", C.c_int, [C.c_char_p, _ip, C.c_int, _dp, _dp, _dp, C.c_int,
                                                C.c_double, _dp, _ip, C.c_int])
_lib.register("ck_toy_sequential_sgd", C.c_int, [_ip, C.c_int, _dp, _dp, _dp, C.c_int, C.c_double, _dp])
_lib.register("ck_toy_check_gradients", C.c_int, [_ip, C.c_int, _dp, _dp, _dp, C.c_int, C.c_double,
                                                  C.POINTER(C.c_double)])
_lib.register("ck_toy_make_model", C.c_int, [_ip, C.c_int, C.c_uint64, _dp])
_lib.register("ck_toy_make_batch", C.c_int, [_ip, C.c_int, C.c_int, C.c_uint64, _dp, _dp])


def n_params(dims) -> int:
    return sum(dims[s] * dims[s + 1] + dims[s + 1] for s in range(len(dims) - 1))


def make_model(dims, seed: int) -> np.ndarray:
    d = np.asarray(dims, np.int32)
    out = np.zeros(n_params(dims))
    check(lib().ck_toy_make_model(d, len(d), seed, out))
    return out


def make_batch(dims, size: int, seed: int):
    d = np.asarray(dims, np.int32)
    x, t = np.zeros(size * dims[0]), np.zeros(size * dims[-1])
    check(lib().ck_toy_make_batch(d, len(d), size, seed, x, t))
    return x, t


def _text(schedule) -> str:
    if isinstance(schedule, str):
        return schedule
    if isinstance(schedule, Schedule):
        return schedule.text or schedule.to_json()
    return generate_json(schedule, None, -1)  # a PipelineConfig


def run_iteration(schedule, dims, params, inputs, targets, lr: float):
    """``oracle::run_iteration_traced`` on the GPU -> (new params, peak stash per worker)."""
    import json
    text = _text(schedule)
    workers = len(json.loads(text)["per_worker"])
    batch = len(inputs) // dims[0]
    d = np.asarray(dims, np.int32)
    out = np.zeros(n_params(dims))
    peak = np.zeros(workers, np.int32)
    check(lib().ck_toy_run_iteration(text.encode(), d, len(d), np.ascontiguousarray(params, np.float64),
                                     np.ascontiguousarray(inputs, np.float64),
                                     np.ascontiguousarray(targets, np.float64), batch, lr, out, peak,
                                     workers))
    return out, peak.tolist()


def sequential_sgd(dims, params, inputs, targets, batch: int, lr: float) -> np.ndarray:
    d = np.asarray(dims, np.int32)
    out = np.zeros(n_params(dims))
    check(lib().ck_toy_sequential_sgd(d, len(d), np.ascontiguousarray(params, np.float64),
                                      np.ascontiguousarray(inputs, np.float64),
                                      np.ascontiguousarray(targets, np.float64), batch, lr, out))
    return out


def check_gradients(dims, params, inputs, targets, batch: int, step: float = 1e-5) -> float:
    """oracle::check_gradients (proj/src/oracle.cpp:358-410) on the GPU: max relative
    error of central finite differences against the analytic gradient."""
    d = np.asarray(dims, np.int32)
    err = C.c_double()
    check(lib().ck_toy_check_gradients(d, len(d), np.ascontiguousarray(params, np.float64),
                                       np.ascontiguousarray(inputs, np.float64),
                                       np.ascontiguousarray(targets, np.float64), batch, step, C.byref(err)))
    return err.value
