"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the two compiled checkers.

``RefLib``  -> oracle/_ref/libpipesim_ref.so (the reference itself, ref_shim.cpp)
``ToyLib``  -> oracle/_build/libtoy_oracle.so (toy_oracle.c restatement)
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpipesim_ref.so")
TOY_SO = os.path.join(HERE, "_build", "libtoy_oracle.so")
REF_SRC = "/root/reference/proj"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile the C restatement (always) and oracle/_ref (when the reference is mounted)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    if ref and os.path.isdir(REF_SRC):
        subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "ref", "reftests"])


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def n_params(dims) -> int:
    return sum(dims[s] * dims[s + 1] + dims[s + 1] for s in range(len(dims) - 1))


def tasks_of(schedule: dict):
    """Schedule JSON (reference to_json layout) -> (counts int32[W], tasks int32[T,6])."""
    kinds = {"Forward": 0, "Backward": 1}
    counts, rows = [], []
    for wl in schedule["per_worker"]:
        counts.append(len(wl))
        for t in wl:
            rows.append([kinds.get(t["kind"], 9), t["pipeline_id"], t["micro_batch"], t["stage"],
                         t["worker"], t["replica_group"]])
    return (np.asarray(counts, dtype=np.int32),
            np.asarray(rows if rows else np.zeros((0, 6)), dtype=np.int32).reshape(-1, 6))


class RefLib:
    """The unmodified reference library (proj/src/*.cpp) behind ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` with /root/reference mounted")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_generate.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_validate_config.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_validate_dependencies.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_bubble_ratio_per_worker.argtypes = [C.c_char_p, C.c_char_p, _lp, _lp, C.c_int]
        L.ref_memory_profile.argtypes = [C.c_char_p, C.c_char_p, _ip, _ip, _dp, _dp,
                                         C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_int]
        L.ref_simulate.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_double,
                                   C.POINTER(C.c_void_p)]
        L.ref_replicas_per_stage.argtypes = [C.c_char_p]
        L.ref_gantt.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_simulate_timeline.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_critical_path.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_predict_T.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
        L.ref_analysis_report.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_plan.argtypes = [C.c_int, C.c_longlong, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_toy_make_model.argtypes = [_ip, C.c_int, C.c_uint64, _dp]
        L.ref_toy_make_batch.argtypes = [_ip, C.c_int, C.c_int, C.c_uint64, _dp, _dp]
        L.ref_toy_run_iteration.argtypes = [C.c_char_p, _ip, C.c_int, _dp, _dp, _dp, C.c_int,
                                            C.c_double, _dp, _ip, C.c_int]
        L.ref_toy_sequential_sgd.argtypes = [_ip, C.c_int, _dp, _dp, _dp, C.c_int, C.c_double, _dp]
        L.ref_toy_check_gradients.argtypes = [_ip, C.c_int, _dp, _dp, _dp, C.c_int,
                                              C.POINTER(C.c_double)]

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def _str(self, fn, *args) -> str:
        out = C.c_void_p()
        self._chk(fn(*args, C.byref(out)))
        s = C.cast(out, C.c_char_p).value.decode()
        self.L.ref_free(out)
        return s

    def generate(self, cfg_json: str, prof_json: str, indent: int = 2) -> str:
        return self._str(self.L.ref_generate, cfg_json.encode(), prof_json.encode(), indent)

    def validate_config(self, cfg_json: str, prof_json: str):
        s = self._str(self.L.ref_validate_config, cfg_json.encode(), prof_json.encode())
        return [x for x in s.split("\n") if x]

    def validate_dependencies(self, sched_json: str):
        s = self._str(self.L.ref_validate_dependencies, sched_json.encode())
        return [x for x in s.split("\n") if x]

    def bubble_per_worker(self, sched_json: str, prof_json: str, workers: int):
        n = np.zeros(workers, np.int64)
        d = np.zeros(workers, np.int64)
        self._chk(self.L.ref_bubble_ratio_per_worker(sched_json.encode(), prof_json.encode(), n, d,
                                                     workers))
        return [(int(a), int(b)) for a, b in zip(n, d)]

    def memory_profile(self, sched_json: str, prof_json: str, workers: int):
        ac = np.zeros(workers, np.int32)
        wc = np.zeros(workers, np.int32)
        ab = np.zeros(workers)
        wb = np.zeros(workers)
        pw, pb = C.c_int(), C.c_double()
        self._chk(self.L.ref_memory_profile(sched_json.encode(), prof_json.encode(), ac, wc, ab, wb,
                                            C.byref(pw), C.byref(pb), workers))
        return {"act_counts": ac.tolist(), "weight_counts": wc.tolist(), "act_bytes": ab.tolist(),
                "weight_bytes": wb.tolist(), "peak_worker": pw.value, "peak_bytes": pb.value}

    def simulate(self, sched_json: str, prof_json: str, policy: int = 0, zero_comm: bool = False,
                 eager_overhead: float = -1.0) -> dict:
        return json.loads(self._str(self.L.ref_simulate, sched_json.encode(), prof_json.encode(),
                                    policy, int(zero_comm), eager_overhead))

    def gantt(self, sched_json: str, prof_json: str, policy: int = 0, eps: float = -1.0,
              svg: bool = False) -> str:
        return self._str(self.L.ref_gantt, sched_json.encode(), prof_json.encode(), policy, C.c_double(eps),
                         int(svg))

    def simulate_timeline(self, sched_json: str, prof_json: str, policy: int = 0, eps: float = -1.0) -> str:
        return self._str(self.L.ref_simulate_timeline, sched_json.encode(), prof_json.encode(), policy,
                         C.c_double(eps))

    def replicas_per_stage(self, cfg_json: str) -> int:
        return self.L.ref_replicas_per_stage(cfg_json.encode())

    def critical_path(self, sched_json: str, prof_json: str):
        a, b = C.c_int(), C.c_int()
        self._chk(self.L.ref_critical_path(sched_json.encode(), prof_json.encode(), C.byref(a),
                                           C.byref(b)))
        return a.value, b.value

    def predict_T(self, cfg_json: str, prof_json: str) -> float:
        t = C.c_double()
        self._chk(self.L.ref_predict_T(cfg_json.encode(), prof_json.encode(), C.byref(t)))
        return t.value

    def analysis_report(self, sched_json: str, prof_json: str) -> dict:
        return json.loads(self._str(self.L.ref_analysis_report, sched_json.encode(), prof_json.encode()))

    def plan(self, P: int, B_hat: int, prof_json: str, scheme: str = "chimera") -> list:
        return json.loads(self._str(self.L.ref_plan, int(P), int(B_hat), prof_json.encode(), scheme.encode()))

    # ToyModel oracle (proj/src/oracle.cpp)
    def make_model(self, dims, seed):
        d = np.asarray(dims, np.int32)
        out = np.zeros(n_params(dims))
        self._chk(self.L.ref_toy_make_model(d, len(d), seed, out))
        return out

    def make_batch(self, dims, size, seed):
        d = np.asarray(dims, np.int32)
        x = np.zeros(size * dims[0])
        t = np.zeros(size * dims[-1])
        self._chk(self.L.ref_toy_make_batch(d, len(d), size, seed, x, t))
        return x, t

    def run_iteration(self, sched_json, dims, params, x, t, batch, lr, workers):
        d = np.asarray(dims, np.int32)
        out = np.zeros_like(params)
        peak = np.zeros(workers, np.int32)
        self._chk(self.L.ref_toy_run_iteration(sched_json.encode(), d, len(d), params, x, t, batch,
                                               lr, out, peak, workers))
        return out, peak.tolist()

    def sequential_sgd(self, dims, params, x, t, batch, lr):
        d = np.asarray(dims, np.int32)
        out = np.zeros_like(params)
        self._chk(self.L.ref_toy_sequential_sgd(d, len(d), params, x, t, batch, lr, out))
        return out

    def check_gradients(self, dims, params, x, t, batch):
        d = np.asarray(dims, np.int32)
        e = C.c_double()
        self._chk(self.L.ref_toy_check_gradients(d, len(d), params, x, t, batch, C.byref(e)))
        return e.value


class ToyLib:
    """toy_oracle.c -- the plain-C restatement of the reference ToyModel engine."""

    def __init__(self, path: str = TOY_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        L.toy_make_model.argtypes = [_ip, C.c_int, C.c_uint64, _dp]
        L.toy_make_batch.argtypes = [_ip, C.c_int, C.c_int, C.c_uint64, _dp, _dp]
        L.toy_list_schedule.argtypes = [C.c_int, _ip, _ip, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_int, _dp, _dp, C.POINTER(C.c_double)]
        L.toy_run_iteration.argtypes = [C.c_int] * 6 + [_ip, _ip, _ip, C.c_int, _dp, _dp, _dp,
                                                        C.c_int, C.c_double, _dp, _ip]
        L.toy_sequential_sgd.argtypes = [_ip, C.c_int, _dp, _dp, _dp, C.c_int, C.c_double, _dp]
        L.toy_max_relative_diff.argtypes = [_ip, C.c_int, _dp, _dp]
        L.toy_max_relative_diff.restype = C.c_double

    def make_model(self, dims, seed):
        d = np.asarray(dims, np.int32)
        out = np.zeros(n_params(dims))
        assert self.L.toy_make_model(d, len(d), seed, out) == 0
        return out

    def make_batch(self, dims, size, seed):
        d = np.asarray(dims, np.int32)
        x = np.zeros(size * dims[0])
        t = np.zeros(size * dims[-1])
        assert self.L.toy_make_batch(d, len(d), size, seed, x, t) == 0
        return x, t

    def list_schedule(self, schedule: dict, f_dur=1.0, b_dur=2.0, p2p_fwd=0.0, p2p_bwd=0.0,
                      relaxed=False):
        counts, tasks = tasks_of(schedule)
        n = int(counts.sum())
        st, en, mk = np.zeros(n), np.zeros(n), C.c_double()
        rc = self.L.toy_list_schedule(len(counts), counts, np.ascontiguousarray(tasks.reshape(-1)),
                                      f_dur, b_dur, p2p_fwd, p2p_bwd, int(relaxed), st, en, C.byref(mk))
        if rc:
            raise RuntimeError("cyclic dependency")
        return st, en, mk.value

    def run_iteration(self, schedule: dict, dims, params, x, t, lr):
        cfg = schedule["config"]
        counts, tasks = tasks_of(schedule)
        batch = cfg["B"] * cfg["N"] * cfg["W"]
        halved = int(cfg["scheme"] == "chimera" and cfg["scaling"] == "backward-halving"
                     and cfg["N"] > cfg["D"])
        d = np.asarray(dims, np.int32)
        out = np.zeros_like(params)
        peak = np.zeros(len(counts), np.int32)
        rc = self.L.toy_run_iteration(cfg["D"], cfg["W"], cfg["N"], cfg["B"], halved, len(counts),
                                      counts, np.ascontiguousarray(tasks.reshape(-1)), d, len(d),
                                      params, x, t, batch, lr, out, peak)
        if rc:
            raise RuntimeError(f"toy oracle error {rc}")
        return out, peak.tolist()

    def sequential_sgd(self, dims, params, x, t, batch, lr):
        d = np.asarray(dims, np.int32)
        out = np.zeros_like(params)
        assert self.L.toy_sequential_sgd(d, len(d), params, x, t, batch, lr, out) == 0
        return out

    def max_relative_diff(self, dims, a, b) -> float:
        d = np.asarray(dims, np.int32)
        return self.L.toy_max_relative_diff(d, len(d), np.ascontiguousarray(a), np.ascontiguousarray(b))
