"""Python mirror of the reference ``pipesim`` schedule API, backed by libchimera.so.

Names and argument meaning follow proj/include/pipesim/{core,schedgen,analysis,
dessim,perfmodel}.hpp; the C++ host layer behind them lives in
``csrc/host`` and produces byte-identical JSON.  Errors: ``InvalidConfigError``
(status 2) for invalid configurations, ``CKError`` otherwise.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import asdict, dataclass, field
from fractions import Fraction
from typing import List, Optional

import numpy as np

from ._lib import CKError, InvalidConfigError, call_str, check, lib  # noqa: F401

SCHEMES = ("gpipe", "dapple", "gems", "pipedream", "pipedream-2bw", "chimera")
SCALINGS = ("direct", "forward-doubling", "backward-halving")
POLICIES = {"end-of-iteration": 0, "eager-sync": 1, "eager-sync-opt": 2}


@dataclass
class PipelineConfig:
    """proj/include/pipesim/core.hpp:53-69."""
    scheme: str = "chimera"
    D: int = 1
    W: int = 1
    N: int = 1
    B: int = 1
    f: int = 1
    scaling: str = "direct"
    recompute: bool = False

    def workers(self) -> int:
        return self.W * self.D

    def mini_batch(self) -> int:
        return self.B * self.N * self.W

    def to_json(self) -> str:
        return json.dumps(asdict(self))


@dataclass
class CostProfile:
    """proj/include/pipesim/core.hpp:110-126."""
    F_t: float = 1.0
    backward_ratio: float = 2.0
    alpha: float = 0.0
    beta: float = 0.0
    L_grad: float = 1.0
    L_act: float = 1.0
    M_theta: float = 1.0
    M_a: float = 1.0
    M_a_ckpt: float = 1.0
    mem_capacity: float = 1e30
    embed_surcharge: bool = False

    def to_json(self) -> str:
        return json.dumps(asdict(self))


@dataclass
class Task:
    kind: str
    pipeline_id: int
    micro_batch: int
    stage: int
    worker: int
    replica_group: int = 0


@dataclass
class Schedule:
    config: PipelineConfig
    per_worker: List[List[Task]]
    timing: Optional[list] = None
    text: str = field(default="", repr=False)  # canonical JSON as produced by the C++ layer

    @staticmethod
    def from_json(text: str) -> "Schedule":
        d = json.loads(text)
        cfg = PipelineConfig(**d["config"])
        pw = [[Task(**t) for t in wl] for wl in d["per_worker"]]
        return Schedule(cfg, pw, d.get("timing"), text)

    def to_json(self, indent: int = -1) -> str:
        d = {"config": asdict(self.config),
             "per_worker": [[asdict(t) for t in wl] for wl in self.per_worker]}
        if self.timing is not None:
            d["timing"] = self.timing
        return json.dumps(d) if indent < 0 else json.dumps(d, indent=indent)

    def task_count(self) -> int:
        return sum(len(w) for w in self.per_worker)

    def signature(self, worker: int) -> str:
        """order_sig of proj/tests/test_schedgen.cpp:31-41."""
        return " ".join(("B" if t.kind == "Backward" else "F") + f"p{t.pipeline_id}{t.micro_batch}"
                        for t in self.per_worker[worker])


def _cfg(c) -> bytes:
    return (c if isinstance(c, str) else c.to_json()).encode()


def _prof(p) -> bytes:
    if p is None:
        p = CostProfile()
    return p.encode() if isinstance(p, str) else p.to_json().encode()


def _sched(s) -> bytes:
    if isinstance(s, str):
        return s.encode()
    return (s.text or s.to_json()).encode()


def generate_json(config, profile=None, indent: int = 2) -> str:
    """``to_json(schedgen::generate(config, profile), indent)``."""
    return call_str(lib().pipesim_generate, _cfg(config), _prof(profile), indent)


def generate(config, profile=None) -> Schedule:
    """``schedgen::generate`` (schedgen.hpp:92)."""
    return Schedule.from_json(generate_json(config, profile, -1))


def validate_config(config, profile=None) -> List[str]:
    s = call_str(lib().pipesim_validate_config, _cfg(config), _prof(profile))
    return [x for x in s.split("\n") if x]


def validate_dependencies(schedule) -> List[str]:
    s = call_str(lib().pipesim_validate_dependencies, _sched(schedule))
    return [x for x in s.split("\n") if x]


def _workers(schedule) -> int:
    if isinstance(schedule, str):
        return len(json.loads(schedule)["per_worker"])
    return len(schedule.per_worker)


def bubble_ratio_per_worker(schedule, profile=None) -> List[Fraction]:
    n = _workers(schedule)
    num, den = np.zeros(n, np.int64), np.zeros(n, np.int64)
    check(lib().pipesim_bubble_ratio_per_worker(_sched(schedule), _prof(profile), num, den, n))
    return [Fraction(int(a), int(b)) for a, b in zip(num, den)]


def bubble_ratio(schedule, profile=None) -> Fraction:
    r = bubble_ratio_per_worker(schedule, profile)
    return r[0] if r else Fraction(0)


def memory_profile(schedule, profile=None) -> dict:
    n = _workers(schedule)
    ac, wc = np.zeros(n, np.int32), np.zeros(n, np.int32)
    ab, wb = np.zeros(n), np.zeros(n)
    pw, pb = C.c_int(), C.c_double()
    check(lib().pipesim_memory_profile(_sched(schedule), _prof(profile), ac, wc, ab, wb,
                                       C.byref(pw), C.byref(pb), n))
    return {"act_counts": ac.tolist(), "weight_counts": wc.tolist(), "act_bytes": ab.tolist(),
            "weight_bytes": wb.tolist(), "peak_worker": pw.value, "peak_bytes": pb.value}


def simulate(schedule, profile=None, policy: str = "end-of-iteration", zero_comm: bool = False,
             eager_overhead: float = -1.0) -> dict:
    """``dessim::simulate`` (dessim.hpp:58); returns the SimResult as a dict."""
    return json.loads(call_str(lib().pipesim_simulate, _sched(schedule), _prof(profile),
                               POLICIES[policy], int(zero_comm), eager_overhead))


def simulate_timeline(schedule, profile=None, policy: str = "end-of-iteration",
                      eager_overhead: float = -1.0) -> str:
    """The ``pipesim simulate -o <prefix>.json`` document (tools/main.cpp:134-170,367)."""
    return call_str(lib().pipesim_simulate_timeline, _sched(schedule), _prof(profile), POLICIES[policy],
                    eager_overhead)


def gantt(schedule, profile=None, policy: str = "end-of-iteration", svg: bool = False,
          eager_overhead: float = -1.0) -> str:
    """``gantt::render_svg`` / ``render_ascii`` (gantt.hpp:28-31) of dessim::simulate."""
    return call_str(lib().pipesim_gantt, _sched(schedule), _prof(profile), POLICIES[policy], eager_overhead,
                    int(svg))


def gantt_timeline(timeline, profile=None, svg: bool = False) -> str:
    """Gantt chart of a timeline document in the simulate -o schema (e.g. a measured GPU
    iteration from ``gpt.measured_timeline``); ASCII columns are F_t of ``profile``."""
    text = timeline if isinstance(timeline, str) else json.dumps(timeline)
    return call_str(lib().pipesim_gantt_timeline, text.encode(), _prof(profile), int(svg))


def replicas_per_stage(config) -> int:
    return lib().pipesim_replicas_per_stage(_cfg(config))


def critical_path(schedule, profile=None):
    a, b = C.c_int(), C.c_int()
    check(lib().pipesim_critical_path(_sched(schedule), _prof(profile), C.byref(a), C.byref(b)))
    return a.value, b.value


def predict_T(config, profile=None) -> float:
    t = C.c_double()
    check(lib().pipesim_predict_T(_cfg(config), _prof(profile), C.byref(t)))
    return t.value


def analysis_report(schedule, profile=None) -> dict:
    """validate_dependencies, per-worker bubble, steady-state idle, memory profile, free
    regions and critical path of one schedule (pipesim_analysis_report)."""
    return json.loads(call_str(lib().pipesim_analysis_report, _sched(schedule), _prof(profile)))


def plan(P: int, B_hat: int, profile=None, scheme: str = "chimera") -> list:
    """perfmodel::plan (proj/src/perfmodel.cpp:225-298): feasible (W, D, B, N, scaling)
    configurations for P workers and mini-batch B_hat, fastest predicted first."""
    return json.loads(call_str(lib().pipesim_plan, int(P), int(B_hat), _prof(profile), scheme.encode()))


def replay_order(schedule):
    n = sum(len(w) for w in (json.loads(schedule)["per_worker"] if isinstance(schedule, str)
                             else schedule.per_worker))
    w, i = np.zeros(n, np.int32), np.zeros(n, np.int32)
    check(lib().pipesim_replay_order(_sched(schedule), w, i, n))
    return list(zip(w.tolist(), i.tolist()))


def closed_form_bubble(D: int, N: int, f: int = 1) -> Fraction:
    """Paper (D-2f)/(2fN+D-2f); f=1 gives (D-2)/(2N+D-2)."""
    return Fraction(D - 2 * f, 2 * f * N + D - 2 * f)
