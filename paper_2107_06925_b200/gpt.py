"""GPT-2 training under a Chimera schedule on B200 -- Python host mirror of the
C-ABI trainer (``ck_gpt_*`` in include/chimera_ck.h, csrc/cuda/gpt.cu).

    tr = Trainer(PRESETS["gpt2-medium"], P.PipelineConfig("chimera", D=4, W=2, N=4, B=4), lr=1e-4)
    tr.init_params(seed=0)
    tr.set_batch(tokens, labels)      # int32 [W*N*B*seq]
    loss = tr.step()

Everything runs on the GPU through libchimera.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import call_str, check, lib
from .pipesim import PipelineConfig, Schedule, generate_json


class ck_gpt_model(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_layer", "hidden", "heads", "ffn", "seq", "vocab", "vocab_padded",
                                        "causal")] + [("stage_layers", C.POINTER(C.c_int)), ("n_stage_layers", C.c_int)]


_vp = C.c_void_p
_lib.register("ck_gpt_create", C.c_int, [C.POINTER(ck_gpt_model), C.c_char_p, C.c_float, C.c_int, C.c_int,
                                         C.POINTER(_vp)])
_lib.register("ck_gpt_destroy", C.c_int, [_vp])
_lib.register("ck_gpt_layout", C.c_int, [_vp, C.POINTER(_vp)])
_lib.register("ck_gpt_stats", C.c_int, [_vp, C.POINTER(_vp)])
_lib.register("ck_gpt_stage_numel", C.c_int, [_vp, C.c_int, C.POINTER(C.c_longlong)])
_lib.register("ck_gpt_set_params", C.c_int, [_vp, C.c_int, _lib._fp])
_lib.register("ck_gpt_get_params", C.c_int, [_vp, C.c_int, _lib._fp])
_lib.register("ck_gpt_set_batch", C.c_int, [_vp, _vp, _vp, C.c_int])
_lib.register("ck_gpt_step", C.c_int, [_vp, C.POINTER(C.c_float)])
_lib.register("ck_gpt_launch", C.c_int, [_vp])
_lib.register("ck_gpt_begin_iteration", C.c_int, [_vp])
_lib.register("ck_gpt_run_task", C.c_int, [_vp, C.POINTER(C.c_int32)])
_lib.register("ck_gpt_end_iteration", C.c_int, [_vp, C.POINTER(C.c_float)])
_lib.register("ck_gpt_profile_step", C.c_int, [_vp, C.POINTER(_vp)])
_lib.register("ck_gpt_set_graph", C.c_int, [_vp, C.c_int])
_lib.register("ck_gpt_set_sync_policy", C.c_int, [_vp, C.c_int])
_lib.register("ck_gpt_set_cost_profile", C.c_int, [_vp, C.c_char_p])
_lib.register("ck_gpt_sync_plan", C.c_int, [_vp, C.POINTER(_vp)])
_lib.register("ck_gpt_set_optimizer", C.c_int, [_vp, C.c_int, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int])
_lib.register("ck_gpt_stream", _vp, [_vp])
_lib.register("ck_gpt_ipc_handles", C.c_int, [_vp, C.c_char_p, C.c_int])
_lib.register("ck_gpt_connect", C.c_int, [_vp, C.c_char_p, C.c_int, C.c_char_p, C.c_int])
_lib.register("ck_nccl_unique_id", C.c_int, [C.c_char_p, C.c_int])


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().ck_nccl_unique_id(buf, 128))
    return buf.raw


@dataclass(frozen=True)
class GPTShape:
    n_layer: int
    hidden: int
    heads: int
    ffn: int
    seq: int
    vocab: int
    vocab_padded: int
    causal: bool = True
    stage_layers: tuple = ()  # layers per pipeline stage; () = even split

    def flops_per_seq(self) -> float:
        """Algorithmic fwd+bwd FLOPs per sequence:
        72 s L h^2 (1 + s/(6h) + V/(12 L h))  (no recompute credit)."""
        s, L, h, V = self.seq, self.n_layer, self.hidden, self.vocab
        return 72.0 * s * L * h * h * (1 + s / (6.0 * h) + V / (12.0 * L * h))

    def params(self) -> int:
        h, L = self.hidden, self.n_layer
        return L * (12 * h * h + 13 * h) + 2 * self.vocab * h + self.seq * h + 2 * h


# BASELINE.json configs; vocab padded to a multiple of 128.
PRESETS = {
    "tiny": GPTShape(8, 256, 4, 1024, 128, 1024, 1024, True),
    "gpt2-medium": GPTShape(24, 1024, 16, 4096, 1024, 50257, 50304, True),
    "bert48": GPTShape(48, 1024, 16, 4096, 128, 30522, 30592, False),
    "gpt2-1.3b": GPTShape(64, 1280, 20, 5120, 632, 50257, 50304, True),
    "gpt2-32l": GPTShape(32, 1280, 20, 5120, 632, 50257, 50304, True),
}


# LM head + loss cost per FLOP relative to a transformer layer's, measured on B200: the
# head stage's tasks of GPT-2 medium D=4 took 2.27 ms for 3 layers + head against 2.86 ms
# for 7 layers (profiles/timelines/r02_d4n8fd_nobwdfuse_graph.*) -> the head costs 2.5
# layers, 0.67 of its FLOP ratio (one large, efficient N = 50304 GEMM per pass)
HEAD_EFFICIENCY = 0.67


def balanced_partition(shape: GPTShape, config, head_efficiency: float = HEAD_EFFICIENCY) -> tuple:
    """Layers per stage minimising the busiest pipeline worker's load (then the busiest
    stage), counting a layer as 1 and the LM head as head_efficiency x its FLOP ratio
    V / (12 h + 2 s*causal_fraction) to a layer.  Chimera worker w holds stage w of the
    down pipelines and the mirrored stage of the up ones, so the stage carrying the
    head should be shorter than the middle ones.  E.g. GPT-2 medium D=4 (head = 2.5
    layers): (7, 6, 7, 4) loads worker 0 with 7 + 4 + 2.5 and worker 1 with 6 + 7, where
    (7, 7, 7, 3) left worker 0 at 12.5 against worker 1's 14."""
    import itertools
    D, L = config.D, shape.n_layer
    attn = shape.seq * (0.5 if shape.causal else 1.0)
    head = head_efficiency * shape.vocab / (12.0 * shape.hidden + 2.0 * attn)
    sched = json.loads(generate_json(config, None, -1))
    holds = [sorted({t["stage"] for t in wl}) for wl in sched["per_worker"]]
    best, best_key = None, None
    lo, hi = max(1, L // D - 3), L // D + 3
    for parts in itertools.product(range(lo, hi + 1), repeat=D - 1):
        last = L - sum(parts)
        if last < 1:
            continue
        p = tuple(parts) + (last,)
        cost = [p[s] + (head if s == D - 1 else 0.0) for s in range(D)]
        key = (round(max(sum(cost[s] for s in h) for h in holds), 6), round(max(cost), 6), p)
        if best_key is None or key < best_key:
            best, best_key = p, key
    return best


def init_stage(layout_stage: dict, seed: int) -> np.ndarray:
    """N(0, 0.02) matrices/embeddings, zero biases, unit LayerNorm gains; host-side,
    deterministic per (seed, stage) so every process and the oracle agree."""
    rng = np.random.default_rng([seed, layout_stage["stage"]])
    flat = np.zeros(layout_stage["numel"], np.float32)
    for t in layout_stage["tensors"]:
        o, n = t["offset"], t["rows"] * t["cols"]
        if t["init"] == "normal":
            flat[o:o + n] = rng.standard_normal(n) * 0.02
        elif t["init"] == "one":
            flat[o:o + n] = 1.0
    return flat


def synthetic_batch(shape: GPTShape, n_samples: int, seed: int = 0):
    """i.i.d. uniform tokens; labels = next token (causal LM) -- SURVEY.md §8(d)."""
    rng = np.random.default_rng(seed)
    seqs = rng.integers(0, shape.vocab, size=(n_samples, shape.seq + 1), dtype=np.int64)
    return (np.ascontiguousarray(seqs[:, :-1].reshape(-1), dtype=np.int32),
            np.ascontiguousarray(seqs[:, 1:].reshape(-1), dtype=np.int32))


class Trainer:
    """Chimera (or GPipe / 1F1B) training of a GPT-2 shape for logical ranks
    [first_rank, first_rank + n_ranks) on the current CUDA device."""

    def __init__(self, shape: GPTShape, schedule, lr: float, first_rank: int = 0, n_ranks: int | None = None):
        if isinstance(schedule, PipelineConfig):
            text = generate_json(schedule, None, -1)
        elif isinstance(schedule, Schedule):
            text = schedule.text or schedule.to_json()
        else:
            text = schedule
        self.schedule_text = text
        cfg = json.loads(text)["config"]
        self.config = PipelineConfig(**cfg)
        self.shape = shape
        if n_ranks is None:
            n_ranks = cfg["W"] * cfg["D"] - first_rank
        self._parts = (C.c_int * max(1, len(shape.stage_layers)))(*shape.stage_layers)
        mdl = ck_gpt_model(shape.n_layer, shape.hidden, shape.heads, shape.ffn, shape.seq, shape.vocab,
                           shape.vocab_padded, int(shape.causal), self._parts, len(shape.stage_layers))
        h = C.c_void_p()
        check(lib().ck_gpt_create(C.byref(mdl), text.encode(), lr, first_rank, n_ranks, C.byref(h)))
        self._h = h
        self.layout = json.loads(call_str(lib().ck_gpt_layout, h))

    def close(self):
        if getattr(self, "_h", None):
            lib().ck_gpt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stages(self):
        return [st["stage"] for st in self.layout]

    def init_params(self, seed: int = 0):
        for st in self.layout:
            self.set_params(st["stage"], init_stage(st, seed))

    def set_params(self, stage: int, flat):
        flat = np.ascontiguousarray(flat, np.float32)
        check(lib().ck_gpt_set_params(self._h, stage, flat))

    def get_params(self, stage: int) -> np.ndarray:
        n = C.c_longlong()
        check(lib().ck_gpt_stage_numel(self._h, stage, C.byref(n)))
        out = np.zeros(n.value, np.float32)
        check(lib().ck_gpt_get_params(self._h, stage, out))
        return out

    def set_batch(self, tokens, labels):
        """Host arrays (numpy int32) or device tensors (anything with data_ptr())."""
        if hasattr(tokens, "data_ptr"):
            check(lib().ck_gpt_set_batch(self._h, C.c_void_p(tokens.data_ptr()), C.c_void_p(labels.data_ptr()),
                                         int(not tokens.is_cuda)))
        else:
            t = np.ascontiguousarray(tokens, np.int32)
            l = np.ascontiguousarray(labels, np.int32)
            check(lib().ck_gpt_set_batch(self._h, t.ctypes.data_as(C.c_void_p), l.ctypes.data_as(C.c_void_p), 1))

    def step(self) -> float:
        loss = C.c_float()
        check(lib().ck_gpt_step(self._h, C.byref(loss)))
        return loss.value

    # Engine-style driving (reference oracle.cpp:304-356): the host walks the schedule.
    def begin_iteration(self):
        check(lib().ck_gpt_begin_iteration(self._h))

    def run_task(self, task):
        """task = (kind, pipeline_id, micro_batch, stage, worker, replica_group) as in
        pipesim::Task (kind 0 Forward, 1 Backward); runs every local replica of it.
        Raises CKError (status 3) if its input activation / gradient is missing."""
        arr = (C.c_int32 * 6)(*[int(x) for x in task])
        check(lib().ck_gpt_run_task(self._h, arr))

    def end_iteration(self) -> float:
        loss = C.c_float()
        check(lib().ck_gpt_end_iteration(self._h, C.byref(loss)))
        return loss.value

    def run_iteration(self, tasks) -> float:
        """One iteration from an explicit task sequence (e.g. pipesim replay order)."""
        self.begin_iteration()
        for t in tasks:
            self.run_task(t)
        return self.end_iteration()

    def profile_step(self) -> dict:
        """One iteration with per-task GPU timestamps and message-wait brackets (see
        measured_bubble): captured and replayed as a CUDA graph in a single-process
        trainer once a graph exists (the GPU, not the host, paces the tasks), issued
        eagerly when the trainer spans processes."""
        return json.loads(call_str(lib().ck_gpt_profile_step, self._h))

    def launch(self):
        check(lib().ck_gpt_launch(self._h))

    def set_sync_policy(self, policy: str):
        """'end-of-iteration' | 'eager-sync' (default) | 'eager-sync-opt' (dessim.hpp:27)."""
        check(lib().ck_gpt_set_sync_policy(self._h, {"end-of-iteration": 0, "eager-sync": 1,
                                                      "eager-sync-opt": 2}[policy]))

    def set_cost_profile(self, profile):
        """Plan the gradient sync (eager-sync-opt set, collective order) on this
        CostProfile -- normally the measured one; identical on every process."""
        check(lib().ck_gpt_set_cost_profile(self._h, profile.to_json().encode()))

    def set_optimizer(self, kind: str = "adamw", beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                      weight_decay: float = 0.0, zero: bool = False):
        """'sgd' (the reference's, default) or 'adamw'; zero=True shards the AdamW moments
        over the processes holding each stage (ZeRO-1).  After connect()."""
        check(lib().ck_gpt_set_optimizer(self._h, {"sgd": 0, "adamw": 1}[kind], beta1, beta2, eps, weight_decay,
                                         int(zero)))

    def sync_plan(self) -> dict:
        return json.loads(call_str(lib().ck_gpt_sync_plan, self._h))

    def use_graph(self, on: bool):
        check(lib().ck_gpt_set_graph(self._h, int(on)))

    def stream_handle(self) -> int:
        return lib().ck_gpt_stream(self._h) or 0

    def stats(self) -> dict:
        return json.loads(call_str(lib().ck_gpt_stats, self._h))

    def ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().ck_gpt_ipc_handles(self._h, buf, 128))
        return buf.raw

    def connect(self):
        """Multi-process wiring over torch.distributed (any backend; gloo is enough):
        all-gather the CUDA-IPC handles of every process's inbox/outbox and broadcast
        one NCCL unique id, then open the peer mappings and the stage communicators."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(), dist.get_rank()
        blobs = [None] * world
        dist.all_gather_object(blobs, self.ipc_handles())
        # one NCCL id per stage: each stage communicator is initialised on its own (no
        # world communicator), see ck_gpt_connect
        uid = [b"".join(nccl_unique_id() for _ in range(self.config.D)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        allb = b"".join(blobs)
        check(lib().ck_gpt_connect(self._h, allb, len(allb), uid[0], len(uid[0])))


def measured_bubble(profile: dict, ranks=None) -> dict:
    """Per-rank idle fraction of a profiled iteration with the dessim definition
    (proj/src/dessim.cpp:168-181): idle_w = (span_end - span_start) - busy_w
    over the iteration span, busy_w = sum of the rank's task durations minus the time
    its stream sat waiting inside a task for an incoming message (`stall_ms`, measured
    by events around each wait) -- dessim's busy time is compute only."""
    tasks = profile["tasks"]
    lo = min(t["start_ms"] for t in tasks)
    hi = max(t["end_ms"] for t in tasks)
    out = {}
    for r in sorted({t["rank"] for t in tasks} if ranks is None else ranks):
        busy = sum(t["end_ms"] - t["start_ms"] - t.get("stall_ms", 0.0) for t in tasks if t["rank"] == r)
        out[r] = ((hi - lo) - busy) / (hi - lo)
    return {"per_rank": out, "span_ms": hi - lo}


def timeline_json(profile: dict, schedule_text: str) -> str:
    """Measured timeline in the reference's Schedule JSON layout with `timing`
    (proj/src/core.cpp:205-216), so reference tooling (bubble_ratio, gantt) can read it.
    Times are milliseconds from the iteration start; replica 0's ranks only."""
    sched = json.loads(schedule_text)
    D = sched["config"]["D"]
    spans = {(t["rank"] % D, t["kind"], t["pipeline"], t["micro"], t["stage"]): (t["start_ms"], t["end_ms"])
             for t in profile["tasks"] if t["rank"] < D}
    timing = []
    for w, wl in enumerate(sched["per_worker"]):
        row = []
        for t in wl:
            a, b = spans.get((w, t["kind"], t["pipeline_id"], t["micro_batch"], t["stage"]), (0.0, 0.0))
            row.append({"start": a, "end": b})
        timing.append(row)
    sched["timing"] = timing
    return json.dumps(sched)


def replay_measured(profile: dict, schedule_text: str, p2p_ms: float = 0.0) -> dict:
    """The reference's list-scheduling semantics (proj/src/listsched.hpp:52-163: a task
    starts when its worker is free and its data predecessors F(s-1) / B(s+1) / F(s) have
    ended, + p2p on cross-worker edges) replayed with the MEASURED compute time of every
    task (span minus message stalls) instead of uniform F_t / B_t: the bubble this
    executor's schedule would have if it added no overhead beyond its own task times.
    Measured bubble vs this isolates the executor's overhead from stage-cost imbalance
    (which the uniform-cost prediction ignores).  Replica 0's ranks (rank = worker)."""
    sched = json.loads(schedule_text)
    D = sched["config"]["D"]
    dur = {(t["rank"], t["kind"], t["pipeline"], t["micro"], t["stage"]):
           max(0.0, t["end_ms"] - t["start_ms"] - t.get("stall_ms", 0.0)) for t in profile["tasks"] if t["rank"] < D}
    pw = sched["per_worker"]
    where = {}
    for w, wl in enumerate(pw):
        for t in wl:
            where.setdefault((t["kind"], t["pipeline_id"], t["micro_batch"], t["stage"]), w)
    end, free, head = {}, [0.0] * len(pw), [0] * len(pw)
    left = sum(len(wl) for wl in pw)
    while left:
        progressed = False
        for w, wl in enumerate(pw):
            if head[w] >= len(wl):
                continue
            t = wl[head[w]]
            k, p, m, st = t["kind"], t["pipeline_id"], t["micro_batch"], t["stage"]
            deps = [("Forward", p, m, st - 1)] if k == "Forward" and st > 0 else \
                   ([("Backward", p, m, st + 1)] if st + 1 < D else []) + [("Forward", p, m, st)] if k == "Backward" else []
            ready, start = True, free[w]
            for d in deps:
                if d not in where:
                    continue
                if d not in end:
                    ready = False
                    break
                start = max(start, end[d] + (p2p_ms if where[d] != w else 0.0))
            if not ready:
                continue
            e = start + dur.get((w, k, p, m, st), 0.0)
            end[(k, p, m, st)] = e
            free[w] = e
            head[w] += 1
            left -= 1
            progressed = True
        if not progressed:
            raise ValueError("replay_measured: dependency cycle")
    span = max(free)
    busy = [sum(dur.get((w, t["kind"], t["pipeline_id"], t["micro_batch"], t["stage"]), 0.0) for t in wl)
            for w, wl in enumerate(pw)]
    per = [(span - b) / span for b in busy]
    return {"per_worker": per, "mean": sum(per) / len(per), "span_ms": span}


def measured_timeline(profile: dict, schedule_text: str, policy: str = "eager-sync") -> str:
    """A profiled GPU iteration (Trainer.profile_step) as the reference's
    ``pipesim simulate -o`` timeline document (tools/main.cpp:134-170): replica 0's
    ranks, milliseconds from the first task start, dessim's idle definition, one
    allreduce event per holder worker of each stage sync.  Render it with
    ``pipesim.gantt_timeline`` (the same code path as the simulated charts)."""
    sched = json.loads(schedule_text)
    D = sched["config"]["D"]
    spans = {(t["rank"], t["kind"], t["pipeline"], t["micro"], t["stage"]): (t["start_ms"], t["end_ms"])
             for t in profile["tasks"] if t["rank"] < D}
    t0 = min(a for a, _ in spans.values())
    events, busy = [], [0.0] * D
    for w, wl in enumerate(sched["per_worker"]):
        for t in wl:
            a, b = spans[(w, t["kind"], t["pipeline_id"], t["micro_batch"], t["stage"])]
            events.append({"worker": w, "kind": t["kind"], "pipeline_id": t["pipeline_id"],
                           "micro_batch": t["micro_batch"], "stage": t["stage"], "start": a - t0, "end": b - t0})
            busy[w] += b - a
    compute = max(e["end"] for e in events)
    ar = [{"worker": r, "stage": c["stage"], "eager": c["eager"], "start": c["start_ms"] - t0,
           "end": c["end_ms"] - t0} for c in profile.get("allreduce", []) for r in c["ranks"] if r < D]
    makespan = max([compute] + [e["end"] for e in ar])
    doc = {"policy": policy, "makespan": makespan, "compute_makespan": compute,
           "allreduce_exposed": makespan - compute, "per_worker_idle": [compute - b for b in busy],
           "events": events, "allreduce": ar}
    return json.dumps(doc, indent=2) + "\n"


def smoke():
    """One Chimera iteration of the tiny GPT on cuda:0 vs the numpy oracle."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import gpt_oracle as O
    shape = PRESETS["tiny"]
    cfg = PipelineConfig("chimera", 4, 1, 4, 1, 1)
    tr = Trainer(shape, cfg, lr=0.1)
    tr.init_params(0)
    p0 = [tr.get_params(s).astype(np.float64) for s in range(cfg.D)]
    tok, lab = synthetic_batch(shape, cfg.mini_batch(), 1)
    tr.set_batch(tok, lab)
    loss = tr.step()
    oshape = O.Shape(**{k: getattr(shape, k) for k in O.Shape.__dataclass_fields__})
    _, ref_loss, _, _ = O.run_iteration(json.loads(tr.schedule_text), oshape, p0, tok, lab, 0.1)
    rel = abs(loss - ref_loss) / abs(ref_loss)
    assert rel < 2e-2, (loss, ref_loss)
    print(f"smoke: gpt tiny chimera D=4 loss={loss:.5f} oracle={ref_loss:.5f} rel={rel:.1e}")
    tr.close()
