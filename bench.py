"""Chimera-B200 benchmark: GPT-2 training throughput under a Chimera schedule.

Workload (BASELINE.json `metric` "GPT-2 seqs/sec at D=8" -> configs[3]): GPT-2 1.3B
(64 layers, h=1280, 20 heads, s=632, V=50257), Chimera D=8 with N=32 micro-batches of
B=2 sequences (B 1-2), forward doubling + recompute -> 8 logical
ranks, 64 sequences per iteration.  At --gpus G the 8 ranks are spread over G GPUs
(G | 8); one process per GPU under torchrun.  A "step" is one full training iteration
(all micro-batches forward+backward, stage gradient allreduce, SGD update) on
synthetic tokens and random-init weights.  `--config gpt2-medium` runs configs[1]
(GPT-2 medium D=4 W=2) as a secondary line; bert48 / q4* the other configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  `value` = sequences/s with inputs resident in HBM
(device-timed, CUDA events on the trainer stream, max over ranks); `e2e` = the same
through the public API with the H2D copy of each step's tokens/labels from pinned host
memory and the D2H loss read inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GPT-2 seqs/sec at D=8 on 8×B200; bubble ratio vs (D-2)/(2N+D-2)"
# BASELINE.json configs (the default, configs[1], is the one the driver measures).
CONFIGS = {
    "gpt2-medium": ("gpt2-medium", dict(scheme="chimera", D=4, W=2, N=4, B=4, f=1, scaling="direct"),
                    "GPT-2 medium Chimera D=4 N=4 W=2 B=4 (BASELINE configs[1])"),
    # one pipeline (W=1) of configs[1]'s model: with --gpus 4 every logical rank owns a GPU,
    # so the per-worker bubble is observable (closed form 1/4 at N=4, 1/9 at N=8)
    "gpt2-medium-d4": ("gpt2-medium", dict(scheme="chimera", D=4, W=1, N=4, B=4, f=1, scaling="direct"),
                       "GPT-2 medium Chimera D=4 N=4 W=1 B=4 (configs[1] model, one pipeline pair)"),
    "gpt2-medium-d4-n8fd": ("gpt2-medium", dict(scheme="chimera", D=4, W=1, N=8, B=4, f=1,
                                                scaling="forward-doubling"),
                            "GPT-2 medium Chimera D=4 N=8 W=1 B=4 forward-doubling + recompute (configs[1] model)"),
    "gpt2-1.3b-d4": ("gpt2-1.3b", dict(scheme="chimera", D=4, W=1, N=16, B=2, f=1, scaling="forward-doubling"),
                     "GPT-2 1.3B s=632 Chimera D=4 N=16 B=2 forward-doubling + recompute (configs[3] model, 4 stages)"),
    "gpt2-medium-d4-n8bh": ("gpt2-medium", dict(scheme="chimera", D=4, W=1, N=8, B=4, f=1,
                                                scaling="backward-halving"),
                            "GPT-2 medium Chimera D=4 N=8 W=1 B=4 backward-halving (configs[1] model)"),
    "bert48": ("bert48", dict(scheme="chimera", D=8, W=1, N=8, B=8, f=1, scaling="direct"),
               "Bert-48 shape (bidirectional, dense MLM head) Chimera D=8 N=8 B=8 (BASELINE configs[2])"),
    "gpt2-1.3b": ("gpt2-1.3b", dict(scheme="chimera", D=8, W=1, N=32, B=2, f=1, scaling="forward-doubling"),
                  "GPT-2 1.3B s=632 Chimera D=8 N=32 B=2 forward-doubling + recompute (BASELINE configs[3])"),
    "q4": ("gpt2-32l", dict(scheme="chimera", D=8, W=1, N=16, B=1, f=2, scaling="direct"),
           "GPT-2 32-layer s=632 Chimera f=2 (4 pipelines) D=8 N=16 (BASELINE configs[4])"),
    "q4-gpipe": ("gpt2-32l", dict(scheme="gpipe", D=8, W=1, N=16, B=1, f=1, scaling="direct"),
                 "GPT-2 32-layer s=632 GPipe D=8 N=16 (configs[4] baseline)"),
    "q4-dapple": ("gpt2-32l", dict(scheme="dapple", D=8, W=1, N=16, B=1, f=1, scaling="direct"),
                  "GPT-2 32-layer s=632 1F1B/DAPPLE D=8 N=16 (configs[4] baseline)"),
}
DEFAULT_CONFIG = "gpt2-1.3b"
SHAPE_NAME, CFG, WORKLOAD = CONFIGS[DEFAULT_CONFIG]


def progress(msg):
    """Phase marks on stderr (the one JSON line stays alone on stdout)."""
    if int(os.environ.get("RANK", "0")) == 0:
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class PortStages:
    """The numpy fp64 port of the reference Engine (oracle/gpt_oracle.py; the reference
    itself has no transformer) timed stage by stage on ONE sequence of the workload:
    stage s forward + backward (stage 0 from tokens, stage D-1 with the LM head and
    cross-entropy), all host BLAS threads.  A sequence's full fwd+bwd time is the sum
    over the D stages -- measured, not FLOP-scaled."""

    def __init__(self, shape):
        import numpy as np
        from oracle import gpt_oracle as O
        self.np, self.O = np, O
        self.m = O.Shape(**shape.__dict__)
        self.D = CFG["D"]
        self.models = [O.StageModel(self.m, self.D, st) for st in range(self.D)]
        tok, lab = O.synthetic_tokens(self.m, 1, 1)
        self.tok, self.lab = tok, lab
        self.times = {}
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=os.cpu_count()):  # spin up the BLAS threads untimed
            w = np.ones((512, 512))
            for _ in range(4):
                w = w @ w * 1e-3

    def time_stage(self, st):
        import time as _t
        np, O, m = self.np, self.O, self.m
        sm = self.models[st]
        # this stage's parameters only (O.init_params' per-stage stream): the whole 1.3B
        # model in fp64 would hold ~10 GB of host memory beside the GPU trainer
        rng = np.random.default_rng([0, st])
        flat = np.zeros(sm.total)
        for _, o, r, c, init in sm.layout:
            if init == "normal":
                flat[o:o + r * c] = rng.standard_normal(r * c) * 0.02
            elif init == "one":
                flat[o:o + r * c] = 1.0
        P = O.unpack(flat, sm.layout)
        x = self.tok if st == 0 else np.random.default_rng(st).standard_normal((m.seq, m.hidden))
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=os.cpu_count()):  # torchrun exports OMP_NUM_THREADS=1
            t0 = _t.perf_counter()
            y, _, cache = sm.forward(P, x, self.lab, 1, 1.0 / m.seq)
            G = {k: np.zeros_like(v) for k, v in P.items()}
            sm.backward(P, G, cache, None if st == self.D - 1 else np.ones_like(y) * 1e-3, 1)
            dt = _t.perf_counter() - t0
        self.times.setdefault(st, []).append(dt)
        return dt

    def seqs_per_s(self):
        per = [sum(v) / len(v) for _, v in sorted(self.times.items())]
        mean = sum(per) / len(per)
        return 1.0 / (sum(per) + mean * (self.D - len(per)))


def threads_used():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count()


def reference_toy_iteration():
    """The reference library itself (oracle/_ref, proj/src/oracle.cpp:304-356, single-
    threaded by design) on SURVEY.md §8(d) CPU-baseline item 1: run_iteration on the
    Chimera D=4 N=4 schedule, dims {256 x 5}, micro-batch B = 128 (B_hat = 512; the survey's
    probe: 0.546 s / iteration) -- seconds per iteration."""
    import time as _t
    try:
        from oracle.libs import RefLib, ref_available
        if not ref_available():
            return None
        from paper_2107_06925_b200 import pipesim as P
        R = RefLib()
        cfg = P.PipelineConfig("chimera", 4, 1, 4, 128, 1)  # B_hat = 512
        text = R.generate(cfg.to_json(), P.CostProfile().to_json(), -1)
        dims = [256] * 5
        p = R.make_model(dims, 42)
        x, t = R.make_batch(dims, 512, 100)
        t0 = _t.perf_counter()
        R.run_iteration(text, dims, p, x, t, 512, 0.05, 4)
        dt = _t.perf_counter() - t0
        flops = 6.0 * 512 * sum(dims[i] * dims[i + 1] for i in range(4))
        return {"s_per_iteration": round(dt, 4), "gflops": round(flops / dt / 1e9, 3), "cores": 1,
                "config": "Chimera D=4 N=4 B=128 W=1, dims {256 x 5}, B_hat = 512 (ToyModel, fp64 + Kahan)"}
    except Exception as e:  # the checker is optional on a box without the built reference
        return {"unavailable": str(e)[:200]}


def cpu_port_sample(shape, stages=None):
    """cpu_baseline: one sequence through every pipeline stage (fwd+bwd, incl. the LM
    head) on the numpy port, all host cores; plus the reference library's own ToyModel
    iteration on 1 core."""
    ps = PortStages(shape)
    for st in (stages if stages is not None else range(ps.D)):
        ps.time_stage(st)
    v = ps.seqs_per_s()
    per = {st: round(sum(t) / len(t), 3) for st, t in sorted(ps.times.items())}
    return {"value": v, "unit": "seqs/s", "cores": threads_used(), "kind": "port", "cpu_model": cpu_model(),
            "sample": f"numpy fp64 port of the reference Engine: ONE sequence of the workload, forward + backward "
                      f"through each of the {ps.D} stages (s per stage {per}); seqs/s = 1 / sum over stages",
            "reference_toy": reference_toy_iteration()}


def roofline_shapes(shape, cfg, bwd_pair_frac=None):
    """(M, N, K, a_mn, b_mn, weight): every stage-GEMM shape one iteration runs, weighted by
    how often it runs per layer-micro-batch.  Forward doubling + recompute (configs[3]):
    fused forward pairs on 2M rows (weight 1/2 per micro-batch); the backward of a pair
    (recompute forward, activation gradient, weight gradient with K = rows) on 2M rows
    when fused (bwd_pair_frac of the micro-batches, from the trainer's stats; default
    all) else on M rows; the LM head's GEMMs with weight 1/L (one head per L layers)."""
    M, h, f, Vp = cfg["B"] * shape.seq, shape.hidden, shape.ffn, shape.vocab_padded
    fd = cfg["scaling"] == "forward-doubling" and cfg["N"] > cfg["D"]
    fp = (1.0 if bwd_pair_frac is None else bwd_pair_frac) if fd else 0.0
    layer = lambda Mm: [(Mm, 3 * h, h), (Mm, h, h), (Mm, f, h), (Mm, h, f)]
    dgrad = lambda Mm: [(Mm, h, 3 * h), (Mm, h, h), (Mm, h, f), (Mm, f, h)]
    wgrad = lambda Kk: [(3 * h, h, Kk), (h, h, Kk), (f, h, Kk), (h, f, Kk)]
    out = []
    if fd:
        out += [(Mm, N, K, 0, 0, 0.5) for (Mm, N, K) in layer(2 * M)]  # fused pair forward
    else:
        out += [(Mm, N, K, 0, 0, 1.0) for (Mm, N, K) in layer(M)]
    for rows, wt in ((2 * M, 0.5 * fp), (M, 1.0 - fp)) if fd else ((M, 1.0),):
        if wt <= 0:
            continue
        if fd:
            out += [(Mm, N, K, 0, 0, wt) for (Mm, N, K) in layer(rows)]  # recompute forward
        out += [(Mm, N, K, 0, 1, wt) for (Mm, N, K) in dgrad(rows)]
        out += [(Mm, N, K, 1, 1, wt) for (Mm, N, K) in wgrad(rows)]
    wl = 1.0 / shape.n_layer
    if fd:
        out += [(2 * M, Vp, h, 0, 0, 0.5 * wl)]
    for rows, wt in ((2 * M, 0.5 * fp), (M, 1.0 - fp)) if fd else ((M, 1.0),):
        if wt <= 0:
            continue
        if fd:
            out += [(rows, Vp, h, 0, 0, wt * wl)]
        else:
            out += [(rows, Vp, h, 0, 0, wt * wl)]
        out += [(rows, h, Vp, 0, 1, wt * wl), (Vp, h, rows, 1, 1, wt * wl)]
    merged = {}  # the same shape from several roles: one entry, weights summed
    for (Mm, N, K, a, b, w) in out:
        merged[(Mm, N, K, a, b)] = merged.get((Mm, N, K, a, b), 0.0) + w
    return [k + (w,) for k, w in merged.items()]


def gemm_roofline(stream_handle, peak_tflops, shape=None, cfg=None, workspace=True, bwd_pair_frac=None):
    """Live CUDA-event timing of the stage GEMMs (the dominant kernel family) at the
    workload's shapes as the step runs them (roofline_shapes), on the trainer's device,
    with the split-K workspace the trainer's chain streams use, each shape's launches
    replayed from a CUDA graph like the step's: achieved = sum_i w_i 2 M N K / sum_i w_i t_i."""
    import torch
    from paper_2107_06925_b200 import kernels as ck
    from paper_2107_06925_b200.gpt import PRESETS
    shape = shape or PRESETS[SHAPE_NAME]
    cfg = cfg or CFG
    shapes = roofline_shapes(shape, cfg, bwd_pair_frac)
    tot_flops, tot_ms, wsum = 0.0, 0.0, 0.0
    rows = []
    ws = torch.zeros(max(Mm * N for (Mm, N, K, a, b, w) in shapes if not (a and b)), device="cuda") \
        if workspace else None
    side = torch.cuda.Stream()
    reps = 20
    for (Mm, N, K, a, b, w) in shapes:
        A = torch.randn((K, Mm) if a else (Mm, K), device="cuda").bfloat16()
        B = torch.randn((K, N) if b else (N, K), device="cuda").bfloat16()
        out = torch.zeros(Mm, N, device="cuda", dtype=torch.float32 if (a and b) else torch.bfloat16)

        def run():
            ck.gemm("acc_f32" if (a and b) else "bf16", A, B, out, a_mn=bool(a), b_mn=bool(b),
                    ws=None if (a and b) else ws, stream=torch.cuda.current_stream())
        # the step replays its kernels from a CUDA graph: time the same way (no host
        # launch cost), `reps` launches captured back to back, CUDA events around replays
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                run()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                run()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / (3 * reps)
        fl = 2.0 * Mm * N * K
        tot_ms += w * ms
        tot_flops += w * fl
        wsum += w
        rows.append({"shape": [Mm, N, K, a, b], "weight": round(w, 4), "us": round(ms * 1e3, 2),
                     "tflops": round(fl / (ms * 1e-3) / 1e12, 1)})
        del g, A, B, out
    del ws
    achieved = tot_flops / (tot_ms * 1e-3) / 1e12
    # DRAM bytes per launch of the same shapes from the committed `ncu --set full`
    # capture (scripts/roofline_shapes.py --config ...); null when not captured
    # (run-weighted like `achieved`: sum_i w_i dram_i / sum_i w_i, beside the algorithmic
    # operand + output bytes with the same weights)
    traffic, tsrc, alg = None, None, None
    root = os.path.dirname(os.path.abspath(__file__))
    for cand in (f"profiles/r02_gemm_roofline_ncu_{SHAPE_NAME}_B{cfg['B']}.json",
                 "profiles/r01y_gemm_roofline_ncu.json" if SHAPE_NAME == "gpt2-medium" and cfg["B"] == 4 else None):
        if cand and os.path.exists(os.path.join(root, cand)):
            with open(os.path.join(root, cand)) as fh:
                cap = json.load(fh)
            by_shape = {tuple(l["shape"]): l for l in cap.get("launches", [])}
            ws = [(w, by_shape.get((Mm, N, K, a, b))) for (Mm, N, K, a, b, w) in shapes]
            if all(l is not None for _, l in ws):
                traffic = sum(w * l["dram_bytes"] for w, l in ws) / sum(w for w, _ in ws)
                alg = sum(w * l["algorithmic_bytes"] for w, l in ws) / sum(w for w, _ in ws)
            else:
                traffic = cap["avg_dram_bytes_per_launch"]
            tsrc = cand
            break
    return {"bound": "tensor", "kernel": "ck gemm_bf16 (tcgen05.mma kind::f16, TMA, TMEM; split-K + finalize "
                                        "where chosen), every stage-GEMM shape of the step, run-count weighted",
            "achieved": round(achieved, 1), "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": round(achieved / peak_tflops, 4), "traffic": traffic, "traffic_unit": "bytes/launch",
            "traffic_source": tsrc, "algorithmic_bytes_per_launch": alg,
            "flops_per_launch_avg": tot_flops / wsum, "avg_launch_ms": tot_ms / wsum, "shapes": rows}


def measure_alpha_beta(world):
    """alpha (ms) and beta (ms/byte) of perfmodel's Rabenseifner allreduce cost
    2 log2(r) alpha + 2 (r-1)/r beta L (perfmodel.cpp:24-28), fitted from NCCL
    allreduce times at two sizes over one process per GPU (max over ranks)."""
    import math
    import torch
    import torch.distributed as dist
    ppg = int(os.environ.get("CK_PROCS_PER_GPU", "1"))
    members = list(range(0, world, ppg))
    g = dist.new_group(members, backend="nccl")
    out = torch.zeros(4, dtype=torch.float64)
    if len(members) > 1 and dist.get_rank() in members:
        times = []
        for n in (1 << 10, 1 << 24):  # 4 KiB and 64 MiB of fp32
            x = torch.ones(n, device="cuda")
            for _ in range(3):
                dist.all_reduce(x, group=g)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                dist.all_reduce(x, group=g)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 10], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=g)
            times.append((4.0 * n, float(t)))
        (s0, t0), (s1, t1) = times
        slope = max(0.0, (t1 - t0) / (s1 - s0))
        icpt = max(0.0, t0 - slope * s0)
        r = float(len(members))
        out = torch.tensor([icpt / (2.0 * math.log2(r)), slope * r / (2.0 * (r - 1.0)), s1, t1], dtype=torch.float64)
    dist.broadcast(out, src=0)  # default (gloo) group
    dist.destroy_process_group(g)
    measure_alpha_beta.big = (float(out[2]), float(out[3]), len(members))
    return float(out[0]), float(out[1])


def comm_report(world, msg_bytes):
    """Achieved NVLink bandwidths: the 64 MiB NCCL allreduce of the alpha/beta fit (algorithmic
    and bus bandwidth, 2(r-1)/r), and a peer copy of one stage message (cudaMemcpyPeerAsync on
    the copy engines, GPU 0 -> GPU 1, timed by rank 0 while the other ranks wait).  The
    executor's own messages are stored into the peer slot by the producing kernel, so they
    have no separately timed transfer."""
    import torch
    import torch.distributed as dist
    rep = {}
    big = getattr(measure_alpha_beta, "big", None)
    if big and big[1] > 0 and big[2] > 1:
        nbytes, t_ms, r = big
        alg = nbytes / (t_ms * 1e-3) / 1e9
        rep["allreduce"] = {"ranks": r, "bytes": int(nbytes), "ms": round(t_ms, 4), "algbw_GBs": round(alg, 1),
                            "busbw_GBs": round(alg * 2.0 * (r - 1) / r, 1), "impl": "NCCL ring/NVLS (torch nccl)"}
    dist.barrier()
    if dist.get_rank() == 0 and torch.cuda.device_count() > 1 and int(os.environ.get("CK_PROCS_PER_GPU", "1")) == 1:
        src = torch.empty(msg_bytes // 2, dtype=torch.bfloat16, device="cuda:0")
        dst = torch.empty(msg_bytes // 2, dtype=torch.bfloat16, device="cuda:1")
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0 = torch.cuda.current_stream(0)
        e0.record(s0)
        for _ in range(20):
            dst.copy_(src, non_blocking=True)
        e1.record(s0)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        t = e0.elapsed_time(e1) / 20
        rep["p2p_copy"] = {"bytes": int(msg_bytes), "ms": round(t, 4), "GBs": round(msg_bytes / (t * 1e-3) / 1e9, 1),
                           "path": "cuda:0 -> cuda:1, copy engine over NVLink"}
        del src, dst
    dist.barrier()
    return rep or None


def config_dict(shape, world):
    """The `config` object of both arms' lines (same workload, same stage partition)."""
    from paper_2107_06925_b200 import pipesim as P
    cfg = P.PipelineConfig(**CFG)
    n_logical = cfg.W * cfg.D
    return {"workload": WORKLOAD,
            "model": SHAPE_NAME, "global_batch": cfg.mini_batch(), "seq_len": shape.seq,
            "stage_layers": list(shape.stage_layers) or None,
            "parallelism": f"{cfg.scheme} D={cfg.D} W={cfg.W} f={cfg.f} {cfg.scaling}"
                           f"{' +recompute' if cfg.scaling == 'forward-doubling' else ''}: "
                           f"{n_logical} logical ranks on {world} GPU(s)",
            "l2": "working set per step >> L2 (weights, grads, stashes ~40 GB)"}


def run_reference(args, shape):
    """--impl reference: the reference path's CPU implementation (the numpy port of the
    reference Engine -- the reference itself has no transformer), all host threads, on
    the SAME workload: every step times one sequence's forward + backward through one
    pipeline stage (stages in turn), so the run covers every stage; value = 1 / (sum over
    stages of the mean per-stage time) sequences/s."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ps = PortStages(shape)
    for k in range(args.warmup):
        ps.time_stage(k % ps.D)
    ps.times = {}
    for k in range(args.steps):
        ps.time_stage((args.warmup + k) % ps.D)
    v = ps.seqs_per_s()
    per = {st: round(sum(t) / len(t), 3) for st, t in sorted(ps.times.items())}
    line = {"metric": METRIC, "value": v, "unit": "seqs/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(shape, args.gpus),
            "cpu_baseline": {"value": v, "unit": "seqs/s", "cores": threads_used(), "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": f"numpy fp64 port of the reference Engine, one sequence per step through one "
                                       f"stage (stages in turn; s per stage {per}); 1 / sum over the {ps.D} stages"},
            "e2e": {"value": v, "unit": "seqs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chimera")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--head-efficiency", type=float, default=None,
                    help="balanced partition: LM head cost per FLOP relative to a layer's (default: measured)")
    ap.add_argument("--diag-timeout", type=float, default=150.0,
                    help="multi-process: seconds allowed for the profiled iteration + sync A/B")
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--B", type=int, default=0, help="override the config's micro-batch size")
    ap.add_argument("--partition", default="balanced", choices=["balanced", "even"],
                    help="layers per stage: balanced per pipeline worker (LM-head stage shorter) or even")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    global SHAPE_NAME, CFG, WORKLOAD
    SHAPE_NAME, CFG, WORKLOAD = CONFIGS[args.config]
    if args.B:
        CFG = dict(CFG, B=args.B)
        WORKLOAD = WORKLOAD.replace(f"B={CONFIGS[args.config][1]['B']}", f"B={args.B}")

    from paper_2107_06925_b200.gpt import PRESETS
    shape = PRESETS[SHAPE_NAME]
    if args.partition == "balanced":  # both arms: the reference port times the same stages
        import dataclasses
        from paper_2107_06925_b200 import pipesim as P
        from paper_2107_06925_b200.gpt import balanced_partition
        shape = dataclasses.replace(shape, stage_layers=balanced_partition(shape, P.PipelineConfig(**CFG),
                                                                           *([args.head_efficiency]
                                                                             if args.head_efficiency else [])))
    if args.impl == "reference":
        return run_reference(args, shape)

    import numpy as np
    import torch
    from paper_2107_06925_b200 import pipesim as P
    from paper_2107_06925_b200.gpt import Trainer, synthetic_batch

    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line
    # one hardware queue per stream (set before the CUDA context exists): a stream blocked
    # in a cross-process flag wait must not stall another stream sharing its queue
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CK_PROCS_PER_GPU=k (validation only): k consecutive processes share one GPU, e.g. the
    # 8-GPU one-rank-per-process layout exercised on 4 GPUs
    torch.cuda.set_device(local // int(os.environ.get("CK_PROCS_PER_GPU", "1")))
    cfg = P.PipelineConfig(**CFG)
    n_logical = cfg.W * cfg.D
    if n_logical % world:
        raise SystemExit(f"--gpus {world} must divide the {n_logical} logical ranks")
    per = n_logical // world
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    tr = Trainer(shape, cfg, lr=1e-4, first_rank=rank * per, n_ranks=per)
    if world > 1:
        tr.connect()
    progress("trainer created; init params")
    tr.init_params(seed=0)
    n_seq = cfg.mini_batch()
    tok, lab = synthetic_batch(shape, n_seq, seed=1)
    tr.set_batch(tok, lab)
    progress("warm-up")
    for _ in range(args.warmup):
        loss = tr.step()
    stream = torch.cuda.ExternalStream(tr.stream_handle())

    progress("timed steps")
    # ---- value: resident inputs, graph replay, CUDA events on the trainer stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            tr.launch()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    value = n_seq / (ms * 1e-3)

    progress("e2e steps")
    # ---- e2e: public API per step: pinned H2D tokens+labels, step, D2H loss
    tok_h = torch.from_numpy(tok).pin_memory()
    lab_h = torch.from_numpy(lab).pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        tr.set_batch(tok_h, lab_h)
        loss = tr.step()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t)

    # ---- launches in the timed region (the captured iteration's kernel nodes, all processes)
    stats = tr.stats()
    launches = int(stats["launches_per_step"] * args.steps)
    if world > 1:
        t = torch.tensor([launches], dtype=torch.float64)
        dist.all_reduce(t)
        launches = int(t)
    base = {
        "metric": METRIC, "value": round(value, 2), "unit": "seqs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens (uniform, next-token labels), random-init weights N(0,0.02)",
        "config": config_dict(shape, world),
        "e2e": {"value": round(n_seq / (e2e_ms * 1e-3), 2), "unit": "seqs/s",
                "h2d_bytes_per_step": int(tok.nbytes + lab.nbytes), "d2h_bytes_per_step": 4},
    }
    clocks = clk.summary()

    # The measured numbers are complete here.  Multi-process: the diagnostics below (eager
    # profiled iteration, sync-policy A/B) run under a watchdog, so a hang there still
    # leaves the bench line (without those sections) and a clean exit on every process.
    watchdog = None
    if world > 1:
        def _diag_timeout():
            if rank == 0:
                print(json.dumps({**base, "gpu_launches": launches, "clocks": clocks, "cpu_baseline": None,
                                  "diagnostics": f"profiled iteration / sync-policy A/B did not finish within "
                                                 f"{args.diag_timeout} s; omitted"}), flush=True)
            os._exit(0)
        watchdog = threading.Timer(args.diag_timeout, _diag_timeout)
        watchdog.daemon = True
        watchdog.start()

    # ---- one profiled (eager) iteration: per-task GPU spans -> measured bubble
    if world > 1:
        dist.barrier()
    progress("profiled iteration")
    prof = tr.profile_step()
    tasks, colls = prof["tasks"], prof.get("allreduce", [])
    if world > 1:  # per-process clocks, each relative to its own iteration start
        allt = [None] * world
        dist.all_gather_object(allt, (tasks, colls))
        tasks = [t for x in allt for t in x[0]]
        colls = [c for x in allt for c in x[1]]

    # ---- alpha / beta of the collective fabric (Eq. 1's allreduce term), NCCL over all ranks
    ab = measure_alpha_beta(world) if world > 1 else (0.0, 0.0)
    comm = comm_report(world, 2 * CFG["B"] * shape.seq * shape.hidden) if world > 1 else None

    # ---- the measured B200 CostProfile, computed identically on every process (from the
    # gathered task spans) so the sync plan built on it is the same everywhere
    from fractions import Fraction
    # task compute time = span minus the stream's waits for incoming messages
    fwd = [t["end_ms"] - t["start_ms"] - t.get("stall_ms", 0.0) for t in tasks if t["kind"] == "Forward"]
    bwd = [t["end_ms"] - t["start_ms"] - t.get("stall_ms", 0.0) for t in tasks if t["kind"] == "Backward"]
    ratio = (sum(bwd) / len(bwd)) / (sum(fwd) / len(fwd))
    l_grad = 4.0 * max(st["numel"] for st in tr.layout)  # fp32 gradient of the largest held stage
    if world > 1:
        t = torch.tensor([l_grad], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        l_grad = float(t)
    prof_b200 = P.CostProfile(F_t=sum(fwd) / len(fwd), backward_ratio=float(Fraction(ratio).limit_denominator(16)),
                              alpha=ab[0], beta=ab[1], L_grad=l_grad,
                              L_act=2.0 * CFG["B"] * shape.seq * shape.hidden)

    # ---- gradient-sync policies on the measured profile (dessim eager rule), one rank per
    # GPU: the paper's eager-sync-opt vs eager-sync vs end-of-iteration
    sync_ab = None
    if world > 1:
        tr.set_cost_profile(prof_b200)
        sync_ab = {}
        for pol in ("end-of-iteration", "eager-sync", "eager-sync-opt"):
            tr.set_sync_policy(pol)
            for _ in range(2):
                tr.step()
            dist.barrier()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(args.steps):
                tr.launch()
            g1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([g0.elapsed_time(g1) / args.steps])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sync_ab[pol] = {"ms_per_step": round(float(t), 3)}
            if pol == "eager-sync-opt":
                sync_ab[pol]["eager_stages"] = [e["stage"] for e in tr.sync_plan()["order"] if e["eager"]]
        tr.set_sync_policy("eager-sync")
    if watchdog is not None:
        watchdog.cancel()

    if world > 1:  # the loss is summed over the processes holding last stages
        t = torch.tensor([loss])
        dist.all_reduce(t)
        loss = float(t)
        for key in ("peak_stash_per_rank", "peak_stash_bytes_per_rank"):
            pk = [None] * world
            dist.all_gather_object(pk, stats[key])
            stats[key] = [v for x in pk for v in x]
    peak, peak_sus, hbm, peak_src = peaks()
    line = None
    if rank == 0:
        sched = tr.schedule_text
        bub = P.bubble_ratio(sched)
        from paper_2107_06925_b200.gpt import measured_bubble, timeline_json
        prof_m = P.CostProfile(backward_ratio=float(Fraction(ratio).limit_denominator(16)))
        bub_at_ratio = P.bubble_ratio(P.generate_json(cfg, prof_m, -1), prof_m)
        one_rank_per_gpu = per == 1
        mb = measured_bubble({"tasks": tasks}) if one_rank_per_gpu else None
        if os.environ.get("CK_TIMELINE"):  # prefix: measured timeline + Gantt charts
            from paper_2107_06925_b200.gpt import measured_timeline
            pre = os.environ["CK_TIMELINE"]
            tl = measured_timeline({"tasks": tasks, "allreduce": colls}, sched)
            ft = P.CostProfile(F_t=max(1e-6, sum(fwd) / len(fwd)))
            for ext, text in ((".json", tl), (".svg", P.gantt_timeline(tl, ft, svg=True)),
                              (".txt", P.gantt_timeline(tl, ft)), (".sched.json", timeline_json({"tasks": tasks}, sched))):
                with open(pre + ext, "w") as fh:
                    fh.write(text)
        # dessim::simulate (proj/src/dessim.cpp:60-181) on the measured F_t, B/F, alpha, beta:
        # per-worker idle / compute span, averaged -- the simulated counterpart of `measured`
        replay_bubble = None
        if one_rank_per_gpu:
            from paper_2107_06925_b200.gpt import replay_measured
            rp = replay_measured({"tasks": tasks}, sched, prof_b200.alpha + prof_b200.beta * prof_b200.L_act)
            replay_bubble = round(rp["mean"], 4)
        sim = P.simulate(sched, prof_b200, "eager-sync")
        span = sim["compute_makespan"]
        dessim_bubble = round(sum(sim["per_worker_idle"]) / len(sim["per_worker_idle"]) / span, 4) if span else None
        mp = P.memory_profile(sched)
        # Eq. 1 (perfmodel::predict_T, perfmodel.cpp:157) on the measured B200 CostProfile
        pred = P.predict_T(cfg, prof_b200)
        # perfmodel::plan (perfmodel.cpp:225-298) on the same profile with the measured
        # memory terms: which (W, D, B) it would pick for 2, 4, 8 GPUs at this mini-batch
        plans = None
        try:
            acts = [a for a in stats["peak_stash_per_rank"] if a] or [1]
            sbytes = [b for b in stats["peak_stash_bytes_per_rank"] if b] or [0]
            m_a = max(sbytes) / max(acts) / CFG["B"] if max(sbytes) else 0.0
            mprof = P.CostProfile(**{**prof_b200.__dict__, "M_theta": 10.0 * l_grad / 4.0, "M_a": m_a,
                                     "M_a_ckpt": 2.0 * shape.seq * shape.hidden, "mem_capacity": 178e9,
                                     "embed_surcharge": True})
            plans = {}
            for Pn in (2, 4, 8):
                ents = P.plan(Pn, n_seq, mprof, "chimera")
                plans[str(Pn)] = [{k: e[k] for k in ("W", "D", "B", "N", "scaling", "recompute")} |
                                  {"T_predicted_ms": round(e["T_predicted"], 3)} for e in ents[:3]]
        except Exception as e:  # the planner may find nothing feasible
            plans = {"error": str(e)[:200]}
        bt = stats.get("backward_tasks") or 0
        progress("GEMM roofline")
        rl = gemm_roofline(tr.stream_handle(), peak, shape, CFG,
                           bwd_pair_frac=(2.0 * stats.get("fused_backward_pairs", 0) / bt) if bt else None)
        flops_seq = shape.flops_per_seq()
        progress("CPU baseline")
        cpu = None if (args.no_cpu_baseline or world > 1) else cpu_port_sample(shape)  # N=1 only
        line = {
            **base,
            "roofline": rl,
            "mfu": {"tflops_per_gpu": round(value * flops_seq / world / 1e12, 1),
                    "frac_of_sustained": round(value * flops_seq / world / 1e12 / peak_sus, 4) if peak_sus else None,
                    "flop_per_seq": flops_seq, "peak_source": peak_src},
            "bubble": {"measured": (round(sum(mb["per_rank"].values()) / len(mb["per_rank"]), 4) if mb else None),
                       "measured_per_rank": ([round(v, 4) for v in mb["per_rank"].values()] if mb else None),
                       "closed_form_(D-2)/(2N+D-2)": str(P.closed_form_bubble(cfg.D, cfg.N)),
                       "reference_schedule_at_B/F=2": str(bub),
                       "measured_B/F": round(ratio, 3),
                       "reference_schedule_at_measured_B/F": str(bub_at_ratio),
                       "dessim_at_measured_profile": dessim_bubble,
                       "list_schedule_at_measured_task_times": replay_bubble,
                       "note": (None if one_rank_per_gpu else
                                f"{per} logical ranks share each GPU: per-rank bubble not observable")},
            "perfmodel": {"predicted_ms": round(pred, 3), "measured_ms": round(ms, 3),
                          "rel_err": round((ms - pred) / ms, 4),
                          "valid": one_rank_per_gpu,
                          "profile": {"F_t_ms": round(prof_b200.F_t, 4), "backward_ratio": prof_b200.backward_ratio,
                                      "alpha_ms": ab[0], "beta_ms_per_byte": ab[1], "L_grad": l_grad,
                                      "L_act": prof_b200.L_act},
                          "note": ("Eq. 1 assumes one worker per GPU" if not one_rank_per_gpu else
                                   "p2p term: alpha + beta * L_act with the allreduce fit (upper bound; "
                                   "stage outputs are stored into the peer slot by the producing kernel)")},
            "comm": comm,
            "sync_policies": sync_ab,
            "plan": plans,
            "act_counts_per_worker": mp["act_counts"],
            "peak_stash_per_rank": stats["peak_stash_per_rank"],
            "peak_stash_bytes_per_rank": stats["peak_stash_bytes_per_rank"],
            "device_bytes": stats["device_bytes"],
            "loss": loss,
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    tr.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
