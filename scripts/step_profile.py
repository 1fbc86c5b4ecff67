"""One bench workload's steps for profiling: W warm-up steps, then K graph-replayed steps
bracketed by cudaProfilerStart/Stop (run under `ncu --profile-from-start off` to get the
launch list of exactly K steps), and a per-task eager profile.

    python scripts/step_profile.py --config gpt2-1.3b [--steps 1] [--warmup 3] [--B 1]
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt2-1.3b")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--B", type=int, default=0)
    ap.add_argument("--tasks", action="store_true", help="print the per-task eager profile summary")
    args = ap.parse_args()
    import torch
    from paper_2107_06925_b200 import pipesim as P
    from paper_2107_06925_b200.gpt import PRESETS, Trainer, balanced_partition, synthetic_batch
    name, cfgd, workload = bench.CONFIGS[args.config]
    cfgd = dict(cfgd)
    if args.B:
        cfgd["B"] = args.B
    shape = PRESETS[name]
    cfg = P.PipelineConfig(**cfgd)
    shape = dataclasses.replace(shape, stage_layers=balanced_partition(shape, cfg))
    tr = Trainer(shape, cfg, lr=1e-4)
    tr.init_params(seed=0)
    n_seq = cfg.mini_batch()
    tok, lab = synthetic_batch(shape, n_seq, seed=1)
    tr.set_batch(tok, lab)
    for _ in range(args.warmup):
        tr.step()
    st = torch.cuda.ExternalStream(tr.stream_handle())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.profiler.start()
    e0.record(st)
    for _ in range(args.steps):
        tr.launch()
    e1.record(st)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    out = {"config": args.config, "B": cfg.B, "ms_per_step": ms, "seqs_per_s": n_seq / ms * 1e3,
           "mfu_tflops": n_seq * shape.flops_per_seq() / (ms * 1e-3) / 1e12,
           "launches_per_step": tr.stats()["launches_per_step"]}
    if args.tasks:
        prof = tr.profile_step()
        tasks = prof["tasks"]
        fwd = [t["end_ms"] - t["start_ms"] for t in tasks if t["kind"] == "Forward"]
        bwd = [t["end_ms"] - t["start_ms"] for t in tasks if t["kind"] == "Backward"]
        out["F_ms_avg"] = sum(fwd) / len(fwd)
        out["B_ms_avg"] = sum(bwd) / len(bwd)
        out["profile_span_ms"] = max(t["end_ms"] for t in tasks) - min(t["start_ms"] for t in tasks)
    print(json.dumps(out), flush=True)
    tr.close()


if __name__ == "__main__":
    main()
