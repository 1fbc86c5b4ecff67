"""Per-kernel device time of bench steps from a CUPTI activity trace (torch.profiler /
kineto: every kernel of the replayed iteration graph, concurrent kernels included, no
replay, real clocks) -- the cheap complement of the ncu launch list.

    python scripts/kernel_trace.py [--config gpt2-1.3b] [--B 2] [--steps 2] [--json out.json]

Prints, per kernel name: launches per step, total and average device time, share of
the summed kernel time; plus summed kernel time / wall time (= average concurrency).
"""
import argparse
import collections
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--B", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2107_06925_b200 import pipesim as P
    from paper_2107_06925_b200.gpt import PRESETS, Trainer, balanced_partition, synthetic_batch
    name, cfgd, _ = bench.CONFIGS[args.config]
    cfgd = dict(cfgd, B=args.B or cfgd["B"])
    cfg = P.PipelineConfig(**cfgd)
    shape = dataclasses.replace(PRESETS[name], stage_layers=balanced_partition(PRESETS[name], cfg))
    tr = Trainer(shape, cfg, lr=1e-4)
    tr.init_params(seed=0)
    tok, lab = synthetic_batch(shape, cfg.mini_batch(), seed=1)
    tr.set_batch(tok, lab)
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(tr.stream_handle())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0.record(st)
        for _ in range(args.steps):
            tr.launch()
        e1.record(st)
        torch.cuda.synchronize()
    wall_ms = e0.elapsed_time(e1)
    agg = collections.defaultdict(lambda: [0, 0.0])
    lo, hi = None, None
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        dur = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        if dur <= 0:
            continue
        k = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").replace("chimera::", "")
        k = k.split("(")[0]
        agg[k][0] += 1
        agg[k][1] += dur / 1e3  # ms
    tot = sum(v[1] for v in agg.values())
    rows = sorted(agg.items(), key=lambda x: -x[1][1])
    out = {"config": args.config, "B": cfg.B, "steps": args.steps, "wall_ms_per_step": wall_ms / args.steps,
           "kernel_ms_per_step": tot / args.steps, "concurrency": tot / wall_ms,
           "launches_per_step": sum(v[0] for v in agg.values()) / args.steps,
           "kernels": [{"name": k[:90], "n_per_step": c / args.steps, "ms_per_step": round(t / args.steps, 3),
                        "avg_us": round(1e3 * t / c, 2), "share": round(t / tot, 4)} for k, (c, t) in rows]}
    print(f"wall {out['wall_ms_per_step']:.2f} ms/step, kernel time {out['kernel_ms_per_step']:.2f} ms/step, "
          f"concurrency {out['concurrency']:.2f}, launches/step {out['launches_per_step']:.0f}")
    for r in out["kernels"][:30]:
        print(f"{r['ms_per_step']:9.2f} ms {100 * r['share']:5.1f}%  n={r['n_per_step']:7.0f}  avg {r['avg_us']:8.2f} us  "
              f"{r['name']}")
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)
    tr.close()


if __name__ == "__main__":
    main()
