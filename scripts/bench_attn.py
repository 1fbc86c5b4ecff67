"""Attention kernels, graph-timed (20 launches captured in a CUDA graph, CUDA events
around replays -- eager ctypes calls would time the host launch path on small shapes).

    python scripts/bench_attn.py > gpurun_out/attn.jsonl

Shapes: the VERDICT target (B=4 s=1024 H=16 causal), Bert (B=8 s=128 H=16 bidirectional)
and the GPT-2 1.3B step's calls (s=632 H=20 causal; B=4 = a fused micro-batch pair at
B=2, B=2 unfused).  FLOPs: 4 s^2 d H B (x1/2 causal) forward, x2.5 backward."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck  # noqa: E402


def graph_us(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (3 * reps) * 1e3


def main():
    res = []
    shapes = [(4, 1024, 16, True), (8, 128, 16, False), (4, 632, 20, True), (2, 632, 20, True)]
    if len(sys.argv) > 1 and sys.argv[1] == "scale":  # fixed vs per-tile cost
        shapes = [(B, 1024, 16, True) for B in (1, 2, 4, 8, 16)]
    for (B, s, H, causal) in shapes:
        qkv = torch.randn(B * s, 3 * H * 64, device="cuda").bfloat16()
        out = torch.empty(B * s, H * 64, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(B * H * s, device="cuda")
        dout = torch.randn_like(out)
        dqkv = torch.empty_like(qkv)
        fl = 4 * s * s * 64 * B * H * (0.5 if causal else 1.0)
        cur = torch.cuda.current_stream
        for name, fn in [("fwd_tc", lambda: ck.attn_fwd_tc(qkv, out, lse, B, s, H, causal, stream=cur())),
                         ("bwd_tc", lambda: ck.attn_bwd(qkv, out, dout, lse, dqkv, B, s, H, causal, impl="tcgen05",
                                                        stream=cur()))]:
            us = graph_us(fn)
            f = fl * (2.5 if name.startswith("bwd") else 1.0)
            res.append({"shape": [B, s, H, causal], "kernel": name, "us": round(us, 2),
                        "tflops": round(f / us / 1e6, 1)})
            print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] == "breakdown"):
    main()


def kernel_breakdown():
    """Per-kernel device time of one attention backward (CUPTI via torch.profiler)."""
    from torch.profiler import ProfilerActivity, profile
    B, s, H = 4, 1024, 16
    qkv = torch.randn(B * s, 3 * H * 64, device="cuda").bfloat16()
    out = torch.empty(B * s, H * 64, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * s, device="cuda")
    dout = torch.randn_like(out)
    dqkv = torch.empty_like(qkv)
    db = torch.zeros(3 * H * 64, device="cuda")
    ck.attn_fwd_tc(qkv, out, lse, B, s, H, True)
    for _ in range(3):
        ck.attn_bwd(qkv, out, dout, lse, dqkv, B, s, H, True, impl="tcgen05", dbias=db)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            ck.attn_bwd(qkv, out, dout, lse, dqkv, B, s, H, True, impl="tcgen05", dbias=db)
        torch.cuda.synchronize()
    agg = {}
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        import re
        mk = re.search(r"(k_\w+)", ev.name)
        k = mk.group(1) if mk else ev.name[:40]
        agg.setdefault(k, []).append(ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total)
    for k, v in agg.items():
        print(json.dumps({"kernel": k, "n": len(v), "avg_us": round(sum(v) / len(v), 2)}), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "breakdown":
    kernel_breakdown()
