"""Runs each of bench.py's roofline GEMM shapes (bench.roofline_shapes: every stage-GEMM
shape one iteration of the workload runs) once after a warm-up, with the split-K
workspace the trainer uses -- the command profiled by
`ncu --set full -k regex:"k_gemm|k_splitk"` for roofline.traffic (profiles/).

    python scripts/roofline_shapes.py [--config gpt2-1.3b] [--B 2]"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2107_06925_b200 import kernels as ck  # noqa: E402
from paper_2107_06925_b200.gpt import PRESETS  # noqa: E402


def shapes_for(config, B=0):
    name, cfg, _ = bench.CONFIGS[config]
    cfg = dict(cfg, B=B or cfg["B"])
    return bench.roofline_shapes(PRESETS[name], cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--B", type=int, default=0)
    args = ap.parse_args()
    shapes = shapes_for(args.config, args.B)
    ws = torch.zeros(max(M * N for (M, N, K, a, b, w) in shapes if not (a and b)), device="cuda")
    bufs = []
    for (Mm, N, K, a, b, w) in shapes:
        A = torch.randn((K, Mm) if a else (Mm, K), device="cuda").bfloat16()
        B = torch.randn((K, N) if b else (N, K), device="cuda").bfloat16()
        out = torch.zeros(Mm, N, device="cuda", dtype=torch.float32 if (a and b) else torch.bfloat16)
        bufs.append((Mm, N, K, a, b, A, B, out))
    for rep in range(2):  # warm-up pass, then one profiled pass (ncu --launch-skip = kernels of pass 1)
        if rep == 1:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        for (Mm, N, K, a, b, A, B, out) in bufs:
            ck.gemm("acc_f32" if (a and b) else "bf16", A, B, out, a_mn=bool(a), b_mn=bool(b),
                    ws=None if (a and b) else ws)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", len(shapes))


if __name__ == "__main__":
    main()
