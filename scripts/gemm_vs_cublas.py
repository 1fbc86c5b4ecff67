"""The bench's roofline GEMM shapes (bench.roofline_shapes, run-weighted) timed with this
repo's tcgen05 kernels and with cuBLAS (torch.matmul, bf16 in / bf16 out, fp32 accumulate)
on the same shapes, both graph-timed.  The weight-gradient shapes accumulate in fp32
here; cuBLAS is timed as a bf16-output matmul of the same size (a lower bound on its cost).

    python scripts/gemm_vs_cublas.py [--config gpt2-1.3b] [--B 2] > gpurun_out/vs_cublas.jsonl"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import bench  # noqa: E402
from gemm_split_sweep import graph_us  # noqa: E402
from paper_2107_06925_b200 import kernels as ck  # noqa: E402
from paper_2107_06925_b200.gpt import PRESETS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--B", type=int, default=0)
    args = ap.parse_args()
    name, cfg, _ = bench.CONFIGS[args.config]
    cfg = dict(cfg, B=args.B or cfg["B"])
    shapes = bench.roofline_shapes(PRESETS[name], cfg)
    # the trainer's split-K / stream-K workspace is >= 74 pairs x 2 x 128 x 256 partial slots
    ws = torch.zeros(max([M * N for (M, N, K, a, b, w) in shapes if not (a and b)] + [74 * 2 * 128 * 256 + 4096]),
                     device="cuda")
    big = torch.zeros(256 << 20, device="cuda")
    tot = {"ours": 0.0, "cublas": 0.0, "w": 0.0}
    for (M, N, K, a, b, w) in shapes:
        A = torch.randn((K, M) if a else (M, K), device="cuda").bfloat16()
        B = torch.randn((K, N) if b else (N, K), device="cuda").bfloat16()
        if a and b:
            off = (M * N * 7) % ((256 << 20) - M * N)
            out = big[off:off + M * N].view(M, N)
            ours = graph_us(lambda: ck.gemm("acc_f32", A, B, out, a_mn=True, b_mn=True,
                                            stream=torch.cuda.current_stream()))
            At, Bt = A.t(), B
        else:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ours = graph_us(lambda: ck.gemm("bf16", A, B, out, a_mn=bool(a), b_mn=bool(b), ws=ws,
                                            stream=torch.cuda.current_stream()))
            At = A
            Bt = B if b else B.t()
        cub = graph_us(lambda: torch.matmul(At, Bt))
        fl = 2.0 * M * N * K
        tot["ours"] += w * ours
        tot["cublas"] += w * cub
        tot["w"] += w
        print(json.dumps({"shape": [M, N, K, a, b], "weight": round(w, 4), "ours_us": round(ours, 2),
                          "cublas_us": round(cub, 2), "ours_tflops": round(fl / ours / 1e6, 1),
                          "cublas_tflops": round(fl / cub / 1e6, 1)}), flush=True)
    print(json.dumps({"weighted_ours_us": round(tot["ours"] / tot["w"], 2),
                      "weighted_cublas_us": round(tot["cublas"] / tot["w"], 2),
                      "ours_over_cublas_time": round(tot["ours"] / tot["cublas"], 3)}))


if __name__ == "__main__":
    main()
