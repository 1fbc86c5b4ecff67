"""Weight-gradient GEMMs (fp32 accumulate into a large, HBM-resident gradient buffer as in
the step) at the configs[3] shapes: every (tile, K-slices) variant, graph-timed.

    python scripts/gemm_wgrad_sweep.py > gpurun_out/wgrad_sweep.jsonl"""
import json
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from gemm_split_sweep import graph_us  # noqa: E402
from paper_2107_06925_b200 import kernels as ck  # noqa: E402

h, f = 1280, 5120


def main():
    # the gradient lives in a 1 GB buffer (a stage's gradients do not fit in L2)
    big = torch.zeros(256 << 20, device="cuda")
    dummy = torch.zeros(8, device="cuda")
    for K in (2528, 1264):
        for (M, N) in ((3 * h, h), (h, h), (f, h), (h, f)):
            A = torch.randn(K, M, device="cuda").bfloat16()   # dY^T operand, MN-major
            B = torch.randn(K, N, device="cuda").bfloat16()   # X, MN-major
            off = (M * N * 7) % ((256 << 20) - M * N)
            out = big[off:off + M * N].view(M, N)
            res = {"shape": [M, N, K]}
            for tile in (0, 256, 128):
                for ks in (1, 2, 3, 4):
                    run = lambda: ck.gemm("acc_f32", A, B, out, a_mn=True, b_mn=True, ws=dummy, ksplit=ks, tile=tile,
                                          stream=torch.cuda.current_stream())
                    res[f"{tile}/{ks}"] = round(graph_us(run), 2)
            res["auto"] = round(graph_us(lambda: ck.gemm("acc_f32", A, B, out, a_mn=True, b_mn=True,
                                                         stream=torch.cuda.current_stream())), 2)
            best = min((v, k) for k, v in res.items() if k != "shape")
            res["best"] = best[1]
            res["best_tflops"] = round(2.0 * M * N * K / (best[0] * 1e-6) / 1e12, 1)
            res["auto_tflops"] = round(2.0 * M * N * K / (res["auto"] * 1e-6) / 1e12, 1)
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
