"""Runs each of bench.py's 12 stage-GEMM roofline shapes once after a warm-up -- the
command profiled by `ncu --set full -k regex:k_gemm` for roofline.traffic (profiles/)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck  # noqa: E402

M, h, f = 4096, 1024, 4096
SHAPES = [(M, 3 * h, h, 0, 0), (M, h, h, 0, 0), (M, f, h, 0, 0), (M, h, f, 0, 0),
          (M, h, 3 * h, 0, 1), (M, h, h, 0, 1), (M, h, f, 0, 1), (M, f, h, 0, 1),
          (3 * h, h, M, 1, 1), (h, h, M, 1, 1), (f, h, M, 1, 1), (h, f, M, 1, 1)]


def main():
    bufs = []
    for (Mm, N, K, a, b) in SHAPES:
        A = torch.randn((K, Mm) if a else (Mm, K), device="cuda").bfloat16()
        B = torch.randn((K, N) if b else (N, K), device="cuda").bfloat16()
        out = torch.zeros(Mm, N, device="cuda", dtype=torch.float32 if (a and b) else torch.bfloat16)
        bufs.append((Mm, N, K, a, b, A, B, out))
    for rep in range(2):  # warm-up pass (not profiled: ncu -s 12), then one profiled pass
        for (Mm, N, K, a, b, A, B, out) in bufs:
            ck.gemm("acc_f32" if (a and b) else "bf16", A, B, out, a_mn=bool(a), b_mn=bool(b))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
