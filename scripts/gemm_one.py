"""One stage GEMM shape, a few launches (the command profiled by ncu for per-line stalls).
usage: python scripts/gemm_one.py M N K epi a_mn b_mn [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
epi, a, b = sys.argv[4], int(sys.argv[5]), int(sys.argv[6])
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 4
A = torch.randn((K, M) if a else (M, K), device="cuda").bfloat16()
B = torch.randn((K, N) if b else (N, K), device="cuda").bfloat16()
f32 = epi in ("acc_f32", "f32")
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
kw = {}
if epi in ("bias_resid", "bias_gelu", "bf16"):
    kw["bias"] = torch.randn(N, device="cuda").bfloat16()
if epi in ("bias_resid", "gelu_bwd"):
    kw["aux"] = torch.randn(M, N, device="cuda").bfloat16()
if epi == "bias_gelu":
    kw["out2"] = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    ck.gemm(epi, A, B, out, a_mn=bool(a), b_mn=bool(b), **kw)
torch.cuda.synchronize()
print("ok")
