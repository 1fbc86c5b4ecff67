"""Microbenchmark: tcgen05 GEMM vs cuBLAS (torch.matmul) on the transformer shapes."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as K  # noqa: E402


def timeit(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


rows = []
for (M, N, Kd, a_mn, b_mn, tag) in [(4096, 3072, 1024, 0, 0, "qkv fwd"), (4096, 1024, 1024, 0, 0, "proj fwd"),
                                    (4096, 4096, 1024, 0, 0, "fc1 fwd"), (4096, 1024, 4096, 0, 0, "fc2 fwd"),
                                    (4096, 1024, 4096, 0, 1, "fc1 dgrad"), (4096, 4096, 1024, 0, 1, "fc2 dgrad"),
                                    (4096, 1024, 4096, 1, 1, "fc1 wgrad(NxK=4096x1024,red 4096)"),
                                    (1024, 4096, 4096, 1, 1, "fc2 wgrad"),
                                    (4096, 50304, 1024, 0, 0, "lm head fwd"),
                                    (8192, 8192, 8192, 0, 0, "8192^3")]:
    A = torch.randn(Kd, M, device="cuda").bfloat16() if a_mn else torch.randn(M, Kd, device="cuda").bfloat16()
    B = torch.randn(Kd, N, device="cuda").bfloat16() if b_mn else torch.randn(N, Kd, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = timeit(lambda: K.gemm("bf16", A, B, out, a_mn=bool(a_mn), b_mn=bool(b_mn)))
    Af = A.t() if a_mn else A
    Bf = B if b_mn else B.t()
    tc = timeit(lambda: torch.matmul(Af, Bf))
    fl = 2.0 * M * N * Kd
    rows.append({"shape": tag, "M": M, "N": N, "K": Kd, "ours_ms": round(t, 4), "ours_tflops": round(fl / t / 1e9, 1),
                 "cublas_ms": round(tc, 4), "cublas_tflops": round(fl / tc / 1e9, 1)})
    print(json.dumps(rows[-1]), flush=True)
