"""Per-shape timing of the GEMMs one GPT-2-medium Chimera step issues (actual epilogues),
weighted by their count per step (D=4 N=4 W=2 B=4: 192 layer fwd+bwd, 8 LM-head fwd+bwd),
next to cuBLAS (torch.matmul, bf16 out) on the same shape."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as K  # noqa: E402


def timeit(fn, it=20):
    """Device time per call: `it` calls captured into one CUDA graph (no host overhead)."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(2):
            fn(st)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for _ in range(it):
            fn(st)
    gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    gr.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


Mt, h, f, V = 4096, 1024, 4096, 50304
L, HEAD = 192, 8
shapes = [  # (tag, epi, M, N, K, a_mn, b_mn, count/step)
    ("qkv fwd", "bf16", Mt, 3 * h, h, 0, 0, L), ("proj fwd +res", "bias_resid", Mt, h, h, 0, 0, L),
    ("fc1 fwd +gelu", "bias_gelu", Mt, f, h, 0, 0, L), ("fc2 fwd +res", "bias_resid", Mt, h, f, 0, 0, L),
    ("fc2 wgrad", "acc_f32", h, f, Mt, 1, 1, L), ("fc2 dgrad +gelu'", "gelu_bwd", Mt, f, h, 0, 1, L),
    ("fc1 wgrad", "acc_f32", f, h, Mt, 1, 1, L), ("fc1 dgrad", "bf16", Mt, h, f, 0, 1, L),
    ("proj wgrad", "acc_f32", h, h, Mt, 1, 1, L), ("proj dgrad", "bf16", Mt, h, h, 0, 1, L),
    ("qkv wgrad", "acc_f32", 3 * h, h, Mt, 1, 1, L), ("qkv dgrad", "bf16", Mt, h, 3 * h, 0, 1, L),
    ("head fwd", "bf16", Mt, V, h, 0, 0, HEAD), ("head dgrad", "bf16", Mt, h, V, 0, 1, HEAD),
    ("head wgrad", "acc_f32", V, h, Mt, 1, 1, HEAD)]
tot_ms, tot_cub = 0.0, 0.0
rows = []
for (tag, epi, M, N, Kd, a_mn, b_mn, cnt) in shapes:
    A = torch.randn((Kd, M) if a_mn else (M, Kd), device="cuda").bfloat16()
    B = torch.randn((Kd, N) if b_mn else (N, Kd), device="cuda").bfloat16()
    f32 = epi == "acc_f32"
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    kw = {}
    if epi in ("bias_resid", "bias_gelu"):
        kw["bias"] = torch.zeros(N, device="cuda").bfloat16()
    if epi == "bias_resid":
        kw["aux"] = torch.randn(M, N, device="cuda").bfloat16()
    if epi == "gelu_bwd":
        kw["aux"] = torch.randn(M, N, device="cuda").bfloat16()
    if epi == "bias_gelu":
        kw["out2"] = torch.empty(M, N, device="cuda").bfloat16()
    ms = timeit(lambda st: K.gemm(epi, A, B, out, a_mn=bool(a_mn), b_mn=bool(b_mn), stream=st, **kw))
    At = A.t() if a_mn else A
    Bt = B if b_mn else B.t()
    cub = timeit(lambda st: torch.matmul(At, Bt))
    fl = 2.0 * M * N * Kd
    tot_ms += ms * cnt
    tot_cub += cub * cnt
    rows.append({"gemm": tag, "shape": [M, N, Kd], "us": round(ms * 1e3, 1), "tflops": round(fl / ms / 1e9),
                 "cublas_us": round(cub * 1e3, 1), "cublas_tflops": round(fl / cub / 1e9), "count": cnt,
                 "ms_per_step": round(ms * cnt, 2)})
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"total_ms_per_step": round(tot_ms, 2), "cublas_total_ms_per_step": round(tot_cub, 2)}))
