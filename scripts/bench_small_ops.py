"""Microbenchmark of the non-GEMM stage kernels (graph-timed).

    python scripts/bench_small_ops.py [M h f]     (default: GPT-2 medium, 4096 1024 4096)"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as K  # noqa: E402


def timeit(fn, it=50):
    """Device time per call: `it` calls captured into one CUDA graph (no host overhead)."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
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
    return s.elapsed_time(e) / it * 1e3


M, h, f = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 1024, 4096)
x = torch.randn(M, h, device="cuda").bfloat16()
dy = torch.randn(M, h, device="cuda").bfloat16()
dres = torch.randn(M, h, device="cuda").bfloat16()
g = torch.randn(h, device="cuda").bfloat16()
b = torch.randn(h, device="cuda").bfloat16()
y = torch.empty_like(x)
dx = torch.empty_like(x)
mean = torch.empty(M, device="cuda")
rstd = torch.empty(M, device="cuda")
dg = torch.zeros(h, device="cuda")
db = torch.zeros(h, device="cuda")
res = {}
res["ln_fwd"] = timeit(lambda st: K.layernorm_fwd(x, g, b, y, mean, rstd, stream=st))
res["ln_bwd"] = timeit(lambda st: K.layernorm_bwd(dy, x, mean, rstd, g, dres, dx, dg, db, stream=st))
dsum = torch.zeros(h, device="cuda")
res["ln_bwd_dsum"] = timeit(lambda st: K.layernorm_bwd(dy, x, mean, rstd, g, dres, dx, dg, db, stream=st, dsum=dsum))
for n in (h, 3 * h, f):
    d = torch.randn(M, n, device="cuda").bfloat16()
    bg = torch.zeros(n, device="cuda")
    res[f"bias_grad_{n}"] = timeit(lambda st: K.bias_grad(d, bg, stream=st))
logits = torch.randn(M, 50304, device="cuda").bfloat16()  # noqa: E305
labels = torch.randint(0, 50257, (M,), device="cuda", dtype=torch.int32)
ls = torch.zeros(1, device="cuda")
res[f"xent_{M}x50304"] = timeit(lambda st: K.xent(logits, labels, 50257, 1.0, 1.0, ls, stream=st), it=10)
import os  # noqa: E402
for k, v in res.items():
    print(json.dumps({"op": k, "M": M, "h": h, "us": round(v, 2), "ln_bwd_rpw": os.environ.get("CK_LN_BWD_RPW", "1")}))
