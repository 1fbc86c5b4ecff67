"""Per-shape time of each GEMM tile configuration (CK_GEMM_TILE=pair|256|128|64, one process
per choice: the choice is read once) on the small-M stage shapes of BASELINE configs 3-5.
usage: CK_GEMM_TILE=<t> python scripts/gemm_tile_sweep.py  -> one JSON line per shape"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as K  # noqa: E402


def timeit(fn, it=20):
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
    return s.elapsed_time(e) / it * 1e3


SHAPES = []
for (Mt, h, f) in [(632, 1280, 5120), (1264, 1280, 5120), (1024, 1024, 4096)]:
    SHAPES += [(Mt, 3 * h, h, 0, 0), (Mt, h, h, 0, 0), (Mt, f, h, 0, 0), (Mt, h, f, 0, 0),
               (Mt, h, 3 * h, 0, 1), (Mt, h, f, 0, 1), (Mt, f, h, 0, 1),
               (3 * h, h, Mt, 1, 1), (h, h, Mt, 1, 1), (f, h, Mt, 1, 1), (h, f, Mt, 1, 1)]
tile = os.environ.get("CK_GEMM_TILE", "auto")
for (M, N, Kd, a, b) in SHAPES:
    A = torch.randn((Kd, M) if a else (M, Kd), device="cuda").bfloat16()
    B = torch.randn((Kd, N) if b else (N, Kd), device="cuda").bfloat16()
    f32 = bool(a and b)
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    us = timeit(lambda st: K.gemm("acc_f32" if f32 else "bf16", A, B, out, a_mn=bool(a), b_mn=bool(b), stream=st))
    print(json.dumps({"tile": tile, "shape": [M, N, Kd, a, b], "us": round(us, 2),
                      "tflops": round(2.0 * M * N * Kd / (us * 1e-6) / 1e12, 1)}), flush=True)
