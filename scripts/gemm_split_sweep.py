"""Time every (tile, K-slices) variant of the bf16-epilogue GEMM on the small-M stage
shapes -> JSON lines.  20 launches are captured in a CUDA graph and the graph replay is
timed with CUDA events (as inside a training step: no host launch cost -- timing eager
ctypes calls measures the ~15 us host path, not the kernel).

    python scripts/gemm_split_sweep.py > gpurun_out/split_sweep.jsonl"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck  # noqa: E402

h, f = 1280, 5120
SHAPES = []
for M in (632, 1264, 2528):
    SHAPES += [(M, 3 * h, h, 0), (M, h, h, 0), (M, f, h, 0), (M, h, f, 0), (M, h, 3 * h, 1), (M, h, f, 1)]


def graph_us(run, reps=20):
    """Average device time of `run` (one GEMM) from a CUDA-graph replay of `reps` calls."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            run()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            run()
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
    ws = torch.zeros(2528 * 5120, device="cuda")
    for (M, N, K, bmn) in SHAPES:
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).bfloat16()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        res = {"shape": [M, N, K, bmn]}
        for tile in (0, 256, 128, 64):
            for ks in (1, 2, 3, 4):
                if tile == 0 and (M < 256 or N < 256):
                    continue
                if ks > 1 and K // 64 // ks < 8:
                    continue
                run = lambda: ck.gemm("bf16", A, B, out, b_mn=bool(bmn), ws=ws, ksplit=ks, tile=tile,
                                      stream=torch.cuda.current_stream())
                res[f"{tile}/{ks}"] = round(graph_us(run), 2)
        # the wave model's own choice
        res["auto"] = round(graph_us(lambda: ck.gemm("bf16", A, B, out, b_mn=bool(bmn), ws=ws,
                                                     stream=torch.cuda.current_stream())), 2)
        best = min((v, k) for k, v in res.items() if k != "shape")
        res["best"] = best[1]
        res["best_tflops"] = round(2.0 * M * N * K / (best[0] * 1e-6) / 1e12, 1)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
