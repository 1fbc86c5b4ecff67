import json, os, subprocess, sys
code = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck
out = []
for epi in ["bf16", "f32"]:
    for K in [128, 256, 512, 1024, 2048, 4096]:
        M = N = 4096
        A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
        o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if epi == "bf16" else torch.float32)
        f = lambda: ck.gemm(epi, A, B, o)
        for _ in range(3): f()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        out.append([epi, K, round(ms * 1000, 1), round(2 * M * N * K / ms / 1e9, 1)])
print(json.dumps(out))
'''
res = {}
for tile in ["pair", "256"]:
    env = dict(os.environ, CK_GEMM_TILE=tile)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    res[tile] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-2000:]
print(json.dumps(res))
