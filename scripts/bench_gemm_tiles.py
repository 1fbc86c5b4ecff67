"""Compare the GEMM tile variants (CK_GEMM_TILE=pair|256|128 set per subprocess)."""
import json, os, subprocess, sys
shapes = [(4096, 3072, 1024, 0, 0), (4096, 1024, 1024, 0, 0), (4096, 4096, 1024, 0, 0), (4096, 1024, 4096, 0, 0),
          (4096, 1024, 4096, 0, 1), (4096, 4096, 1024, 0, 1), (3072, 1024, 4096, 1, 1), (1024, 4096, 4096, 1, 1),
          (4096, 50304, 1024, 0, 0), (8192, 8192, 8192, 0, 0)]
code = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck
shapes = json.loads(sys.argv[1])
out = []
for (M, N, K, a, b) in shapes:
    A = torch.randn((K, M) if a else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b else (N, K), device="cuda").bfloat16()
    o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = lambda: ck.gemm("bf16", A, B, o, a_mn=bool(a), b_mn=bool(b))
    f(); torch.cuda.synchronize()
    ref = (A.float().t() if a else A.float()) @ (B.float() if b else B.float().t())
    err = ((o.float() - ref).norm() / ref.norm()).item()
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    out.append({"shape": [M, N, K, a, b], "tflops": round(2 * M * N * K / ms / 1e9, 1), "err": err})
print(json.dumps(out))
'''
res = {}
for tile in ["pair", "256", "128"]:
    env = dict(os.environ, CK_GEMM_TILE=tile)
    p = subprocess.run([sys.executable, "-c", code, json.dumps(shapes)], env=env, capture_output=True, text=True, timeout=240)
    res[tile] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-2000:]
print(json.dumps(res))
