"""Bitwise run-to-run determinism of each forward kernel at the tiny-GPT shapes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck

torch.manual_seed(0)
M, h, f, V, B, s, H = 256, 256, 1024, 1024, 2, 128, 4
def r(*sh): return (torch.randn(*sh, device="cuda") * 0.5).bfloat16()

def check(name, fn, n=30):
    outs = [fn().clone() for _ in range(n)]
    torch.cuda.synchronize()
    bad = sum(int(not torch.equal(outs[0], o)) for o in outs[1:])
    print(f"{name:30s} mismatching runs {bad}/{n-1}", flush=True)

x, g, b = r(M, h), r(h), r(h)
y = torch.empty_like(x); mean = torch.empty(M, device="cuda"); rstd = torch.empty(M, device="cuda")
check("layernorm_fwd", lambda: (ck.layernorm_fwd(x, g, b, y, mean, rstd), y)[1])
for (N, K) in [(3 * h, h), (h, h), (f, h), (h, f), (V, h)]:
    A, W_ = r(M, K), r(N, K)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    check(f"gemm bf16 M={M} N={N} K={K}", lambda: (ck.gemm("bf16", A, W_, out), out)[1])
    ref = A.float() @ W_.float().t()
    print("   rel err", ((out.float() - ref).norm() / ref.norm()).item())
qkv = r(M, 3 * h)
o = torch.empty(M, h, device="cuda", dtype=torch.bfloat16); lse = torch.empty(B * H * s, device="cuda")
check("attn_fwd", lambda: (ck.attn_fwd(qkv, o, lse, B, s, H, True), o)[1])
tok = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
wte, wpe = r(V, h), r(s, h)
check("embed_fwd", lambda: (ck.embed_fwd(tok, wte, wpe, y, s), y)[1])
logits = r(M, V)
lab = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
ls = torch.zeros(1, device="cuda")
def xe():
    w = logits.clone(); ck.xent(w, lab, V, 1e-3, 1e-3, ls); return w
check("xent", xe)
# many back-to-back small GEMMs on 4 streams (executor-like concurrency)
streams = [torch.cuda.Stream() for _ in range(4)]
As = [r(M, h) for _ in range(4)]; Ws = [r(3 * h, h) for _ in range(4)]
outs = [torch.empty(M, 3 * h, device="cuda", dtype=torch.bfloat16) for _ in range(4)]
refs = [(a.float() @ w.float().t()) for a, w in zip(As, Ws)]
worst = 0
for it in range(200):
    for k in range(4):
        with torch.cuda.stream(streams[k]):
            ck.gemm("bf16", As[k], Ws[k], outs[k], stream=streams[k])
    torch.cuda.synchronize()
    for k in range(4):
        worst = max(worst, ((outs[k].float() - refs[k]).norm() / refs[k].norm()).item())
print("concurrent gemm worst rel err over 200 iters", worst)
