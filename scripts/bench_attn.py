import sys, torch, json
sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck
res = []
for (B, s, H, causal) in [(4, 1024, 16, True), (8, 128, 16, False), (1, 632, 20, True)]:
    qkv = torch.randn(B * s, 3 * H * 64, device="cuda").bfloat16()
    out = torch.empty(B * s, H * 64, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * s, device="cuda")
    dout = torch.randn_like(out); dqkv = torch.empty_like(qkv)
    fl = 4 * s * s * 64 * B * H * (0.5 if causal else 1.0)
    for name, fn in [("fwd_mma", lambda: ck.attn_fwd(qkv, out, lse, B, s, H, causal)),
                     ("fwd_tc", lambda: ck.attn_fwd_tc(qkv, out, lse, B, s, H, causal)),
                     ("bwd_mma", lambda: ck.attn_bwd(qkv, out, dout, lse, dqkv, B, s, H, causal)),
                     ("bwd_tc", lambda: ck.attn_bwd(qkv, out, dout, lse, dqkv, B, s, H, causal, impl="tcgen05"))]:
        for _ in range(3): fn()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        f = fl * (2.5 if name.startswith("bwd") else 1.0)
        res.append({"shape": [B, s, H, causal], "kernel": name, "us": round(ms * 1000, 1), "tflops": round(f / ms / 1e9, 1)})
        print(json.dumps(res[-1]), flush=True)
