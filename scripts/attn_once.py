"""One tcgen05 attention forward + backward at the GPT-2-medium stage shape (B=4, s=1024,
H=16, causal) after a warm-up -- the command profiled by ncu for profiles/."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_06925_b200 import kernels as ck  # noqa: E402

B, s, H = 4, 1024, 16
qkv = torch.randn(B * s, 3 * H * 64, device="cuda").bfloat16()
out = torch.empty(B * s, H * 64, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * s, device="cuda")
dout = torch.randn_like(out)
dqkv = torch.empty_like(qkv)
for _ in range(2):
    ck.attn_fwd_tc(qkv, out, lse, B, s, H, True)
    ck.attn_bwd(qkv, out, dout, lse, dqkv, B, s, H, True, impl="tcgen05")
torch.cuda.synchronize()
print("ok")
