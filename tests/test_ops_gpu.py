"""Memory-bound stage kernels and flash attention vs plain fp32 PyTorch references.

Tolerances (bf16 storage, fp32 math): relative Frobenius error <= 1e-2 for bf16
outputs, <= 1e-4 for fp32 statistics / reductions.
"""
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2107_06925_b200 import kernels as ck  # noqa: E402

F = torch.nn.functional


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("M,h", [(4096, 1024), (130, 256), (632, 1280)])
def test_layernorm(M, h):
    x = torch.randn(M, h, device="cuda").bfloat16()
    g = (1 + 0.1 * torch.randn(h, device="cuda")).bfloat16()
    b = (0.1 * torch.randn(h, device="cuda")).bfloat16()
    y = torch.empty_like(x)
    mean = torch.empty(M, device="cuda")
    rstd = torch.empty(M, device="cuda")
    ck.layernorm_fwd(x, g, b, y, mean, rstd)
    xf = x.float().requires_grad_()
    gf = g.float().requires_grad_()
    bf = b.float().requires_grad_()
    ref = F.layer_norm(xf, (h,), gf, bf, 1e-5)
    assert rel(y, ref) < 1e-2
    assert rel(mean, x.float().mean(1)) < 1e-4
    dy = torch.randn(M, h, device="cuda").bfloat16()
    dres = torch.randn(M, h, device="cuda").bfloat16()
    dx = torch.empty_like(x)
    dg = torch.zeros(h, device="cuda")
    db = torch.zeros(h, device="cuda")
    ck.layernorm_bwd(dy, x, mean, rstd, g, dres, dx, dg, db)
    rdx, rdg, rdb = torch.autograd.grad(ref, (xf, gf, bf), dy.float())
    assert rel(dx, rdx + dres.float()) < 1e-2
    assert rel(dg, rdg) < 1e-3 and rel(db, rdb) < 1e-3
    # fused bias gradient: dsum += column sums of the bf16 dx the kernel wrote
    dx2 = torch.empty_like(x)
    ds = torch.full((h,), 0.5, device="cuda")
    ck.layernorm_bwd(dy, x, mean, rstd, g, dres, dx2, torch.zeros(h, device="cuda"), torch.zeros(h, device="cuda"),
                     dsum=ds)
    assert torch.equal(dx2, dx)
    assert rel(ds, dx.float().sum(0) + 0.5) < 1e-5


def test_embedding():
    V, S, h, B, s = 1000, 64, 256, 3, 64
    wte = torch.randn(V, h, device="cuda").bfloat16()
    wpe = torch.randn(S, h, device="cuda").bfloat16()
    tok = torch.randint(0, V, (B * s,), device="cuda", dtype=torch.int32)
    x = torch.empty(B * s, h, device="cuda", dtype=torch.bfloat16)
    ck.embed_fwd(tok, wte, wpe, x, s)
    ref = wte.float()[tok.long()] + wpe.float()[torch.arange(B * s, device="cuda") % s]
    assert rel(x, ref) < 1e-2
    dx = torch.randn(B * s, h, device="cuda").bfloat16()
    dwte = torch.zeros(V, h, device="cuda")
    dwpe = torch.zeros(S, h, device="cuda")
    ck.embed_bwd(tok, dx, dwte, dwpe, s)
    rw = torch.zeros(V, h, device="cuda").index_add_(0, tok.long(), dx.float())
    rp = dx.float().view(B, s, h).sum(0)
    assert rel(dwte, rw) < 1e-5 and rel(dwpe, rp) < 1e-5


# register-resident row (Vp <= 16 * 4096: several footprints) and the two-pass fallback
@pytest.mark.parametrize("M,V,Vp", [(256, 50257, 50304), (64, 1000, 1024), (32, 30522, 30592), (16, 5000, 5120),
                                   (8, 120000, 120064)])
def test_xent(M, V, Vp):
    logits = (3 * torch.randn(M, Vp, device="cuda")).bfloat16()
    labels = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
    lf = logits.float()[:, :V].requires_grad_()
    loss = F.cross_entropy(lf, labels.long(), reduction="sum")
    (grad,) = torch.autograd.grad(loss, lf)
    ls = torch.zeros(1, device="cuda")
    work = logits.clone()
    ck.xent(work, labels, V, 0.5, 1.0 / M, ls)
    assert abs(ls.item() - loss.item() / M) < 1e-3 * max(1.0, loss.item() / M)
    assert rel(work[:, :V], 0.5 * grad) < 1e-2
    assert work[:, V:].float().abs().max().item() == 0.0


def test_bias_grad():
    dy = torch.randn(1000, 3072, device="cuda").bfloat16()
    db = torch.ones(3072, device="cuda")
    ck.bias_grad(dy, db)
    assert rel(db, dy.float().sum(0) + 1) < 1e-5


@pytest.mark.parametrize("impl", ["mma_sync", "tcgen05"])
@pytest.mark.parametrize("B,seq,H,causal", [(2, 256, 4, True), (1, 1024, 2, True), (2, 128, 16, False),
                                             (1, 200, 2, True), (1, 632, 2, False), (3, 632, 2, True),
                                             (2, 203, 3, True), (2, 384, 2, False)])
def test_attention(B, seq, H, causal, impl):
    d = 64
    qkv = (torch.randn(B * seq, 3 * H * d, device="cuda")).bfloat16()
    out = torch.empty(B * seq, H * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * seq, device="cuda")
    (ck.attn_fwd if impl == "mma_sync" else ck.attn_fwd_tc)(qkv, out, lse, B, seq, H, causal)
    q, k, v = qkv.float().view(B, seq, 3, H, d).permute(2, 0, 3, 1, 4)
    q, k, v = (t.contiguous().requires_grad_() for t in (q, k, v))
    s = q @ k.transpose(-1, -2) / math.sqrt(d)
    if causal:
        s = s.masked_fill(torch.ones(seq, seq, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
    ref_lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    ref = o.permute(0, 2, 1, 3).reshape(B * seq, H * d)
    assert rel(out, ref) < 1e-2
    assert rel(lse, ref_lse.reshape(-1)) < 1e-4
    dout = torch.randn_like(out)
    dqkv = torch.empty_like(qkv)
    ck.attn_bwd(qkv, out, dout, lse, dqkv, B, seq, H, causal, impl=impl)
    dq, dk, dv = torch.autograd.grad(ref, (q, k, v), dout.float())
    got = dqkv.float().view(B, seq, 3, H, d).permute(2, 0, 3, 1, 4)
    assert rel(got[0], dq) < 2e-2
    assert rel(got[1], dk) < 2e-2
    assert rel(got[2], dv) < 2e-2
    if impl == "tcgen05":  # fused QKV bias gradient: column sums of the dqkv written
        db = torch.full((3 * H * d,), 0.5, device="cuda")
        dqkv2 = torch.empty_like(qkv)
        ck.attn_bwd(qkv, out, dout, lse, dqkv2, B, seq, H, causal, impl=impl, dbias=db)
        assert rel(dqkv2, dqkv) < 1e-3  # dQ is reduce-added in L2: order-dependent fp32 sums
        assert rel(db, dqkv2.float().sum(0) + 0.5) < 1e-5
