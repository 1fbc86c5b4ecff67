"""tcgen05/TMA GEMM vs a plain fp32 PyTorch reference of the same op.

bf16 inputs, fp32 accumulation: fp32 outputs must match the fp32 reference to
1e-3 relative (accumulation-order noise only); bf16 outputs to one bf16 ulp (2^-8).
"""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2107_06925_b200 import kernels as ck  # noqa: E402

SHAPES = [(128, 128, 64), (256, 384, 192), (4096, 3072, 1024), (304, 200, 136), (632, 5120, 1280),
          (1000, 1000, 72), (1024, 1024, 4096), (768, 256, 4096),
          # the stage shapes (64 / 256 CTA-pair tiles, split-K weight gradient) and
          # ragged multi-wave ones
          (4096, 1024, 1024), (4096, 1024, 4096), (4096, 4096, 1024), (3000, 1800, 1000),
          (3072, 1024, 4096), (2560, 2048, 520)]


def _rand(*shape):
    return (torch.randn(*shape, device="cuda") * 0.5).to(torch.bfloat16)


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_layouts_f32(a_mn, b_mn, M, N, K):
    A = _rand(K, M) if a_mn else _rand(M, K)
    B = _rand(K, N) if b_mn else _rand(N, K)
    Af = A.float().t() if a_mn else A.float()
    Bf = B.float() if b_mn else B.float().t()
    ref = Af @ Bf
    out = torch.full((M, N), float("nan"), device="cuda")
    ck.gemm("f32", A, B, out, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-3
    acc = torch.ones(M, N, device="cuda")
    ck.gemm("acc_f32", A, B, acc, a_mn=a_mn, b_mn=b_mn)
    assert _rel(acc, ref + 1) < 1e-3


@pytest.mark.parametrize("M,N,K", SHAPES[:4] + SHAPES[8:12])
def test_fused_epilogues(M, N, K):
    A, B = _rand(M, K), _rand(N, K)
    bias = _rand(N)
    ref = A.float() @ B.float().t() + bias.float()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ck.gemm("bf16", A, B, out, bias=bias)
    assert _rel(out, ref) < 8e-3
    resid = _rand(M, N)
    ck.gemm("bias_resid", A, B, out, bias=bias, aux=resid)
    assert _rel(out, ref + resid.float()) < 8e-3
    g = torch.empty_like(out)
    ck.gemm("bias_gelu", A, B, out, bias=bias, out2=g)
    assert _rel(out, ref) < 8e-3
    assert _rel(g, torch.nn.functional.gelu(out.float(), approximate="tanh")) < 8e-3
    # dgrad with fused gelu': D = dY W (W MN-major), scaled by gelu'(U)
    Wt = _rand(N, K)  # as [rows = reduction N, cols = K]
    dY = _rand(M, N)
    U = _rand(M, K)
    d = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
    ck.gemm("gelu_bwd", dY, Wt, d, b_mn=True, aux=U)
    u = U.float().requires_grad_()
    gl = torch.nn.functional.gelu(u, approximate="tanh")
    (gp,) = torch.autograd.grad(gl.sum(), u)
    assert _rel(d, (dY.float() @ Wt.float()) * gp) < 8e-3


@pytest.mark.parametrize("M,N,K", [(4096, 1024, 4096), (4096, 4096, 1024), (3000, 1800, 1000)])
def test_deterministic(M, N, K):
    """Repeated runs of a bf16-output GEMM are bit-identical."""
    A, B = _rand(M, K), _rand(N, K)
    outs = []
    for _ in range(3):
        o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ck.gemm("bf16", A, B, o)
        outs.append(o)
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])


def test_gelu_bwd_colsum():
    """kGeluBwd with the fused bias gradient: colsum += column sums of the bf16 output."""
    M, N, K = 4096, 4096, 1024
    dY, Wt, U = _rand(M, K), _rand(K, N), _rand(M, N)
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.full((N,), 0.25, device="cuda")
    ck.gemm("gelu_bwd", dY, Wt, d, b_mn=True, aux=U, colsum=cs)
    d0 = torch.empty_like(d)
    ck.gemm("gelu_bwd", dY, Wt, d0, b_mn=True, aux=U)
    torch.cuda.synchronize()
    assert torch.equal(d, d0)
    assert _rel(cs, d.float().sum(0) + 0.25) < 1e-5


# split-K through a workspace for the bf16 epilogues (the small-M stage shapes of
# GPT-2 1.3B: N = h with a deep K) -- forced slice counts and the wave model's own choice
SPLIT_SHAPES = [(632, 1280, 5120), (632, 1280, 3840), (1264, 1280, 5120), (632, 1280, 50304), (300, 264, 1000)]


@pytest.mark.parametrize("M,N,K", SPLIT_SHAPES)
@pytest.mark.parametrize("ks", [0, 2, 3, 4])
def test_split_k_bf16_epilogues(M, N, K, ks):
    ws = torch.zeros(M * max(N, K), device="cuda")
    A, B = _rand(M, K), _rand(N, K)
    bias = _rand(N)
    ref = A.float() @ B.float().t() + bias.float()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ck.gemm("bf16", A, B, out, bias=bias, ws=ws, ksplit=ks)
    assert _rel(out, ref) < 8e-3
    resid = _rand(M, N)
    ck.gemm("bias_resid", A, B, out, bias=bias, aux=resid, ws=ws, ksplit=ks)
    assert _rel(out, ref + resid.float()) < 8e-3
    g = torch.empty_like(out)
    ck.gemm("bias_gelu", A, B, out, bias=bias, out2=g, ws=ws, ksplit=ks)
    assert _rel(out, ref) < 8e-3
    assert _rel(g, torch.nn.functional.gelu(out.float(), approximate="tanh")) < 8e-3
    # dgrad layout (B MN-major) with gelu' and the fused column sums
    Wt = _rand(K, N)
    dY = _rand(M, K)
    U = _rand(M, N)
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.zeros(N, device="cuda")
    ck.gemm("gelu_bwd", dY, Wt, d, b_mn=True, aux=U, colsum=cs, ws=ws, ksplit=ks)
    u = U.float().requires_grad_()
    gl = torch.nn.functional.gelu(u, approximate="tanh")
    (gp,) = torch.autograd.grad(gl.sum(), u)
    assert _rel(d, (dY.float() @ Wt.float()) * gp) < 8e-3
    assert _rel(cs, d.float().sum(0)) < 1e-4
    torch.cuda.synchronize()
    assert int(torch.count_nonzero(ws)) == 0  # the finalize pass leaves the workspace zeroed


# stream-K (CTA-pair kernel): tiles that leave pairs idle in the last wave are cut into
# equal K-block ranges per pair; bf16 epilogues fix up through the workspace
SK_SHAPES = [(2528, 1280, 1280), (2528, 1280, 5120), (2528, 3840, 1280), (2528, 5120, 1280), (1264, 1280, 3840),
             (600, 2000, 3000)]


@pytest.mark.parametrize("M,N,K", SK_SHAPES)
def test_stream_k_bf16_epilogues(M, N, K):
    ws = torch.zeros(8 << 20, device="cuda")  # room for 74 pair slots of 256 x 256 fp32
    A, B = _rand(M, K), _rand(N, K)
    bias = _rand(N)
    ref = A.float() @ B.float().t() + bias.float()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):  # twice: the completion counters re-arm
        ck.gemm("bf16", A, B, out, bias=bias, ws=ws)
        assert _rel(out, ref) < 8e-3
    resid = _rand(M, N)
    ck.gemm("bias_resid", A, B, out, bias=bias, aux=resid, ws=ws)
    assert _rel(out, ref + resid.float()) < 8e-3
    g = torch.empty_like(out)
    ck.gemm("bias_gelu", A, B, out, bias=bias, out2=g, ws=ws)
    assert _rel(out, ref) < 8e-3
    assert _rel(g, torch.nn.functional.gelu(out.float(), approximate="tanh")) < 8e-3
    Wt = _rand(K, N)
    dY = _rand(M, K)
    U = _rand(M, N)
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.zeros(N, device="cuda")
    ck.gemm("gelu_bwd", dY, Wt, d, b_mn=True, aux=U, colsum=cs, ws=ws)
    u = U.float().requires_grad_()
    (gp,) = torch.autograd.grad(torch.nn.functional.gelu(u, approximate="tanh").sum(), u)
    assert _rel(d, (dY.float() @ Wt.float()) * gp) < 8e-3
    assert _rel(cs, d.float().sum(0)) < 1e-4
    torch.cuda.synchronize()
    flags = ws[-320:].view(torch.int32)
    assert int(torch.count_nonzero(flags)) == 0  # every counter re-armed


@pytest.mark.parametrize("M,N,K", [(3840, 1280, 2528), (5120, 1280, 2528), (1280, 5120, 1264), (3000, 2000, 900)])
def test_stream_k_weight_gradient(M, N, K):
    """fp32 accumulate (MN-major operands, the weight-gradient layout): stream-K segments
    reduce-add straight into the output."""
    A, B = _rand(K, M), _rand(K, N)
    ref = A.float().t() @ B.float()
    acc = torch.ones(M, N, device="cuda")
    ck.gemm("acc_f32", A, B, acc, a_mn=True, b_mn=True)
    assert _rel(acc, ref + 1) < 1e-3


def test_stream_k_bf16_path_enabled():
    """The bf16 stream-K fix-up is off by default (slower than whole tiles): run
    the epilogue checks above with it forced on (CK_GEMM_STREAMK=2 is read once per
    process, hence the subprocess)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, CK_GEMM_STREAMK="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.abspath(__file__) + "::test_stream_k_bf16_epilogues"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# CTA-pair 256 x 192 tiles (K-major B): forced through the `tile` argument on the stage
# shapes the wave model gives them (N = 1280) and ragged edges in both dimensions
@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("M,N,K", [(2528, 1280, 1280), (2528, 1280, 5120), (600, 1000, 200), (256, 192, 64),
                                   (1000, 1300, 520), (1264, 3840, 1280)])
def test_pair192_tiles(a_mn, M, N, K):
    A = _rand(K, M) if a_mn else _rand(M, K)
    B = _rand(N, K)
    Af = A.float().t() if a_mn else A.float()
    ref = Af @ B.float().t()
    ws = torch.zeros(M * N + 4096, device="cuda")
    out = torch.full((M, N), float("nan"), device="cuda")
    ck.gemm("f32", A, B, out, a_mn=a_mn, ws=ws, ksplit=1, tile=1)
    assert _rel(out, ref) < 1e-3
    acc = torch.ones(M, N, device="cuda")
    ck.gemm("acc_f32", A, B, acc, a_mn=a_mn, ws=ws, ksplit=1, tile=1)
    assert _rel(acc, ref + 1) < 1e-3
    if a_mn:
        return
    bias, resid = _rand(N), _rand(M, N)
    o16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ck.gemm("bf16", A, B, o16, bias=bias, ws=ws, ksplit=1, tile=1)
    assert _rel(o16, ref + bias.float()) < 8e-3
    ck.gemm("bias_resid", A, B, o16, bias=bias, aux=resid, ws=ws, ksplit=1, tile=1)
    assert _rel(o16, ref + bias.float() + resid.float()) < 8e-3
    g = torch.empty_like(o16)
    ck.gemm("bias_gelu", A, B, o16, bias=bias, out2=g, ws=ws, ksplit=1, tile=1)
    assert _rel(o16, ref + bias.float()) < 8e-3
    assert _rel(g, torch.nn.functional.gelu(o16.float(), approximate="tanh")) < 8e-3
