"""Direct launchers for the sm_100a kernels (device pointers through the C-ABI).

Used by the kernel tests and microbenchmarks; torch is only the allocator here.
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import check, lib

_vp, _ll, _i = C.c_void_p, C.c_longlong, C.c_int
_lib.register("ck_gemm_bf16", _i, [_i, _i, _i, _i, _i, _i, _vp, _ll, _vp, _ll, _vp, _ll, _vp, _vp, _ll,
                                   _vp, _ll, _vp])
_lib.register("ck_gemm_bf16_ex", _i, [_i, _i, _i, _i, _i, _i, _vp, _ll, _vp, _ll, _vp, _ll, _vp, _vp, _ll,
                                      _vp, _ll, _vp, _vp])
_lib.register("ck_gemm_bf16_split", _i, [_i, _i, _i, _i, _i, _i, _vp, _ll, _vp, _ll, _vp, _ll, _vp, _vp, _ll,
                                         _vp, _ll, _vp, _vp, _ll, _i, _i, _vp])

EPI = {"bf16": 0, "bias_gelu": 1, "bias_resid": 2, "gelu_bwd": 3, "acc_f32": 4, "f32": 5}


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def gemm(epi, A, B, out, *, a_mn=False, b_mn=False, M=None, N=None, K=None, bias=None, aux=None,
         out2=None, stream=None, colsum=None, ws=None, ksplit=0, tile=-1):
    """D[m,n] = sum_k A(m,k) B(n,k) with A/B K-major ([M,K]/[N,K]) or MN-major ([K,M]/[K,N]).
    `colsum` (fp32 [N], gelu_bwd only) accumulates the column sums of the bf16 output."""
    M = M if M is not None else (A.shape[1] if a_mn else A.shape[0])
    K = K if K is not None else (A.shape[0] if a_mn else A.shape[1])
    N = N if N is not None else (B.shape[1] if b_mn else B.shape[0])
    args = (EPI[epi], int(a_mn), int(b_mn), M, N, K, _p(A), A.stride(0), _p(B), B.stride(0), _p(out),
            out.stride(0), _p(bias), _p(aux), aux.stride(0) if aux is not None else 0, _p(out2),
            out2.stride(0) if out2 is not None else 0)
    if ws is not None:  # split-K workspace route (fp32, zero-filled, >= M*N)
        check(lib().ck_gemm_bf16_split(*args, _p(colsum), _p(ws), ws.numel(), int(ksplit), int(tile),
                                       _stream(stream)))
    elif colsum is None:
        check(lib().ck_gemm_bf16(*args, _stream(stream)))
    else:
        check(lib().ck_gemm_bf16_ex(*args, _p(colsum), _stream(stream)))
    return out

_fp = C.POINTER(C.c_float)
_lib.register("ck_layernorm_fwd", _i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp])
_lib.register("ck_layernorm_bwd", _i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp])
_lib.register("ck_layernorm_bwd_dsum", _i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp])
_lib.register("ck_embed_fwd", _i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp])
_lib.register("ck_embed_bwd", _i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp])
_lib.register("ck_xent_fwd_bwd", _i, [_vp, _ll, _vp, _i, _i, _i, C.c_float, C.c_float, _vp, _vp])
_lib.register("ck_bias_grad", _i, [_vp, _vp, _i, _i, _vp])
_lib.register("ck_sgd_update", _i, [_vp, _vp, _vp, _i, _ll, C.c_float, _vp])
_lib.register("ck_attn_fwd", _i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp])
_lib.register("ck_attn_fwd_tc", _i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp])
_lib.register("ck_attn_bwd", _i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp])
_lib.register("ck_attn_bwd_scratch_floats", _ll, [_i, _i, _i])
_lib.register("ck_attn_bwd_tc", _i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp])
_lib.register("ck_attn_bwd_tc_dbias", _i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp])


def layernorm_fwd(x, g, b, y, mean, rstd, stream=None):
    M, h = x.shape
    check(lib().ck_layernorm_fwd(_p(x), _p(g), _p(b), _p(y), _p(mean), _p(rstd), M, h, _stream(stream)))


def layernorm_bwd(dy, x, mean, rstd, g, dres, dx, dgamma, dbeta, stream=None, dsum=None):
    M, h = x.shape
    if dsum is None:
        check(lib().ck_layernorm_bwd(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), _p(dres), _p(dx), _p(dgamma),
                                     _p(dbeta), M, h, _stream(stream)))
    else:
        check(lib().ck_layernorm_bwd_dsum(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), _p(dres), _p(dx),
                                          _p(dgamma), _p(dbeta), _p(dsum), M, h, _stream(stream)))


def embed_fwd(tok, wte, wpe, x, seq, stream=None):
    check(lib().ck_embed_fwd(_p(tok), _p(wte), _p(wpe), _p(x), x.shape[0], seq, x.shape[1], _stream(stream)))


def embed_bwd(tok, dx, dwte, dwpe, seq, stream=None):
    check(lib().ck_embed_bwd(_p(tok), _p(dx), _p(dwte), _p(dwpe), dx.shape[0], seq, dx.shape[1],
                             _stream(stream)))


def xent(logits, labels, V, grad_scale, loss_scale, loss_sum, stream=None):
    M, Vp = logits.shape
    check(lib().ck_xent_fwd_bwd(_p(logits), logits.stride(0), _p(labels), M, V, Vp, grad_scale, loss_scale,
                                _p(loss_sum), _stream(stream)))


def bias_grad(dy, db, stream=None):
    check(lib().ck_bias_grad(_p(dy), _p(db), dy.shape[0], dy.shape[1], _stream(stream)))


def attn_fwd(qkv, out, lse, B, seq, H, causal=True, stream=None):
    check(lib().ck_attn_fwd(_p(qkv), _p(out), _p(lse), B, seq, H, int(causal), _stream(stream)))


def attn_fwd_tc(qkv, out, lse, B, seq, H, causal=True, stream=None):
    check(lib().ck_attn_fwd_tc(_p(qkv), _p(out), _p(lse), B, seq, H, int(causal), _stream(stream)))


def attn_bwd(qkv, out, dout, lse, dqkv, B, seq, H, causal=True, stream=None, impl="mma_sync", dbias=None):
    """dbias (fp32 [3 H 64], tcgen05 only) accumulates the column sums of dqkv (QKV bias grad)."""
    import torch
    n = lib().ck_attn_bwd_scratch_floats(B, seq, H)
    scratch = torch.empty(n, device=qkv.device, dtype=torch.float32)
    if dbias is not None:
        check(lib().ck_attn_bwd_tc_dbias(_p(qkv), _p(out), _p(dout), _p(lse), _p(dqkv), _p(scratch), _p(dbias), B,
                                         seq, H, int(causal), _stream(stream)))
        return
    fn = lib().ck_attn_bwd if impl == "mma_sync" else lib().ck_attn_bwd_tc
    check(fn(_p(qkv), _p(out), _p(dout), _p(lse), _p(dqkv), _p(scratch), B, seq, H,
                            int(causal), _stream(stream)))
