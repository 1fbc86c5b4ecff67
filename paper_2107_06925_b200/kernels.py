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

EPI = {"bf16": 0, "bias_gelu": 1, "bias_resid": 2, "gelu_bwd": 3, "acc_f32": 4, "f32": 5}


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def gemm(epi, A, B, out, *, a_mn=False, b_mn=False, M=None, N=None, K=None, bias=None, aux=None,
         out2=None, stream=None):
    """D[m,n] = sum_k A(m,k) B(n,k) with A/B K-major ([M,K]/[N,K]) or MN-major ([K,M]/[K,N])."""
    M = M if M is not None else (A.shape[1] if a_mn else A.shape[0])
    K = K if K is not None else (A.shape[0] if a_mn else A.shape[1])
    N = N if N is not None else (B.shape[1] if b_mn else B.shape[0])
    check(lib().ck_gemm_bf16(EPI[epi], int(a_mn), int(b_mn), M, N, K, _p(A), A.stride(0), _p(B),
                             B.stride(0), _p(out), out.stride(0), _p(bias), _p(aux),
                             aux.stride(0) if aux is not None else 0, _p(out2),
                             out2.stride(0) if out2 is not None else 0, _stream(stream)))
    return out
