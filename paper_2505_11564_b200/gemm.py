"""Thin wrapper over sd_gemm_tf32 / sd_split_tf32 (tcgen05 kind::tf32 GEMM)."""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import check, lib


class GemmDesc(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("k", C.c_int),
                ("a", C.c_void_p), ("a_small", C.c_void_p), ("lda", C.c_longlong), ("a_mn", C.c_int),
                ("b", C.c_void_p), ("b_small", C.c_void_p), ("ldb", C.c_longlong), ("b_mn", C.c_int),
                ("c", C.c_void_p), ("ldc", C.c_longlong), ("alpha", C.c_float), ("beta", C.c_float),
                ("z1", C.c_int), ("z2", C.c_int),
                ("sa1", C.c_longlong), ("sa2", C.c_longlong), ("sb1", C.c_longlong), ("sb2", C.c_longlong),
                ("sc1", C.c_longlong), ("sc2", C.c_longlong)]


_configured = False


def _cfg():
    global _configured
    if not _configured:
        L = lib()
        L.sd_gemm_tf32.argtypes = [C.POINTER(GemmDesc), C.c_void_p]
        L.sd_gemm_tf32.restype = C.c_int
        L.sd_gemm_tf32_dual.argtypes = [C.POINTER(GemmDesc), C.POINTER(GemmDesc), C.c_void_p]
        L.sd_gemm_tf32_dual.restype = C.c_int
        if hasattr(L, "sd_gemm_tf32_ex"):
            L.sd_gemm_tf32_ex.argtypes = [C.POINTER(GemmDesc), C.POINTER(GemmDesc), C.c_int, C.c_void_p]
            L.sd_gemm_tf32_ex.restype = C.c_int
        L.sd_split_tf32.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
        L.sd_split_tf32.restype = C.c_int
        _configured = True
    return lib()


def _ptr(t):
    return None if t is None else t.data_ptr()


def split(x: torch.Tensor, mode: int = 0) -> torch.Tensor:
    s = torch.empty_like(x)
    check(_cfg().sd_split_tf32(x.data_ptr(), s.data_ptr(), x.numel(), mode,
                               torch.cuda.current_stream().cuda_stream))
    return s


ONCHIP_RESIDUAL, B_EXACT, B2_EXACT = 1, 2, 4


def gemm(m, n, k, a, lda, a_mn, b, ldb, b_mn, c, ldc, alpha=1.0, beta=0.0, a_small=None, b_small=None,
         z1=1, z2=1, sa=(0, 0), sb=(0, 0), sc=(0, 0), onchip=False, b_exact=False):
    """onchip=True: 3xTF32 with the operand residuals computed in shared memory.
    b_exact=True: B is tf32-exact (bf16-valued); b_small may be None, 2 MMAs per product."""
    d = GemmDesc(m, n, k, _ptr(a), _ptr(a_small), lda, int(a_mn), _ptr(b), _ptr(b_small), ldb, int(b_mn), _ptr(c),
                 ldc, alpha, beta, z1, z2, sa[0], sa[1], sb[0], sb[1], sc[0], sc[1])
    stream = torch.cuda.current_stream().cuda_stream
    if onchip or b_exact:
        flags = (ONCHIP_RESIDUAL if onchip else 0) | (B_EXACT if b_exact else 0)
        check(_cfg().sd_gemm_tf32_ex(C.byref(d), None, flags, stream))
    else:
        check(_cfg().sd_gemm_tf32(C.byref(d), stream))


def gemm_dual(m, n, k, a, lda, a_mn, b, ldb, b_mn, a2, lda2, b2, ldb2, c, ldc, alpha=1.0, beta=0.0,
              a_small=None, b_small=None, a2_small=None, b2_small=None, z1=1, z2=1, sa=(0, 0), sb=(0, 0),
              sa2=(0, 0), sb2=(0, 0), sc=(0, 0), onchip=False):
    """C = alpha (op(A) op(B) + op(A2) op(B2)) + beta C in one launch."""
    d1 = GemmDesc(m, n, k, _ptr(a), _ptr(a_small), lda, int(a_mn), _ptr(b), _ptr(b_small), ldb, int(b_mn), _ptr(c),
                  ldc, alpha, beta, z1, z2, sa[0], sa[1], sb[0], sb[1], sc[0], sc[1])
    d2 = GemmDesc(m, n, k, _ptr(a2), _ptr(a2_small), lda2, int(a_mn), _ptr(b2), _ptr(b2_small), ldb2, int(b_mn),
                  _ptr(c), ldc, alpha, beta, z1, z2, sa2[0], sa2[1], sb2[0], sb2[1], sc[0], sc[1])
    check(_cfg().sd_gemm_tf32_ex(C.byref(d1), C.byref(d2), ONCHIP_RESIDUAL if onchip else 0,
                                 torch.cuda.current_stream().cuda_stream))


def matmul(A: torch.Tensor, B: torch.Tensor, three: bool = True, a_t: bool = False, b_t: bool = False,
           mode: int = 0) -> torch.Tensor:
    """C = op(A) @ op(B) with op = transpose when a_t / b_t (inputs contiguous fp32)."""
    M = A.shape[1] if a_t else A.shape[0]
    K = A.shape[0] if a_t else A.shape[1]
    N = B.shape[0] if b_t else B.shape[1]
    C_ = torch.empty(M, N, dtype=torch.float32, device=A.device)
    As = split(A, mode) if three else None
    Bs = split(B, mode) if three else None
    gemm(M, N, K, A, A.shape[1], a_t, B, B.shape[1], not b_t, C_, N, a_small=As, b_small=Bs)
    return C_
