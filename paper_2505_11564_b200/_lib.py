"""Loads libspecden_b200.so (the C-ABI of include/specden_b200.h) and maps its
status codes onto the reference's error taxonomy
(proj/include/specden/errors.hpp:13-41).

There is no fallback: if the CUDA library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SD_LIB_OVERRIDE"]) if os.environ.get("SD_LIB_OVERRIDE") else PKG / "libspecden_b200.so"


class SpecdenError(RuntimeError):
    pass


class ConfigError(SpecdenError):
    """config_error, errors.hpp:13-17"""


class LayoutError(SpecdenError):
    """layout_error, errors.hpp:19-22"""


class ArgumentError(SpecdenError):
    """argument_error, errors.hpp:24-27"""


class NumericalError(SpecdenError):
    """numerical_error, errors.hpp:29-32"""


class StateError(SpecdenError):
    """state_error, errors.hpp:34-38"""


class ProtocolError(SpecdenError):
    """protocol_error, errors.hpp:40-43"""


class CudaError(SpecdenError):
    pass


class NcclError(SpecdenError):
    pass


_ERRORS = {1: ConfigError, 2: LayoutError, 3: ArgumentError, 4: NumericalError, 5: StateError, 6: ProtocolError,
           7: CudaError, 8: NcclError}

u64 = C.c_uint64
u64p = C.POINTER(C.c_uint64)
dp = C.POINTER(C.c_double)
vp = C.c_void_p
i32 = C.c_int


class LanczosConfig(C.Structure):
    _fields_ = [("k_max", u64), ("eps", C.c_double), ("reorth", i32), ("prec", i32), ("probe_seed", u64),
                ("probe_dist", i32), ("selective_window", u64), ("reduction", i32)]


class LanczosInfo(C.Structure):
    _fields_ = [("n_alpha", u64), ("n_beta", u64), ("breakdown", i32), ("numerical_failure", i32),
                ("ms_apply", C.c_double), ("ms_recurrence", C.c_double), ("ms_reorth", C.c_double),
                ("ms_comm", C.c_double)]


APPLY_FN = C.CFUNCTYPE(i32, vp, vp, vp, vp)

_SIGS = {
    "sd_last_error": (C.c_char_p, []),
    "sd_abi_version": (i32, []),
    "sd_launch_count": (u64, []),
    "sd_gemm_profile_begin": (i32, []),
    "sd_gemm_profile_end": (i32, [dp, dp, u64p]),
    "sd_keyed_counter": (u64, [u64, u64]),
    "sd_rademacher": (C.c_double, [u64, u64]),
    "sd_uniform_index": (u64, [u64, u64, u64]),
    "sd_split_evenly": (i32, [u64, u64, u64p, u64p, u64p]),
    "sd_validate_layout": (i32, [u64, u64, u64p, u64p]),
    "sd_layout_owner": (i32, [u64, u64p, u64, u64p]),
    "sd_partial_shape": (i32, [u64, u64, u64, u64p, u64p, u64p]),
    "sd_partial_len": (u64, [u64, u64, u64]),
    "sd_combine_partials_host": (i32, [u64, u64p, u64p, u64, C.POINTER(dp), dp]),
    "sd_k_probe_fill": (i32, [vp, u64, u64, u64, i32, u64, i32, vp]),
    "sd_k_dot_partial": (i32, [vp, vp, u64, u64, u64, i32, vp, vp]),
    "sd_k_combine": (i32, [u64, u64p, u64p, u64, u64, vp, vp, vp]),
    "sd_k_axpy": (i32, [vp, vp, u64, vp, C.c_double, i32, vp]),
    "sd_k_scale": (i32, [vp, vp, u64, vp, i32, i32, vp]),
    "sd_k_axpy_dot": (i32, [vp, vp, vp, vp, u64, u64, u64, i32, vp, vp]),
    "sd_k_cgs": (i32, [vp, u64, u64, vp, vp, i32, u64, u64, u64, i32, vp, vp]),
    "sd_k_dense_apply": (i32, [vp, u64, vp, vp, u64, u64, i32, vp]),
    "sd_k_abs_stats": (i32, [vp, u64, i32, vp, i32, vp, vp, vp]),
    "sd_k_abs_histogram": (i32, [vp, u64, i32, C.c_double, i32, vp, vp]),
    "sd_ritz_decompose": (i32, [u64, dp, dp, dp, dp, dp]),
    "sd_smooth_density": (i32, [u64, dp, dp, C.c_double, u64, dp, dp, dp]),
    "sd_wigner_dense": (i32, [u64, C.c_double, u64, dp]),
    "sd_spiked_dense": (i32, [u64, C.c_double, dp, u64, u64, dp]),
    "sd_nccl_unique_id": (i32, [C.c_char_p]),
    "sd_comm_nccl_create": (i32, [C.c_char_p, i32, i32, C.POINTER(vp)]),
    "sd_comm_destroy": (i32, [vp]),
    "sd_comm_local_create": (i32, [i32, C.POINTER(vp)]),
    "sd_comm_abort": (i32, [vp]),
    "sd_comm_allreduce_f32": (i32, [vp, vp, u64, vp]),
    "sd_comm_allgather": (i32, [vp, vp, vp, u64, vp]),
    "sd_operator_custom": (i32, [u64, APPLY_FN, vp, C.POINTER(vp)]),
    "sd_operator_dense": (i32, [u64, dp, C.POINTER(vp)]),
    "sd_operator_diag": (i32, [u64, vp, i32, C.POINTER(vp)]),
    "sd_operator_apply": (i32, [vp, vp, vp, i32, vp]),
    "sd_operator_dim": (u64, [vp]),
    "sd_operator_destroy": (i32, [vp]),
    "sd_lanczos_workspace_bytes": (u64, [u64p, u64p, u64, C.POINTER(LanczosConfig), i32, i32]),
    "sd_lanczos_run": (i32, [vp, vp, u64p, u64p, u64, C.POINTER(LanczosConfig), vp, u64, dp, dp,
                             C.POINTER(LanczosInfo), vp]),
    "sd_lanczos_begin": (i32, [vp, vp, u64p, u64p, u64, C.POINTER(LanczosConfig), vp, u64, vp, C.POINTER(vp)]),
    "sd_lanczos_step": (i32, [vp, C.POINTER(i32)]),
    "sd_lanczos_result": (i32, [vp, dp, dp, C.POINTER(LanczosInfo)]),
    "sd_lanczos_current": (vp, [vp]),
    "sd_lanczos_basis": (i32, [vp, C.POINTER(vp), u64p]),
    "sd_lanczos_basis_ld": (u64, [vp]),
    "sd_lanczos_orthogonality": (i32, [vp, dp]),
    "sd_lanczos_end": (i32, [vp]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded CUDA library; raises if it is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2505_11564_b200.build` "
                              "(the product has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name, None)
            if f is None:
                continue
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().sd_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, SpecdenError)(msg)


def exported_symbols() -> list[str]:
    return list(_SIGS)
