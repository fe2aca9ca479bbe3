"""ctypes binding of libofrr_b200.so (the C ABI in include/ofrr_b200.h).

The product path has no CPU fallback: if the shared library is missing or cannot be
loaded, every entry point raises ``NativeLibraryError`` instead of computing anything
on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libofrr_b200.so")

# format codes (include/ofrr_b200.h; ofrr/precision.py:20-25 + extensions)
F16, F32, F64, BF16, FP8E4M3 = 0, 1, 2, 3, 4

OK = 0
ERR_INVALID, ERR_CUDA, ERR_OVERFLOW, ERR_EMPTY_BASIS, ERR_EMPTY_PENCIL, ERR_CONVERGENCE, \
    ERR_UNSUPPORTED = 1, 2, 3, 4, 5, 6, 7
FLAG_NONFINITE, FLAG_NOCONV, FLAG_INEXACT = 1, 2, 4

_lock = threading.Lock()
_lib = None

c_int, c_i64, c_sz, c_dbl, c_vp = ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_double, ctypes.c_void_p

_SIGS = {
    "ofrr_abi_version": ([], c_int),
    "ofrr_last_error": ([], ctypes.c_char_p),
    "ofrr_device_sm_count": ([c_int], c_int),
    "ofrr_gemm_av_workspace": ([c_i64, c_i64, c_int, c_int, c_int], c_sz),
    "ofrr_gemm_av": ([c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_vp, c_i64, c_int, c_vp, c_i64, c_int,
                      c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "ofrr_gemm_av2": ([c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_vp, c_i64, c_int, c_vp, c_i64, c_int,
                       c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_gemm_av_split_workspace": ([c_i64, c_i64, c_int], c_sz),
    "ofrr_gemm_av_split": ([c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp, c_vp,
                            c_vp, c_i64, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_gemm_av_split_slices": ([c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp,
                                   c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_residual_estimate_workspace": ([c_i64, c_int], c_sz),
    "ofrr_residual_estimate": ([c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_i64, c_int, c_vp, c_int, c_vp, c_vp,
                                c_int, c_vp, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_prof_gemm_enable": ([c_int], None),
    "ofrr_prof_gemm_read": ([c_vp, c_int], c_int),
    "ofrr_prof_gemm_active": ([], c_int),
    "ofrr_prof_gemm_collect": ([], c_int),
    "ofrr_prof_gemm_claim": ([], c_int),
    "ofrr_prof_gemm_collect_group": ([c_int], c_int),
    "ofrr_prof_k1_stamp": ([c_int], c_int),
    "ofrr_prof_k1_read": ([c_vp, c_vp], c_int),
    "ofrr_prof_oz_stamp": ([c_int], c_int),
    "ofrr_prof_oz_read": ([c_vp, c_vp], c_int),
    "ofrr_prof_oz_read_tier": ([c_int, c_vp, c_vp], c_int),
    "ofrr_loop_ctl_bytes": ([], c_sz),
    "ofrr_loop_build": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_int, c_int, c_int,
                         c_dbl, c_vp], c_int),
    "ofrr_loop_build_rung": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_int, c_int, c_int,
                              c_dbl, c_vp], c_int),
    "ofrr_loop_launch": ([c_vp, c_vp], c_int),
    "ofrr_loop_destroy": ([c_vp], c_int),
    "ofrr_scale_columns": ([c_vp, c_i64, c_int, c_i64, c_int, c_int, c_vp, c_vp], c_int),
    "ofrr_hessenberg_workspace": ([c_i64, c_int, c_int], c_sz),
    "ofrr_hessenberg": ([c_vp, c_i64, c_int, c_i64, c_int, c_int, c_dbl, c_vp, c_i64, c_vp, c_vp, c_vp,
                         c_vp, c_sz, c_vp], c_int),
    "ofrr_gram_workspace": ([c_i64, c_int, c_int], c_sz),
    "ofrr_gram": ([c_vp, c_i64, c_vp, c_i64, c_i64, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp,
                   c_sz, c_vp], c_int),
    "ofrr_small_eig_workspace": ([c_int], c_sz),
    "ofrr_sym_def_gen_eig": ([c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "ofrr_sym_eig": ([c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp], c_int),
    "ofrr_ritz_recover": ([c_vp, c_i64, c_int, c_i64, c_int, c_vp, c_int, c_vp, c_int, c_dbl, c_vp, c_i64,
                           c_vp, c_i64, c_int, c_vp, c_vp], c_int),
    "ofrr_reuse_power": ([c_vp, c_i64, c_int, c_i64, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_i64, c_int, c_vp,
                          c_vp, c_vp], c_int),
    "ofrr_residual_workspace": ([c_i64, c_int], c_sz),
    "ofrr_residual_workspace2": ([c_i64, c_i64, c_int, c_int, c_int], c_sz),
    "ofrr_ozaki_operator_workspace": ([c_i64, c_i64], c_sz),
    "ofrr_ozaki_workspace": ([c_i64, c_i64, c_int], c_sz),
    "ofrr_ozaki_operator_info": ([c_vp, c_i64, c_vp, c_vp], c_int),
    "ofrr_ozaki_gemm_levels": ([c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp,
                                c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_orthonormalize_workspace": ([c_i64, c_int], c_sz),
    "ofrr_orthonormalize": ([c_vp, c_i64, c_int, c_i64, c_int, c_int, c_int, c_dbl, c_int, c_int, c_vp, c_i64, c_vp,
                             c_vp, c_vp, c_sz, c_vp], c_int),
    "ofrr_gaussian_kernel": ([c_vp, c_i64, c_vp, c_i64, c_dbl, c_dbl, c_dbl, c_vp, c_i64, c_int, c_vp], c_int),
    "ofrr_ozaki_prepare": ([c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_ozaki_gemm": ([c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp, c_vp,
                         c_vp, c_i64, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_ozaki_residual": ([c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_int, c_vp,
                             c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_residual_eig": ([c_vp, c_i64, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_int, c_vp, c_vp, c_sz,
                           c_vp], c_int),
    "ofrr_residual_pair": ([c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp,
                            c_int, c_vp, c_int, c_vp, c_sz, c_vp], c_int),
    "ofrr_generate_sym": ([c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_i64, c_int,
                           c_vp], c_int),
    "ofrr_start_block_pcg64": ([ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, c_i64, c_int,
                                c_vp, c_i64, c_int, c_vp], c_int),
    "ofrr_convert": ([c_vp, c_int, c_i64, c_vp, c_int, c_i64, c_i64, c_i64, c_vp, c_vp], c_int),
    "ofrr_transpose_convert": ([c_vp, c_int, c_i64, c_vp, c_int, c_i64, c_i64, c_i64, c_vp, c_vp], c_int),
    "ofrr_restart_workspace": ([c_i64, c_int], c_sz),
    "ofrr_restart": ([c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_i64, c_int, c_vp, c_int, c_vp, c_int, c_vp, c_i64,
                      c_int, c_vp, c_vp, c_i64, c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_int, c_vp, c_sz,
                      c_vp], c_int),
    "ofrr_upload_sym": ([c_vp, c_i64, c_vp, c_i64, c_i64, c_int, c_int, c_i64, c_vp, c_vp], c_int),
    "ofrr_host_gemm_mixed": ([c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_int,
                              c_int, c_vp], c_int),
    "ofrr_host_jacobi_eig": ([c_vp, c_i64, c_int, c_dbl, c_vp, c_vp, c_vp, c_vp], c_int),
}

EXPORTED = tuple(_SIGS)


class NativeLibraryError(RuntimeError):
    """libofrr_b200.so is missing or unusable (there is deliberately no fallback)."""


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle; raises NativeLibraryError."""
    global _lib
    if _lib is not None:
        return _lib
    # A/B experiments only: another build of the same library (scripts/)
    path = os.environ.get("OFRR_LIB_OVERRIDE", path)
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} not found: build it with `python -m paper_2505_00281_b200.build` "
                "(nvcc, sm_100a); there is no CPU fallback")
        try:
            lib = ctypes.CDLL(path)
        except OSError as e:  # pragma: no cover - environment specific
            raise NativeLibraryError(f"cannot load {path}: {e}") from e
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def last_error() -> str:
    return load().ofrr_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Map a C status onto the reference's exception classes."""
    if rc == OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_OVERFLOW:
        raise errors.OverflowDiagnostic(msg)
    if rc == ERR_EMPTY_BASIS:
        raise errors.EmptyBasisError(msg)
    if rc == ERR_EMPTY_PENCIL:
        raise errors.EmptyPencilError(msg)
    if rc == ERR_CONVERGENCE:
        raise errors.ConvergenceError(msg, float("nan"))
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)
