"""The B200 kernel backend for the REFERENCE package's plugin slot ``ofrr.backend.kernels``
(ofrr/backend.py:14-22; the module the reference CLI swaps at run time, ofrr/cli.py:324-336).

This is the file INTEGRATION.md section 2 tells a maintainer to add as
``ofrr/_kernels_b200.py``: a ctypes binding of libofrr_b200.so's host-buffer entry points
with the reference kernel module's exact signatures (ofrr/_kernels.pyx:23-150):

* ``gemm_mixed(a, b, compute, accumulate, out_fmt)`` -> ``ofrr_host_gemm_mixed``
* ``jacobi_eig(a, max_sweeps, tol)`` -> ``ofrr_host_jacobi_eig``
* ``dot_mixed`` / ``spmv_mixed`` stay the reference's own host kernels (off the OFRR path;
  taken from the reference's ``_kernels_py`` when this module is installed into it).

Host numpy in, host numpy out; the copies run inside each call.  It depends only on ctypes,
numpy and the shared library, not on torch.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

BACKEND_NAME = "b200"
_HERE = os.path.dirname(os.path.abspath(__file__))
_L = None
_dp = ctypes.POINTER(ctypes.c_double)


def _lib():
    global _L
    if _L is None:
        L = ctypes.CDLL(os.environ.get("OFRR_B200_LIB", os.path.join(_HERE, "libofrr_b200.so")))
        i64, ci, cd = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.ofrr_host_gemm_mixed.argtypes = [_dp, i64, i64, _dp, i64, i64, i64, i64, i64, ci, ci, ci, _dp]
        L.ofrr_host_gemm_mixed.restype = ci
        L.ofrr_host_jacobi_eig.argtypes = [_dp, i64, ci, cd, _dp, _dp, ctypes.POINTER(ci), ctypes.POINTER(cd)]
        L.ofrr_host_jacobi_eig.restype = ci
        L.ofrr_last_error.restype = ctypes.c_char_p
        _L = L
    return _L


def _check(rc: int) -> None:
    if rc:
        raise RuntimeError(_lib().ofrr_last_error().decode())


def gemm_mixed(a, b, compute, accumulate, out_fmt):
    """ofrr/_kernels.pyx:60: the mixed-precision product, F-order float64 out."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError(f"gemm_mixed dimension mismatch: {a.shape} x {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    out = np.empty((m, n), dtype=np.float64, order="F")
    _check(_lib().ofrr_host_gemm_mixed(a.ctypes.data_as(_dp), a.strides[0] // 8, a.strides[1] // 8,
                                       b.ctypes.data_as(_dp), b.strides[0] // 8, b.strides[1] // 8, m, k, n,
                                       int(compute), int(accumulate), int(out_fmt), out.ctypes.data_as(_dp)))
    return out


def jacobi_eig(a_in, max_sweeps, tol):
    """ofrr/_kernels.pyx:105: (vals, vecs, sweeps, off) of a symmetric matrix."""
    a = np.ascontiguousarray(a_in, dtype=np.float64)
    n = a.shape[0]
    vals = np.empty(n)
    vecs = np.empty((n, n))
    sw, off = ctypes.c_int(0), ctypes.c_double(0.0)
    _check(_lib().ofrr_host_jacobi_eig(a.ctypes.data_as(_dp), n, int(max_sweeps), float(tol),
                                       vals.ctypes.data_as(_dp), vecs.ctypes.data_as(_dp), ctypes.byref(sw),
                                       ctypes.byref(off)))
    return vals, vecs, sw.value, off.value


def __getattr__(name):
    # dot_mixed / spmv_mixed: the reference's own host kernels (ofrr._kernels_py)
    if name in ("dot_mixed", "spmv_mixed"):
        from ofrr import _kernels_py
        return getattr(_kernels_py, name)
    raise AttributeError(name)
