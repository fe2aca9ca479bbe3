"""CPU oracle for the OFRR hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the thing measured or shipped: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import it.  The product package (``paper_2505_00281_b200``) never imports
anything under ``oracle/``.

It restates, in numpy + the plain-C kernels of ``ofrr_oracle.c``, the reference
algorithm of /root/reference/pkg/src/ofrr (cited as ``ofrr/<file>:<line>``):

* round_to / scale_columns_inf / axpy          ofrr/precision.py:90-104, 159-180
* mixed_gemm (sequential mixed dot per entry)  ofrr/precision.py:122-135, ofrr/_kernels.pyx:34-84
* hessenberg_basis (+ pivot rule)              ofrr/basis.py:151-204
* sym_eig / _sorted_desc / sym_def_gen_eig     ofrr/smallsolve.py:34-88, ofrr/_kernels.pyx:105-161
* projection_policy / ofrr_eig / ofrr_svd      ofrr/projection.py:42-133
* residual_report                              ofrr/projection.py:136-158
* subspace_iter_eig / subspace_iter_svd        ofrr/driver.py:84-111, 141-173

Extensions (absent from the reference, so pinned only against this restatement):
format codes BF16=3 and FP8_E4M3=4, and the projection rule for them (FP64 Grams,
as BASELINE.json's "bf16 basis / fp64 Gram" configuration states).

Pinning: tests/test_oracle_golden.py checks every function here against golden
vectors produced by importing the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

F16, F32, F64, BF16, FP8E4M3 = 0, 1, 2, 3, 4
EPS = {F16: 2.0**-10, F32: 2.0**-23, F64: 2.0**-52, BF16: 2.0**-7, FP8E4M3: 2.0**-3}
POSITIVE_EIG_TOL = 1e-8          # ofrr/projection.py:21
MAX_SWEEPS = 30                  # ofrr/smallsolve.py:17

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libofrr_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile ofrr_oracle.c into oracle/libofrr_oracle.so (gcc, no GPU needed)."""
    src = os.path.join(_HERE, "ofrr_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_long)
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_round.argtypes = [dp, dp, ctypes.c_long, ctypes.c_int]
        L.oracle_dot_mixed.argtypes = [dp, dp, ctypes.c_long, ctypes.c_int, ctypes.c_int]
        L.oracle_dot_mixed.restype = ctypes.c_double
        L.oracle_gemm_mixed.argtypes = [dp, ctypes.c_long, ctypes.c_long, dp, ctypes.c_long,
                                        ctypes.c_long, ctypes.c_long, ctypes.c_long,
                                        ctypes.c_long, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, dp]
        L.oracle_jacobi_eig.argtypes = [dp, dp, ctypes.c_long, ctypes.c_int, ctypes.c_double, dp]
        L.oracle_jacobi_eig.restype = ctypes.c_int
        L.oracle_hessenberg.argtypes = [dp, ctypes.c_long, ctypes.c_long, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_double, dp, lp, ip]
        L.oracle_hessenberg.restype = ctypes.c_long
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ----------------------------------------------------------------------------------
# precision (ofrr/precision.py)
# ----------------------------------------------------------------------------------
@dataclass(frozen=True)
class Pol:
    """PrecisionPolicy restated with integer format codes (ofrr/precision.py:53-74)."""
    storage: int
    compute: int
    accumulate: int
    drop_tol_factor: float = 1.0

    @property
    def drop_tol(self) -> float:
        return self.drop_tol_factor * EPS[self.storage]


NATIVE_F16 = Pol(F16, F16, F16)      # ofrr/precision.py:77
MIXED_HALF = Pol(F16, F16, F32)      # ofrr/precision.py:78
FULL_F32 = Pol(F32, F32, F32)        # ofrr/precision.py:79
FULL_F64 = Pol(F64, F64, F64)        # ofrr/precision.py:80
TC_F16 = Pol(F16, F32, F32)          # tensor-core semantics: exact products, fp32 sums
TC_BF16 = Pol(BF16, F32, F32)        # extension
TC_FP8 = Pol(FP8E4M3, F32, F32)      # extension


def as_pol(p) -> Pol:
    if isinstance(p, Pol):
        return p
    return Pol(int(p.storage), int(p.compute), int(p.accumulate),
               float(getattr(p, "drop_tol_factor", 1.0)))


def round_to(x, fmt: int):
    """ofrr/precision.py:90-104 (RNE, overflow -> inf, subnormals kept)."""
    x = np.asarray(x, dtype=np.float64)
    if fmt == F64:
        return x.copy()
    xc = np.ascontiguousarray(x)
    out = np.empty_like(xc)
    lib().oracle_round(_dp(xc), _dp(out), xc.size, int(fmt))
    return out.reshape(x.shape)


def mixed_dot(x, y, compute: int, accumulate: int) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return lib().oracle_dot_mixed(_dp(x), _dp(y), x.size, compute, accumulate)


def mixed_gemm(a, b, compute: int, accumulate: int, out_fmt: int) -> np.ndarray:
    """ofrr/precision.py:122-135 -> ofrr/_kernels.pyx:60-84; F-order float64 out."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError(f"mixed_gemm dimension mismatch: {a.shape} x {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    out = np.zeros((m, n), dtype=np.float64, order="F")
    if m == 0 or n == 0:
        return out
    ac = a if a.flags.c_contiguous or a.flags.f_contiguous else np.ascontiguousarray(a)
    bc = b if b.flags.c_contiguous or b.flags.f_contiguous else np.ascontiguousarray(b)
    ars, acs = ac.strides[0] // 8, ac.strides[1] // 8
    brs, bcs = bc.strides[0] // 8, bc.strides[1] // 8
    lib().oracle_gemm_mixed(_dp(ac), ars, acs, _dp(bc), brs, bcs, m, k, n,
                            int(compute), int(accumulate), int(out_fmt), _dp(out))
    return out


def apply_dense(a, x, pol: Pol, transpose: bool = False):
    """ofrr/matrix.py:242-254 (dense branch)."""
    m = a.T if transpose else a
    return mixed_gemm(m, x, pol.compute, pol.accumulate, pol.storage)


def scale_columns_inf(x, pol: Pol):
    """ofrr/precision.py:159-169."""
    x = np.asarray(x, dtype=np.float64)
    out = x.copy(order="F")
    for j in range(x.shape[1]):
        mx = np.max(np.abs(x[:, j])) if x.shape[0] else 0.0
        if mx != 0.0:
            out[:, j] = round_to(round_to(x[:, j] / mx, pol.compute), pol.storage)
    return out


# ----------------------------------------------------------------------------------
# basis (ofrr/basis.py)
# ----------------------------------------------------------------------------------
class EmptyBasisError(RuntimeError):
    pass


def hessenberg_basis(x, pol: Pol):
    """ofrr/basis.py:151-196 -> (q n x k' F-order, pivots int64[k'], kept bool[k])."""
    xw = np.array(x, dtype=np.float64, order="F")
    n, k = xw.shape
    if k == 0:
        raise EmptyBasisError("no input columns")
    q = np.zeros((n, k), dtype=np.float64, order="F")
    piv = np.zeros(k, dtype=np.int64)
    kept = np.zeros(k, dtype=np.int32)
    nk = lib().oracle_hessenberg(_dp(xw), n, k, pol.storage, pol.compute, float(pol.drop_tol),
                                 _dp(q), piv.ctypes.data_as(ctypes.POINTER(ctypes.c_long)),
                                 kept.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    if nk == 0:
        raise EmptyBasisError("all columns skipped in Hessenberg process")
    return np.asfortranarray(q[:, :nk]), piv[:nk].copy(), kept.astype(bool)


def safe_norm2(x, pol: Pol) -> float:
    """ofrr/precision.py:138-156 (overflow-safe 2-norm under the policy)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    m = float(np.max(np.abs(x)))
    if m == 0.0:
        return 0.0
    u = round_to(x / m, pol.compute)
    ss = mixed_dot(u, u, pol.compute, pol.accumulate)
    r = float(round_to(np.sqrt(ss), pol.compute))
    return float(round_to(m * r, pol.compute))


def axpy(y, alpha, x, pol: Pol):
    """ofrr/precision.py:172-180: y - c(alpha) * x with compute-format roundings, stored."""
    c = pol.compute
    t = round_to(float(round_to(alpha, c)) * np.asarray(x, dtype=np.float64), c)
    return round_to(round_to(np.asarray(y, dtype=np.float64) - t, c), pol.storage)


REORTH_THRESHOLD = np.sqrt(2.0) / 2.0   # ofrr/basis.py:20


def orthonormalize(x, method: str, pol: Pol, reorth: bool = True):
    """ofrr/basis.py:65-116 (+ _mgs_project :119-123, _cgs_project :126-130, _mgs_right
    :133-148) -> (q n x k' F-order, kept bool[k]).  Products / differences are exact in fp64
    before the compute-format rounding (storage <= compute), so the numpy formulation
    rounds exactly like the reference's typed arrays."""
    a = np.array(x, dtype=np.float64, order="F")
    n, k = a.shape
    if k == 0:
        raise EmptyBasisError("no input columns")
    kept = np.zeros(k, dtype=bool)
    cols = []
    if method == "mgs-r":
        pre = np.array([safe_norm2(a[:, j], pol) for j in range(k)])
        for j in range(k):
            v = a[:, j]
            nrm = safe_norm2(v, pol)
            if nrm < pol.drop_tol * pre[j] or nrm == 0.0:
                continue
            q = round_to(round_to(v / nrm, pol.compute), pol.storage)
            kept[j] = True
            cols.append(q)
            for i in range(j + 1, k):
                h = mixed_dot(q, a[:, i], pol.compute, pol.accumulate)
                a[:, i] = axpy(a[:, i], h, q, pol)
    else:
        def mgs(v):
            for qi in cols:
                v = axpy(v, mixed_dot(qi, v, pol.compute, pol.accumulate), qi, pol)
            return v, safe_norm2(v, pol)

        def cgs(v):
            coeffs = [mixed_dot(qi, v, pol.compute, pol.accumulate) for qi in cols]
            for h, qi in zip(coeffs, cols):
                v = axpy(v, h, qi, pol)
            return v

        for j in range(k):
            v = a[:, j].copy()
            pre = safe_norm2(v, pol)
            if method == "mgs-l":
                v, nrm = mgs(v)
                if reorth and nrm < REORTH_THRESHOLD * pre:
                    v, nrm = mgs(v)
            elif method in ("cgs", "cgs2"):
                v = cgs(v)
                nrm = safe_norm2(v, pol)
                if method == "cgs2":
                    n1 = nrm
                    v = cgs(v)
                    nrm = safe_norm2(v, pol)
                    if nrm < REORTH_THRESHOLD * n1:
                        continue
            else:
                raise ValueError(f"{method} is not a Gram-Schmidt method")
            if nrm < pol.drop_tol * pre or nrm == 0.0:
                continue
            kept[j] = True
            cols.append(round_to(round_to(v / nrm, pol.compute), pol.storage))
    if not cols:
        raise EmptyBasisError("all columns dropped during orthonormalization")
    return np.asfortranarray(np.column_stack(cols)), kept


# ----------------------------------------------------------------------------------
# small solves (ofrr/smallsolve.py)
# ----------------------------------------------------------------------------------
class ConvergenceError(RuntimeError):
    pass


def jacobi_eig(a, max_sweeps=MAX_SWEEPS, tol=0.0):
    a = np.array(a, dtype=np.float64, order="C")
    n = a.shape[0]
    v = np.zeros((n, n), dtype=np.float64)
    off = np.zeros(1)
    sweeps = lib().oracle_jacobi_eig(_dp(a), _dp(v), n, int(max_sweeps), float(tol), _dp(off))
    return np.diag(a).copy(), v, sweeps, float(off[0])


def _sorted_desc(vals, vecs):
    """ofrr/smallsolve.py:52-61."""
    order = np.argsort(-vals, kind="stable")
    vals = vals[order]
    vecs = vecs[:, order]
    for j in range(vecs.shape[1]):
        i = int(np.argmax(np.abs(vecs[:, j])))
        if vecs[i, j] < 0:
            vecs[:, j] = -vecs[:, j]
    return vals, vecs


def sym_eig(s):
    """ofrr/smallsolve.py:34-49."""
    s = np.asarray(s, dtype=np.float64)
    s = (s + s.T) / 2.0
    norm = float(np.linalg.norm(s))
    if s.shape[0] == 0:
        return np.zeros(0), np.zeros((0, 0))
    tol = 1e-14 * norm
    vals, vecs, _, off = jacobi_eig(s, MAX_SWEEPS, tol)
    if off > tol and norm > 0.0:
        raise ConvergenceError(f"Jacobi eigendecomposition did not converge ({off:.3e})")
    return _sorted_desc(vals, vecs)


def sym_def_gen_eig(b, m):
    """ofrr/smallsolve.py:64-88 (whitening + k*eps*mu_max independence safeguard)."""
    b = np.asarray(b, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    k = m.shape[0]
    mv, mvec = sym_eig(m)
    mu_max = mv[0] if k else 0.0
    if k == 0 or mu_max <= 0.0:
        return np.zeros(0), np.zeros((k, 0))
    keep = mv > k * np.finfo(np.float64).eps * mu_max
    p = mvec[:, keep]
    d = mv[keep]
    if p.shape[1] == 0:
        return np.zeros(0), np.zeros((k, 0))
    dis = 1.0 / np.sqrt(d)
    t = (dis[:, None] * (p.T @ b @ p)) * dis[None, :]
    tv, tvec = sym_eig(t)
    y = p @ (dis[:, None] * tvec)
    return _sorted_desc(tv, y)


# ----------------------------------------------------------------------------------
# projections (ofrr/projection.py)
# ----------------------------------------------------------------------------------
class OverflowDiagnostic(RuntimeError):
    pass


class EmptyPencilError(RuntimeError):
    pass


def projection_policy(pol: Pol):
    """ofrr/projection.py:42-53, extended: BF16 / FP8 storage -> FP64 Grams."""
    if pol.storage == F64:
        return F64, F64, F64
    if pol.storage in (F32, BF16, FP8E4M3):
        return F64, F64, F64
    return F32, F32, F32


def _project(u, w, pol: Pol):
    """ofrr/projection.py:56-61."""
    c, a, o = projection_policy(pol)
    b = mixed_gemm(np.asarray(u).T, w, c, a, o)
    if not np.all(np.isfinite(b)):
        raise OverflowDiagnostic("non-finite entries in projected matrix")
    return b


@dataclass
class Ritz:
    values: np.ndarray
    vectors: np.ndarray
    kind: str
    right_vectors: Optional[np.ndarray] = None
    residuals: Optional[np.ndarray] = None
    diagnostics: str = ""


def rr_eig(a, q, pol: Pol) -> Ritz:
    """ofrr/projection.py:64-72: eig of Q'AQ, vectors Q Y in FP64."""
    w = apply_dense(a, q, pol)
    b = _project(q, w, pol)
    b = (b + b.T) / 2.0
    vals, vecs = sym_eig(b)
    return Ritz(vals, np.asarray(q) @ vecs, "eig")


def ofrr_eig(a, u, pol: Pol) -> Ritz:
    """ofrr/projection.py:75-87."""
    w = apply_dense(a, u, pol)
    b = _project(u, w, pol)
    m = _project(u, u, pol)
    b = (b + b.T) / 2.0
    m = (m + m.T) / 2.0
    vals, vecs = sym_def_gen_eig(b, m)
    if vals.size == 0:
        raise EmptyPencilError("mass matrix retained no eigenvalues")
    return Ritz(vals, np.asfortranarray(u @ vecs), "eig")


def ofrr_svd(a, u, v, pol: Pol) -> Ritz:
    """ofrr/projection.py:99-133."""
    k1, k2 = u.shape[1], v.shape[1]
    w = apply_dense(a, v, pol)
    g = _project(u, w, pol)
    mu = _project(u, u, pol)
    mvv = _project(v, v, pol)
    bmat = np.zeros((k1 + k2, k1 + k2))
    bmat[:k1, k1:] = g
    bmat[k1:, :k1] = g.T
    mmat = np.zeros((k1 + k2, k1 + k2))
    mmat[:k1, :k1] = (mu + mu.T) / 2.0
    mmat[k1:, k1:] = (mvv + mvv.T) / 2.0
    vals, vecs = sym_def_gen_eig(bmat, mmat)
    if vals.size == 0:
        raise EmptyPencilError("mass matrix retained no eigenvalues")
    smax = float(np.max(vals))
    pos = vals > POSITIVE_EIG_TOL * smax if smax > 0 else vals > 0
    sig = vals[pos]
    y = vecs[:k1, pos]
    z = vecs[k1:, pos]
    diag = ""
    if sig.size < min(k1, k2):
        diag = f"{sig.size} positive eigenvalues (pencil admits {min(k1, k2)})"
    return Ritz(sig, np.asfortranarray(np.sqrt(2.0) * (u @ y)), "svd",
                right_vectors=np.asfortranarray(np.sqrt(2.0) * (v @ z)), diagnostics=diag)


def residual_report(a, rs: Ritz) -> Ritz:
    """ofrr/projection.py:136-158 (FP64 from A as stored)."""
    ad = np.asarray(a, dtype=np.float64)
    vals = rs.values
    res = np.empty_like(vals)
    if rs.kind == "eig":
        av = ad @ rs.vectors
        for i, lam in enumerate(vals):
            res[i] = np.inf if lam == 0.0 else \
                np.linalg.norm(av[:, i] - lam * rs.vectors[:, i]) / abs(lam)
    else:
        av = ad @ rs.right_vectors
        atu = ad.T @ rs.vectors
        for i, sig in enumerate(vals):
            if sig == 0.0:
                res[i] = np.inf
                continue
            r1 = np.linalg.norm(av[:, i] - sig * rs.vectors[:, i])
            r2 = np.linalg.norm(atu[:, i] - sig * rs.right_vectors[:, i])
            res[i] = max(r1, r2) / sig
    rs.residuals = res
    return rs


# ----------------------------------------------------------------------------------
# drivers (ofrr/driver.py)
# ----------------------------------------------------------------------------------
def start_block(n: int, k: int, seed: int, storage: int) -> np.ndarray:
    """ofrr/driver.py:97-99: PCG64(seed) U(0,1), rounded to the MatVec storage."""
    rng = np.random.default_rng(seed)
    return round_to(np.asfortranarray(rng.random((n, k))), storage)


def _check_finite(x, stage):
    if not np.all(np.isfinite(x)):
        raise OverflowDiagnostic(f"non-finite entries after {stage}")


def subspace_iter_eig(a, k, m=1, iters=1, pol=TC_BF16, mv_pol=None, seed=0,
                      top=None, tol=None, history=None, method="hess-l", projection="ofrr") -> Ritz:
    """ofrr/driver.py:84-111 with hess-l/hess-r + ofrr.

    ``top``/``tol`` add the time-to-tolerance stop: after each
    outer iteration the FP64 residuals of the leading ``top`` pairs are checked and
    the loop stops once their max is below ``tol`` (``m`` is then the cap).
    ``history`` (a list) receives (iteration, max residual over top) tuples."""
    pol = as_pol(pol)
    mv = as_pol(mv_pol) if mv_pol is not None else pol
    n = a.shape[0]
    if k > n:
        raise ValueError("k exceeds the operator dimension")
    x = start_block(n, k, seed, mv.storage)
    rs = None
    for it in range(m):
        for _ in range(iters):
            x = apply_dense(a, x, mv)
            _check_finite(x, "MatVec")
            x = scale_columns_inf(x, mv)
        q = hessenberg_basis(x, pol)[0] if method in ("hess-l", "hess-r") else orthonormalize(x, method, pol)[0]
        rs = rr_eig(a, q, pol) if projection == "rr" else ofrr_eig(a, q, pol)
        x = round_to(np.asfortranarray(rs.vectors), mv.storage)
        _check_finite(x, "projection")
        if tol is not None:
            t = top or len(rs.values)
            r = residual_report(a, Ritz(rs.values[:t], rs.vectors[:, :t], "eig")).residuals
            worst = float(np.max(r)) if len(r) >= t else float("inf")
            if history is not None:
                history.append((it + 1, worst))
            if worst < tol:
                break
    return residual_report(a, rs)


def subspace_iter_svd(a, k, m=1, iters=1, pol=TC_BF16, mv_pol=None, seed=0) -> Ritz:
    """ofrr/driver.py:141-173 with hess-l/hess-r + ofrr."""
    pol = as_pol(pol)
    mv = as_pol(mv_pol) if mv_pol is not None else pol
    n1, n2 = a.shape
    if k > min(n1, n2):
        raise ValueError("k exceeds min(n1, n2)")
    v = start_block(n2, k, seed, mv.storage)
    rs = None
    for _ in range(m):
        u = v
        for _ in range(iters):
            u = apply_dense(a, v, mv)
            _check_finite(u, "MatVec")
            u = scale_columns_inf(u, mv)
            v = apply_dense(a, u, mv, transpose=True)
            _check_finite(v, "MatVec")
            v = scale_columns_inf(v, mv)
        qu, _, _ = hessenberg_basis(u, pol)
        qv, _, _ = hessenberg_basis(v, pol)
        rs = ofrr_svd(a, qu, qv, pol)
        v = round_to(np.asfortranarray(rs.right_vectors), mv.storage)
        _check_finite(v, "projection")
    return residual_report(a, rs)


# ----------------------------------------------------------------------------------
# synthetic inputs: generated in FP64, rounded once to storage
# ----------------------------------------------------------------------------------
def sym_from_factors(n, hadamard, c, s, Wf, Mf, fmt: int = F64) -> np.ndarray:
    """Host evaluation of the synthetic generator (K8) in the device's exact operation
    order: acc = base; for each s: acc += W[i,s]*M[j,s]; acc += M[i,s]*W[j,s]; then one
    rounding to ``fmt``.  Returns the n x n matrix (row i = A[i, :])."""
    i = np.arange(n)
    if hadamard:
        base = (s[:, None] * s[None, :]) * c[i[:, None] ^ i[None, :]]
    else:
        base = np.diag(c).astype(np.float64)
    acc = base.copy()
    for t in range(Wf.shape[1]):
        acc = acc + Wf[:, t][:, None] * Mf[:, t][None, :]
        acc = acc + Mf[:, t][:, None] * Wf[:, t][None, :]
    return round_to(acc, fmt)


def geometric_symmetric(n: int, top: int, k: int, seed: int, fmt: int = F64,
                        rho: Optional[float] = None):
    """A = Q diag(lambda) Q^T, lambda_i = rho^i (rho = 0.1^(1/(k-top+1)) by default),
    Q a seeded Haar orthogonal matrix (QR of a Gaussian).  Returns (A, lambda)."""
    if rho is None:
        rho = 0.1 ** (1.0 / (k - top + 1))
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    q, r = np.linalg.qr(g)
    q = q * np.sign(np.diag(r))[None, :]
    lam = rho ** np.arange(n, dtype=np.float64)
    a = (q * lam[None, :]) @ q.T
    a = (a + a.T) / 2.0
    return round_to(a, fmt), lam
