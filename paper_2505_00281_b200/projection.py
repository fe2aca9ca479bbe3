"""Orthogonalization-free Rayleigh-Ritz projections on the device + FP64 residuals.

Same names and contracts as ofrr/projection.py:21-158 (``ofrr_eig``, ``ofrr_svd``,
``residual_report``, ``RitzSet``, ``projection_policy``, the error classes), plus the
classical ``rr_eig`` / ``rr_svd`` comparators (ofrr/projection.py:64-96) for bases from the
Gram-Schmidt builders.

Per ofrr_eig call: W = A U (K1, tensor cores for 16/8-bit storage), the projected
matrices B = U^T W and M = U^T U (K4, fp64 sums), the symmetric-definite pencil solve
with the independence safeguard (K5), and the Ritz vectors U Y (K6) -- all on the GPU;
the host only reads the handful of status words.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from .errors import EmptyPencilError, OverflowDiagnostic, ConvergenceError
from .matrix import DenseMatrix, to_dense_f64
from .precision import FpFormat, PrecisionPolicy, projection_policy

POSITIVE_EIG_TOL = 1e-8  # ofrr/projection.py:21


@dataclass(frozen=True)
class RitzSet:
    """ofrr/projection.py:32-39.  ``vectors`` / ``right_vectors`` are FP64 DenseMatrix
    objects that live on the device; ``.data`` copies them to the host on first use."""
    values: np.ndarray
    vectors: DenseMatrix
    kind: str
    right_vectors: Optional[DenseMatrix] = None
    residuals: Optional[np.ndarray] = None
    diagnostics: str = ""


def _status(st_cpu, eig_slot: int, flag_slot: int, what: str):
    fl = int(st_cpu[flag_slot])
    if fl & 1:
        raise OverflowDiagnostic(f"non-finite entries in {what}")
    es = int(st_cpu[eig_slot])
    if es == 6:
        raise ConvergenceError("Jacobi eigendecomposition did not converge", float("nan"))
    if es == 5:
        raise EmptyPencilError("mass matrix retained no eigenvalues")


def ofrr_eig(a: DenseMatrix, u: DenseMatrix, policy: PrecisionPolicy) -> RitzSet:
    """ofrr/projection.py:75-87: solve the pencil (U'AU, U'U) on the device."""
    import torch
    from . import ops
    A = a.device_operator(policy.storage)
    U = u.device_block(policy.storage)
    k = U.k
    _, out_fmt = projection_policy(policy)
    st = torch.zeros(8, dtype=torch.int32, device=A.device)
    W = ops.new_block(A.rows, k, policy.storage, A.device)
    ops.gemm_av(A, U, W, flags=st[0:1])
    B, M = ops.gram(U, W, out_fmt, flags=st[1:2])
    eig = ops.sym_def_gen_eig(B, M, k)
    st[2:3].copy_(eig.status)
    st[3:4].copy_(eig.n_out)
    U64, _ = ops.ritz(U, eig.vectors, k, eig.n_out, k, 1.0, want64=True)
    s = st.cpu().numpy()
    if s[0] & 1:
        raise OverflowDiagnostic("non-finite entries in projected matrix")
    _status(s, 2, 1, "projected matrix")
    r = int(s[3])
    if r == 0:
        raise EmptyPencilError("mass matrix retained no eigenvalues")
    vals = eig.values[:r].cpu().numpy()
    return RitzSet(vals, DenseMatrix.from_block(U64.narrow(r)), "eig")


def rr_eig(a: DenseMatrix, q: DenseMatrix, policy: PrecisionPolicy) -> RitzSet:
    """ofrr/projection.py:64-72: classical Rayleigh-Ritz, eig of Q'AQ (Q intended-orthonormal,
    deliberately unchecked) and the vectors Q Y in FP64."""
    import torch
    from . import ops
    A = a.device_operator(policy.storage)
    Q = q.device_block(policy.storage)
    k = Q.k
    _, out_fmt = projection_policy(policy)
    st = torch.zeros(8, dtype=torch.int32, device=A.device)
    W = ops.new_block(A.rows, k, policy.storage, A.device)
    ops.gemm_av(A, Q, W, flags=st[0:1])
    B, _ = ops.gram(Q, W, out_fmt, flags=st[1:2], want_m=False)
    eig = ops.sym_eig(B, k)
    st[2:3].copy_(eig.status)
    U64, _ = ops.ritz(Q, eig.vectors, k, None, k, 1.0, want64=True)
    s = st.cpu().numpy()
    if s[0] & 1:
        raise OverflowDiagnostic("non-finite entries in projected matrix")
    _status(s, 2, 1, "projected matrix")
    return RitzSet(eig.values[:k].cpu().numpy(), DenseMatrix.from_block(U64.narrow(k)), "eig")


def rr_svd(a: DenseMatrix, u: DenseMatrix, v: DenseMatrix, policy: PrecisionPolicy) -> RitzSet:
    """ofrr/projection.py:90-96: classical two-sided Rayleigh-Ritz, the SVD of U'AV -- taken
    from the symmetric eigenproblem of [[0, U'AV], [(U'AV)', 0]] (the ofrr_svd block pencil
    with identity mass matrices), singular vectors sqrt(2)-scaled."""
    from . import driver
    eng = driver.SvdEngine.single(a, policy, policy)
    U = u.device_block(policy.storage)
    V = v.device_block(policy.storage)
    return eng.project(U, V, want64=True, classical=True)[0]


def ofrr_svd(a: DenseMatrix, u: DenseMatrix, v: DenseMatrix, policy: PrecisionPolicy) -> RitzSet:
    """ofrr/projection.py:99-133: block pencil [[0, U'AV], [(U'AV)', 0]] vs
    diag(U'U, V'V); the eigenvalues above POSITIVE_EIG_TOL of the largest are the
    singular values, sqrt(2)-scaled eigenvector blocks give the singular vectors."""
    from . import driver
    eng = driver.SvdEngine.single(a, policy, policy)
    U = u.device_block(policy.storage)
    V = v.device_block(policy.storage)
    return eng.project(U, V, want64=True)[0]


def residual_report(a: DenseMatrix, rs: RitzSet) -> RitzSet:
    """ofrr/projection.py:136-158: FP64 relative residuals from A as stored."""
    import torch
    from . import ops
    r = int(len(rs.values))
    if r == 0:
        return replace(rs, residuals=np.zeros(0))
    A = a.residual_operator(a.fmt)
    dev = A.device
    vals = torch.as_tensor(np.asarray(rs.values, dtype=np.float64), device=dev)
    V = rs.vectors.device_block(FpFormat.F64)
    if rs.kind == "eig":
        res = ops.residual_eig(A, V, vals, None, r)
    else:
        U = rs.vectors.device_block(FpFormat.F64)
        Vr = rs.right_vectors.device_block(FpFormat.F64)
        At = a.residual_operator_t(a.fmt)
        res = torch.zeros(r, dtype=torch.float64, device=dev)
        ops.residual_pair(A, False, Vr, U, vals, None, r, res, accumulate_max=False)
        ops.residual_pair(At, False, U, Vr, vals, None, r, res, accumulate_max=True)
    return replace(rs, residuals=res[:r].cpu().numpy())


__all__ = ["RitzSet", "ofrr_eig", "ofrr_svd", "rr_eig", "rr_svd", "residual_report", "projection_policy", "POSITIVE_EIG_TOL",
           "OverflowDiagnostic", "EmptyPencilError", "to_dense_f64"]
