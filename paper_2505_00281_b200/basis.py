"""Basis builders on the device: the Hessenberg process (hess-l / hess-r, the basis OFRR
uses in place of QR) and the Gram-Schmidt family (mgs-l, mgs-r, cgs, cgs2 -- the QR
comparators of SURVEY.md 8(f) rank 4, csrc/gs.cu).

Same names as ofrr/basis.py:23-148.  The Krylov builders (arnoldi-mgs, krylov-hess) belong
to the reference's sparse Krylov solver and are rejected with ValueError (no CPU fallback).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .errors import EmptyBasisError
from .matrix import DenseMatrix
from .precision import PrecisionPolicy


class BasisMethod(enum.Enum):
    """ofrr/basis.py:23-31 (same values)."""
    MGS_LEFT = "mgs-l"
    MGS_RIGHT = "mgs-r"
    CGS = "cgs"
    CGS2 = "cgs2"
    HESS_LEFT = "hess-l"
    HESS_RIGHT = "hess-r"
    ARNOLDI_MGS = "arnoldi-mgs"
    KRYLOV_HESS = "krylov-hess"


GRAM_SCHMIDT_METHODS = {BasisMethod.MGS_LEFT, BasisMethod.MGS_RIGHT, BasisMethod.CGS, BasisMethod.CGS2}
HESSENBERG_METHODS = {BasisMethod.HESS_LEFT, BasisMethod.HESS_RIGHT}
KRYLOV_METHODS = {BasisMethod.ARNOLDI_MGS, BasisMethod.KRYLOV_HESS}


@dataclass(frozen=True)
class BasisFactorization:
    """ofrr/basis.py:45-51.  ``q`` holds the kept columns only (device resident)."""
    q: DenseMatrix
    pivots: np.ndarray
    kept: np.ndarray
    method: BasisMethod
    policy: PrecisionPolicy


def build_basis(x: DenseMatrix, method: BasisMethod, policy: PrecisionPolicy) -> BasisFactorization:
    """ofrr/basis.py:54-62 dispatch."""
    if method in GRAM_SCHMIDT_METHODS:
        return orthonormalize(x, method, policy)
    if method in HESSENBERG_METHODS:
        return hessenberg_basis(x, "left" if method is BasisMethod.HESS_LEFT else "right", policy)
    raise ValueError(f"{method} is not a block basis method")


def orthonormalize(x: DenseMatrix, method: BasisMethod, policy: PrecisionPolicy,
                   reorth: bool = True) -> BasisFactorization:
    """Gram-Schmidt family under an explicit precision policy (ofrr/basis.py:65-116), on the
    device (K3g, csrc/gs.cu): drop rule nrm < drop_tol * pre, MGS-L's single
    re-orthogonalization, CGS2's two sweeps, MGS-R's right-looking sweep."""
    from . import ops
    if method not in GRAM_SCHMIDT_METHODS:
        raise ValueError(f"{method} is not a Gram-Schmidt method")
    if x.cols == 0:
        raise EmptyBasisError("no input columns")
    X = x.device_block(policy.storage)
    h = ops.orthonormalize(X, method.value, policy.storage, policy.compute, policy.accumulate, policy.drop_tol,
                           reorth=reorth)
    nk = int(h.n_kept.item())
    if nk == 0:
        raise EmptyBasisError("all columns dropped during orthonormalization")
    q = DenseMatrix.from_block(h.Q.narrow(nk))
    return BasisFactorization(q, np.zeros(0, dtype=np.int64), h.kept[: x.cols].cpu().numpy().astype(bool), method,
                              policy)


def hessenberg_basis(x: DenseMatrix, layout: str, policy: PrecisionPolicy) -> BasisFactorization:
    """Inner-product-free basis by pivot scaling and elimination (ofrr/basis.py:151-196).

    Both layouts run the identical update sequence (the reference pins left == right
    bitwise, tests/test_basis.py:92-98), so one device kernel (K3) serves both."""
    from . import ops
    if layout not in ("left", "right"):
        raise ValueError("layout must be 'left' or 'right'")
    if x.cols == 0:
        raise EmptyBasisError("no input columns")
    X = x.device_block(policy.storage)
    h = ops.hessenberg(X, policy.storage, policy.compute, policy.drop_tol)
    nk = int(h.n_kept.item())
    if nk == 0:
        raise EmptyBasisError("all columns skipped in Hessenberg process")
    method = BasisMethod.HESS_LEFT if layout == "left" else BasisMethod.HESS_RIGHT
    q = DenseMatrix.from_block(h.Q.narrow(nk))
    return BasisFactorization(q, h.pivots[:nk].cpu().numpy().astype(np.int64),
                              h.kept[: x.cols].cpu().numpy().astype(bool), method, policy)
