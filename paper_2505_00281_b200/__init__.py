"""B200-native (sm_100a) OFRR: orthogonalization-free Rayleigh-Ritz eigen / partial-SVD
solver (arXiv 2505.00281), a drop-in for the reference package's OFRR path.

Public names follow the reference's ``ofrr/__init__.py:4-68`` for that path.  The
compute runs in libofrr_b200.so (hand-written tcgen05/TMA/TMEM CUDA kernels) through a
C ABI (include/ofrr_b200.h); PyTorch only holds device memory, streams and
torch.distributed.  There is no CPU fallback.
"""

from . import _lib
from .basis import BasisFactorization, BasisMethod, build_basis, hessenberg_basis, orthonormalize
from .comm import Comm
from .driver import IterConfig, RunStats, subspace_iter_eig, subspace_iter_svd
from .errors import ConvergenceError, EmptyBasisError, EmptyPencilError, OverflowDiagnostic
from .matrix import (DenseMatrix, clustered_spectrum, geometric_spectrum, sym_factors,
                     synthetic_lowrank, synthetic_symmetric, to_dense_f64)
from .precision import (FULL_F32, FULL_F64, MIXED_HALF, NATIVE_F16, POLICY_PRESETS, TC_BF16, TC_F16,
                        TC_FP8, FpFormat, PrecisionPolicy, projection_policy, round_to)
from .projection import POSITIVE_EIG_TOL, RitzSet, ofrr_eig, ofrr_svd, residual_report, rr_eig, rr_svd
from .smallsolve import EigResult, sym_def_gen_eig, sym_eig

__version__ = "0.1.0"
active_backend = "b200"


def available_backends() -> dict:
    """Name -> module map, mirroring ofrr/backend.py:25-34 (one backend: the GPU)."""
    from . import ops
    return {"b200": ops}


__all__ = [
    "active_backend", "available_backends",
    "BasisFactorization", "BasisMethod", "EmptyBasisError", "build_basis", "hessenberg_basis", "orthonormalize",
    "IterConfig", "RunStats", "subspace_iter_eig", "subspace_iter_svd",
    "DenseMatrix", "to_dense_f64", "geometric_spectrum", "clustered_spectrum", "sym_factors",
    "synthetic_symmetric", "synthetic_lowrank",
    "FULL_F32", "FULL_F64", "MIXED_HALF", "NATIVE_F16", "TC_F16", "TC_BF16", "TC_FP8", "POLICY_PRESETS",
    "FpFormat", "PrecisionPolicy", "round_to", "projection_policy",
    "EmptyPencilError", "OverflowDiagnostic", "RitzSet", "ofrr_eig", "ofrr_svd", "residual_report", "rr_eig", "rr_svd",
    "POSITIVE_EIG_TOL", "ConvergenceError", "EigResult", "sym_def_gen_eig", "sym_eig", "Comm",
]
