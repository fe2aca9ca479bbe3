"""Floating-point formats and precision policies (same names as the reference).

Mirrors ofrr/precision.py:20-104: ``FpFormat`` (F16/F32/F64, with eps, max_finite,
dtype), ``PrecisionPolicy`` (storage <= compute <= accumulate, ``drop_tol``), the four
presets and ``round_to``.  Extensions for the B200 path: ``FpFormat.BF16`` and
``FpFormat.FP8_E4M3`` (the tensor-core storage formats) and presets built on them.

Arithmetic semantics on the device:
* block products A.X run on tensor cores for 16/8-bit storage: products are exact and
  sums are fp32 (TMEM).  That is the reference's (storage, F32, F32) policy up to the
  summation order.  A policy whose *compute* format is F16 (``native-f16``,
  ``mixed-half``) therefore gets exact products instead of F16-rounded products in the
  MatVec; every other step (scaling, Hessenberg axpys) honours the compute format
  op for op.
* F32 / F64 storage uses CUDA-core FMA (there is no exact fp32 tensor-core path).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

try:  # bfloat16 / fp8 host dtypes
    import ml_dtypes as _mld
except Exception:  # pragma: no cover
    _mld = None


class FpFormat(enum.IntEnum):
    """Format identifiers; codes 0-2 are the reference's (ofrr/precision.py:20-25)."""

    F16 = 0
    F32 = 1
    F64 = 2
    BF16 = 3
    FP8_E4M3 = 4

    # partial "widening" order: a <= b iff every value of a is representable in b
    def _widens_to(self, other: "FpFormat") -> bool:
        return other in _WIDER_OR_EQUAL[self]

    def __le__(self, other):
        return self._widens_to(FpFormat(other))

    def __ge__(self, other):
        return FpFormat(other)._widens_to(self)

    def __lt__(self, other):
        other = FpFormat(other)
        return self != other and self._widens_to(other)

    def __gt__(self, other):
        other = FpFormat(other)
        return self != other and other._widens_to(self)

    __hash__ = enum.IntEnum.__hash__

    @property
    def eps(self) -> float:
        return _EPS[self]

    @property
    def max_finite(self) -> float:
        return _MAX_FINITE[self]

    @property
    def dtype(self) -> np.dtype:
        return _DTYPE[self]

    @property
    def itemsize(self) -> int:
        return {0: 2, 1: 4, 2: 8, 3: 2, 4: 1}[int(self)]

    @property
    def torch_dtype(self):
        import torch
        return {0: torch.float16, 1: torch.float32, 2: torch.float64, 3: torch.bfloat16,
                4: torch.float8_e4m3fn}[int(self)]

    @property
    def tensor_core(self) -> bool:
        return self in (FpFormat.F16, FpFormat.BF16, FpFormat.FP8_E4M3)


_WIDER_OR_EQUAL = {
    FpFormat.FP8_E4M3: {FpFormat.FP8_E4M3, FpFormat.F16, FpFormat.BF16, FpFormat.F32, FpFormat.F64},
    FpFormat.F16: {FpFormat.F16, FpFormat.F32, FpFormat.F64},
    FpFormat.BF16: {FpFormat.BF16, FpFormat.F32, FpFormat.F64},
    FpFormat.F32: {FpFormat.F32, FpFormat.F64},
    FpFormat.F64: {FpFormat.F64},
}
_EPS = {FpFormat.F16: 2.0**-10, FpFormat.F32: 2.0**-23, FpFormat.F64: 2.0**-52,
        FpFormat.BF16: 2.0**-7, FpFormat.FP8_E4M3: 2.0**-3}
_MAX_FINITE = {
    FpFormat.F16: 65504.0,
    FpFormat.F32: float(np.finfo(np.float32).max),
    FpFormat.F64: float(np.finfo(np.float64).max),
    FpFormat.BF16: float.fromhex("0x1.fep127"),
    FpFormat.FP8_E4M3: 448.0,
}
_DTYPE = {
    FpFormat.F16: np.dtype(np.float16),
    FpFormat.F32: np.dtype(np.float32),
    FpFormat.F64: np.dtype(np.float64),
}
if _mld is not None:
    _DTYPE[FpFormat.BF16] = np.dtype(_mld.bfloat16)
    _DTYPE[FpFormat.FP8_E4M3] = np.dtype(_mld.float8_e4m3fn)


@dataclass(frozen=True)
class PrecisionPolicy:
    """Storage/compute/accumulate triple plus column-drop tolerance
    (ofrr/precision.py:53-74)."""

    storage: FpFormat
    compute: FpFormat
    accumulate: FpFormat
    drop_tol_factor: float = 1.0
    # extension: the accuracy tier of the split products on a 16/8-bit operator -- fp64 blocks
    # (int8 Ozaki digits): 6 levels ~2^-46 of |A||x| per term, 4 levels ~2^-30 (full-f64-lite);
    # fp32 blocks on bf16 (bf16 slices): 6 -> 3 slices (24-bit block), 4 -> 2 slices (16-bit,
    # full-f32-lite).  Ladder rungs only; no effect on any other product.
    product_levels: int = 6

    def __post_init__(self):
        object.__setattr__(self, "storage", FpFormat(self.storage))
        object.__setattr__(self, "compute", FpFormat(self.compute))
        object.__setattr__(self, "accumulate", FpFormat(self.accumulate))
        if not (self.accumulate >= self.compute >= self.storage):
            raise ValueError(
                "precision policy must widen: storage <= compute <= accumulate"
            )
        if self.product_levels not in (4, 6):
            raise ValueError("product_levels must be 6 (FP64-accurate) or 4 (lite)")

    @property
    def drop_tol(self) -> float:
        return self.drop_tol_factor * self.storage.eps


NATIVE_F16 = PrecisionPolicy(FpFormat.F16, FpFormat.F16, FpFormat.F16)
MIXED_HALF = PrecisionPolicy(FpFormat.F16, FpFormat.F16, FpFormat.F32)
FULL_F32 = PrecisionPolicy(FpFormat.F32, FpFormat.F32, FpFormat.F32)
FULL_F64 = PrecisionPolicy(FpFormat.F64, FpFormat.F64, FpFormat.F64)
# extensions: tensor-core semantics (exact products, fp32 sums)
TC_F16 = PrecisionPolicy(FpFormat.F16, FpFormat.F32, FpFormat.F32)
TC_BF16 = PrecisionPolicy(FpFormat.BF16, FpFormat.F32, FpFormat.F32)
TC_FP8 = PrecisionPolicy(FpFormat.FP8_E4M3, FpFormat.F32, FpFormat.F32)
# extension: an fp64 basis whose products on a 16/8-bit operator keep ~30 bits (ladder rung)
FULL_F64_LITE = PrecisionPolicy(FpFormat.F64, FpFormat.F64, FpFormat.F64, product_levels=4)
FULL_F32_LITE = PrecisionPolicy(FpFormat.F32, FpFormat.F32, FpFormat.F32, product_levels=4)

POLICY_PRESETS = {
    "native-f16": NATIVE_F16,
    "mixed-half": MIXED_HALF,
    "full-f32": FULL_F32,
    "full-f64": FULL_F64,
    "tc-f16": TC_F16,
    "tc-bf16": TC_BF16,
    "tc-fp8": TC_FP8,
    "full-f64-lite": FULL_F64_LITE,
    "full-f32-lite": FULL_F32_LITE,
}


def round_to(x, fmt: FpFormat):
    """Round into ``fmt`` (RNE; beyond max_finite -> +-inf; subnormals kept), returned
    as float64 holding representable values (ofrr/precision.py:90-104).

    Host numpy input is rounded with numpy/ml_dtypes casts (an input-preparation
    utility); a torch CUDA tensor is rounded on the device by the library's convert
    kernel."""
    fmt = FpFormat(fmt)
    try:
        import torch
        if isinstance(x, torch.Tensor) and x.is_cuda:
            from . import ops
            return ops.round_tensor(x, fmt)
    except ImportError:  # pragma: no cover
        pass
    if fmt == FpFormat.F64:
        if np.isscalar(x):
            return float(x)
        return np.asarray(x, dtype=np.float64)
    scalar = np.isscalar(x)
    a = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        if fmt in (FpFormat.F16, FpFormat.F32):
            r = a.astype(fmt.dtype).astype(np.float64)
        elif fmt == FpFormat.BF16:
            r = a.astype(np.float32).astype(fmt.dtype).astype(np.float64)
        else:
            r = a.astype(np.float32).astype(fmt.dtype).astype(np.float64)
            big = np.abs(a) > 464.0
            r = np.where(big & np.isfinite(a), np.copysign(np.inf, a), r)
            r = np.where(np.isinf(a), a, r)
    return float(r) if scalar else r


def projection_policy(policy: PrecisionPolicy):
    """(gemm policy, output format) for the projected matrices
    (ofrr/projection.py:42-53); BF16 / FP8 storage project into FP64 (the
    "bf16 basis / fp64 Gram" configuration)."""
    if policy.storage == FpFormat.F64:
        return FULL_F64, FpFormat.F64
    if policy.storage in (FpFormat.F32, FpFormat.BF16, FpFormat.FP8_E4M3):
        return PrecisionPolicy(policy.storage, FpFormat.F64, FpFormat.F64), FpFormat.F64
    return PrecisionPolicy(policy.storage, FpFormat.F32, FpFormat.F32), FpFormat.F32
