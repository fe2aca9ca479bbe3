"""CPU-only checks of the boundary and the host logic (no GPU needed):
the C ABI library loads and exports every symbol include/ofrr_b200.h declares; the
reference's option names / validation / presets / known answers hold for the package."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "ofrr_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ofrr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes
    from paper_2505_00281_b200 import _lib
    L = _lib.load()                      # loads without a GPU (no compute calls here)
    syms = _header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # every header symbol has a ctypes signature in the binding (and vice versa)
    assert set(syms) - {"ofrr_debug_k5_profile"} <= set(_lib.EXPORTED) | {"ofrr_debug_k5_profile"}
    assert L.ofrr_abi_version() == 1
    assert isinstance(L.ofrr_last_error(), (bytes, type(None)))


def test_status_codes_map_to_reference_exceptions():
    import paper_2505_00281_b200 as p
    from paper_2505_00281_b200 import _lib
    for code, exc in ((_lib.ERR_INVALID, ValueError), (_lib.ERR_OVERFLOW, p.OverflowDiagnostic),
                      (_lib.ERR_EMPTY_BASIS, p.EmptyBasisError), (_lib.ERR_EMPTY_PENCIL, p.EmptyPencilError),
                      (_lib.ERR_CONVERGENCE, p.ConvergenceError)):
        with pytest.raises(exc):
            _lib.check(code, "x")
    _lib.check(_lib.OK, "x")


def test_formats_and_policies():
    """tests/test_precision.py:11-55 known answers, plus the bf16/fp8 extensions."""
    import paper_2505_00281_b200 as p
    F = p.FpFormat
    assert F.F16.eps == 2.0**-10 and F.F32.eps == 2.0**-23 and F.F64.eps == 2.0**-52
    assert F.BF16.eps == 2.0**-7 and F.FP8_E4M3.eps == 2.0**-3
    assert F.F16.max_finite == 65504.0 and F.FP8_E4M3.max_finite == 448.0
    assert F.F16 < F.F32 < F.F64
    assert not (F.BF16 <= F.F16) and not (F.F16 <= F.BF16)      # incomparable
    assert F.FP8_E4M3 <= F.BF16 <= F.F32
    for pol in (p.NATIVE_F16, p.MIXED_HALF, p.FULL_F32, p.FULL_F64, p.TC_BF16, p.TC_F16, p.TC_FP8):
        assert pol.accumulate >= pol.compute >= pol.storage
    with pytest.raises(ValueError):
        p.PrecisionPolicy(F.F32, F.F16, F.F16)
    with pytest.raises(ValueError):
        p.PrecisionPolicy(F.BF16, F.F16, F.F32)
    assert p.NATIVE_F16.drop_tol == 2.0**-10
    assert p.PrecisionPolicy(F.F16, F.F16, F.F16, drop_tol_factor=4.0).drop_tol == 2.0**-8
    assert set(["native-f16", "mixed-half", "full-f32", "full-f64"]) <= set(p.POLICY_PRESETS)


def test_round_to_known_answers():
    """tests/test_precision.py:55-90."""
    import paper_2505_00281_b200 as p
    F = p.FpFormat
    assert p.round_to(1.0 + 2.0**-11, F.F16) == 1.0
    assert p.round_to(7.0e4, F.F16) == np.inf and p.round_to(-7.0e4, F.F16) == -np.inf
    assert p.round_to(65504.0, F.F16) == 65504.0
    assert p.round_to(2.0**-24, F.F16) == 2.0**-24 and p.round_to(2.0**-26, F.F16) == 0.0
    assert np.isnan(p.round_to(np.nan, F.F16))
    x = np.random.default_rng(11).standard_normal(300) * 10.0 ** np.random.default_rng(1).integers(-6, 6, 300)
    for fmt in (F.F16, F.F32, F.F64, F.BF16, F.FP8_E4M3):
        once = p.round_to(x, fmt)
        np.testing.assert_array_equal(p.round_to(once, fmt), once)
    assert p.round_to(500.0, F.FP8_E4M3) == np.inf and p.round_to(464.0, F.FP8_E4M3) == 448.0


def test_round_to_matches_oracle(oracle):
    import paper_2505_00281_b200 as p
    rng = np.random.default_rng(3)
    x = np.sign(rng.standard_normal(5000)) * 2.0 ** rng.uniform(-30, 17, 5000)
    for fmt in (0, 1, 2, 3):
        np.testing.assert_array_equal(p.round_to(x, p.FpFormat(fmt)), oracle.round_to(x, fmt))


def test_iterconfig_validation():
    """tests/test_driver.py:26-39 + the tol/top extension."""
    import paper_2505_00281_b200 as p
    with pytest.raises(ValueError):
        p.IterConfig(k=0, policy=p.FULL_F64)
    with pytest.raises(ValueError):
        p.IterConfig(k=2, projection="qr", policy=p.FULL_F64)
    with pytest.raises(ValueError):
        p.IterConfig(k=2)
    with pytest.raises(ValueError):
        p.IterConfig(k=4, policy=p.FULL_F64, top=5)
    with pytest.raises(ValueError):   # a ladder switches on the residual estimate: needs tol
        p.IterConfig(k=4, policy=p.FULL_F64, ladder=p.FULL_F32)
    cfg = p.IterConfig(k=2, policy=p.FULL_F64)
    assert cfg.mv_policy is p.FULL_F64 and cfg.m == 1 and cfg.iter == 1 and cfg.seed == 0
    assert cfg.basis_method is p.BasisMethod.MGS_LEFT and cfg.projection == "rr"   # reference defaults
    cfg2 = p.IterConfig(k=2, policy=p.FULL_F64, matvec_policy=p.MIXED_HALF)
    assert cfg2.mv_policy is p.MIXED_HALF


def test_driver_rejects_non_ofrr_paths_before_touching_the_gpu():
    import paper_2505_00281_b200 as p
    a = p.DenseMatrix(np.eye(4), p.FpFormat.F64)
    with pytest.raises(ValueError):   # Krylov builders: ofrr/driver.py:92-93
        p.subspace_iter_eig(a, p.IterConfig(k=2, basis_method=p.BasisMethod.ARNOLDI_MGS, policy=p.FULL_F64))
    with pytest.raises(ValueError):   # Krylov builders are not block builders for the SVD either
        p.subspace_iter_svd(a, p.IterConfig(k=2, basis_method=p.BasisMethod.KRYLOV_HESS, policy=p.FULL_F64))
    with pytest.raises(ValueError):   # the eig-path extensions are rejected by the SVD driver
        p.subspace_iter_svd(a, p.IterConfig(k=2, basis_method=p.BasisMethod.HESS_LEFT, policy=p.FULL_F64,
                                            tol=1e-6, ladder=p.FULL_F32))
    with pytest.raises(ValueError):   # k > n: ofrr/driver.py:94-96
        p.subspace_iter_eig(p.DenseMatrix(np.eye(3), p.FpFormat.F64),
                            p.IterConfig(k=5, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                                         policy=p.FULL_F64))
    with pytest.raises(ValueError):
        p.build_basis(a, p.BasisMethod.ARNOLDI_MGS, p.FULL_F64)


def test_projection_policy_rule():
    """ofrr/projection.py:42-53 (tests/test_projection.py:34-51) + bf16/fp8 -> fp64."""
    import paper_2505_00281_b200 as p
    F = p.FpFormat
    proj, out = p.projection_policy(p.NATIVE_F16)
    assert proj.compute is F.F32 and proj.accumulate is F.F32 and out is F.F32
    proj, out = p.projection_policy(p.FULL_F32)
    assert proj.storage is F.F32 and proj.compute is F.F64 and out is F.F64
    assert p.projection_policy(p.FULL_F64) == (p.FULL_F64, F.F64)
    assert p.projection_policy(p.TC_BF16)[1] is F.F64


def test_synthetic_factors_spectrum():
    """The host factors of the device generator (K8) give A = Q B Q^T with the prescribed
    spectrum (checked in FP64 on the host at a small size)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as o
    import paper_2505_00281_b200 as p
    for n in (64, 100):
        lam = p.geometric_spectrum(n, 8, 16)
        f = p.sym_factors(lam, seed=5)
        a = o.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, o.F64)
        np.testing.assert_allclose(a, a.T, atol=1e-15)
        np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(a))[::-1], lam, atol=1e-13)
    c = p.clustered_spectrum(200)
    assert np.all(np.diff(c) <= 0) and len(c) == 200
