"""The drop-in boundary exercised from the reference's side: the
UNMODIFIED reference package (installed into baseline/_ref by pip) runs with its kernel
plugin slot ``ofrr.backend.kernels`` swapped to paper_2505_00281_b200.reference_backend --
the reference's own driver, projection and small-solve code calling libofrr_b200.so's
``ofrr_host_gemm_mixed`` / ``ofrr_host_jacobi_eig`` -- and its results are held against the
same calls with the reference's compiled kernels.  The checks mirror the reference's own
tests (tests/test_driver.py:53-79, tests/test_projection.py:71-86, tests/test_smallsolve.py)
with the tolerances of a device backend (products exact, sums in parallel order).
Skipped when baseline/_ref is not installed."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "ofrr")), reason="baseline/_ref not installed")]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    import ofrr
    import ofrr.backend
    from paper_2505_00281_b200 import reference_backend
    return ofrr, ofrr.backend, reference_backend


def _swap(backend, mod):
    saved = backend.kernels
    backend.kernels = mod
    return saved


def test_plugin_module_has_the_reference_interface(ref):
    ofrr, backend, b200 = ref
    for name in ("gemm_mixed", "dot_mixed", "spmv_mixed", "jacobi_eig", "BACKEND_NAME"):
        assert hasattr(b200, name)
        assert hasattr(backend.kernels, name)


@pytest.mark.parametrize("pname", ["full-f64", "full-f32", "mixed-half", "native-f16"])
def test_mixed_gemm_through_the_plugin(ref, pname):
    ofrr, backend, b200 = ref
    from ofrr.precision import POLICY_PRESETS, FpFormat, mixed_gemm, round_to
    pol = POLICY_PRESETS[pname]
    rng = np.random.default_rng(3)
    a = round_to(rng.standard_normal((70, 300)), pol.storage)
    b = round_to(rng.standard_normal((300, 9)), pol.storage)
    want = mixed_gemm(a, b, pol, FpFormat.F64)
    saved = _swap(backend, b200)
    try:
        got = mixed_gemm(a, b, pol, FpFormat.F64)
    finally:
        backend.kernels = saved
    # exact products (the reference rounds each to the compute format), fp32 / fp64 sums in
    # another order: agreement to the coarser of the compute and accumulate formats
    e = {FpFormat.F64: 2.0 ** -52, FpFormat.F32: 2.0 ** -23, FpFormat.F16: 2.0 ** -10}
    eps = max(e[pol.compute], e[pol.accumulate])
    bound = 64 * eps * (np.abs(a) @ np.abs(b))
    assert np.all(np.abs(got - want) <= bound)


def test_sym_eig_through_the_plugin(ref):
    ofrr, backend, b200 = ref
    from ofrr.smallsolve import sym_def_gen_eig, sym_eig
    rng = np.random.default_rng(4)
    s = rng.standard_normal((30, 30))
    s = (s + s.T) / 2
    r = rng.standard_normal((30, 30))
    m = r.T @ r + np.eye(30)
    want, want_g = sym_eig(s), sym_def_gen_eig(s, m)
    saved = _swap(backend, b200)
    try:
        got, got_g = sym_eig(s), sym_def_gen_eig(s, m)
    finally:
        backend.kernels = saved
    np.testing.assert_allclose(got.values, want.values, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(got.vectors, want.vectors, atol=1e-10)       # same sign rule
    np.testing.assert_allclose(got_g.values, want_g.values, rtol=1e-11, atol=1e-12)


def test_rayleigh_quotient_known_answer_through_the_plugin(ref):
    """tests/test_projection.py:71-75 with the plugin in place."""
    ofrr, backend, b200 = ref
    from ofrr.matrix import DenseMatrix
    from ofrr.precision import FULL_F64, FpFormat
    from ofrr.projection import ofrr_eig
    saved = _swap(backend, b200)
    try:
        rs = ofrr_eig(DenseMatrix(np.diag([3.0, 1.0]), FpFormat.F64), DenseMatrix(np.ones((2, 1)), FpFormat.F64),
                      FULL_F64)
    finally:
        backend.kernels = saved
    assert rs.values[0] == pytest.approx(2.0, abs=1e-14)


@pytest.mark.parametrize("pname,method,proj", [("full-f64", "hess-l", "ofrr"), ("full-f32", "hess-r", "ofrr"),
                                                ("full-f64", "mgs-l", "rr"), ("mixed-half", "hess-l", "ofrr")])
def test_reference_driver_through_the_plugin(ref, pname, method, proj):
    """The reference's subspace_iter_eig (tests/test_driver.py:53-70 style) on a kernel
    matrix with the plugin vs the compiled reference kernels: north-star criteria."""
    ofrr, backend, b200 = ref
    from ofrr.basis import BasisMethod
    from ofrr.driver import IterConfig, subspace_iter_eig
    from ofrr.matrix import KernelConfig, gaussian_kernel, sample_uniform_square
    from ofrr.precision import POLICY_PRESETS, FpFormat
    pts = sample_uniform_square(150, float(np.sqrt(150)), 11)
    a = gaussian_kernel(KernelConfig(1.0, 10.0, 0.01, pts), FpFormat.F64)
    cfg = IterConfig(k=16, m=4, iter=2, basis_method=BasisMethod(method), projection=proj,
                     policy=POLICY_PRESETS[pname], seed=20240901)
    want = subspace_iter_eig(a, cfg)
    saved = _swap(backend, b200)
    try:
        got = subspace_iter_eig(a, cfg)
    finally:
        backend.kernels = saved
    exact = np.sort(np.linalg.eigvalsh(a.data))[::-1]
    top = 6
    ref_err = np.abs(want.values[:top] - exact[:top]) / exact[:top]
    err = np.abs(got.values[:top] - exact[:top]) / exact[:top]
    if pname == "full-f64":                       # per pair
        assert np.all(err <= np.maximum(10 * ref_err, 1e-6)), (err, ref_err)
        assert np.all(got.residuals[:top] <= 2 * want.residuals[:top] + 1e-13)
    else:                                         # fp32 / 16-bit sums in another order: error levels
        assert np.max(err) <= max(10 * np.max(ref_err), 1e-6), (err, ref_err)
        assert np.max(got.residuals[:top]) <= 2 * np.max(want.residuals[:top]) + 1e-13
