"""End-to-end GPU parity of the OFRR drivers against the reference (golden vectors) and
the oracle, with the north-star criteria: Ritz values within
max(10 x the reference's error vs exact, 1e-6 relative), residuals within 2x."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 20240901


def _criteria(vals, res, ref_vals, ref_res, exact, top, per_pair=False):
    """North-star parity: Ritz values within max(10 x the reference's error vs exact,
    1e-6 relative) and residuals within 2 x the reference's.

    ``per_pair`` (fp32 / fp64 bases): every pair on its own.  Otherwise (16-bit storage) the
    reference's error level over the checked pairs (max over the top pairs): a single pair's
    error is a rounding lottery between eps-sized outcomes there, so a per-pair 10x bound
    would test luck, not parity."""
    ref_err = np.abs(ref_vals[:top] - exact[:top]) / np.abs(exact[:top])
    err = np.abs(vals[:top] - exact[:top]) / np.abs(exact[:top])
    if per_pair:
        assert np.all(err <= np.maximum(10 * ref_err, 1e-6)), (err, ref_err)
        assert np.all(res[:top] <= 2 * ref_res[:top] + 1e-13), (res[:top], ref_res[:top])
        return
    assert np.max(err) <= max(10 * np.max(ref_err), 1e-6), (err, ref_err)
    assert np.max(res[:top]) <= 2 * np.max(ref_res[:top]) + 1e-13, (res[:top], ref_res[:top])


@pytest.mark.parametrize("pname", ["full-f64", "full-f32", "tc-f16"])
@pytest.mark.parametrize("method", ["hess-l", "hess-r"])
def test_driver_eig_vs_reference_golden(ofrr_gpu, golden, pname, method):
    """subspace_iter_eig(kernel matrix n=120, k=20, m=3, iter=2) vs the reference's run."""
    p = ofrr_gpu
    pol = p.POLICY_PRESETS[pname]
    key = f"driver_eig/{pname}/{method}"
    a = p.DenseMatrix(golden[key + "/a"], p.FpFormat.F64)
    cfg = p.IterConfig(k=20, m=3, iter=2, basis_method=p.BasisMethod(method), projection="ofrr", policy=pol, seed=2)
    rs = p.subspace_iter_eig(a, cfg)
    exact = golden["driver_eig/exact"] if pname == "full-f64" else \
        np.sort(np.linalg.eigvalsh(golden[key + "/a"]))[::-1]
    _criteria(rs.values, rs.residuals, golden[key + "/vals"], golden[key + "/res"], exact, 6,
              per_pair=pname in ("full-f64", "full-f32"))
    assert rs.vectors.data.shape == golden[key + "/vecs"].shape


def test_driver_eig_deterministic(ofrr_gpu, golden):
    """tests/test_driver.py:72-79: bitwise determinism of repeated runs."""
    p = ofrr_gpu
    a = p.DenseMatrix(golden["driver_eig/tc-f16/hess-l/a"], p.FpFormat.F64)
    cfg = p.IterConfig(k=8, m=2, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.TC_F16, seed=5)
    r1 = p.subspace_iter_eig(a, cfg)
    r2 = p.subspace_iter_eig(a, cfg)
    np.testing.assert_array_equal(r1.values, r2.values)
    np.testing.assert_array_equal(r1.vectors.data, r2.vectors.data)


@pytest.mark.parametrize("pname", ["full-f64", "full-f32"])
def test_driver_svd_vs_reference_golden(ofrr_gpu, golden, pname):
    p = ofrr_gpu
    key = f"driver_svd/{pname}"
    a = p.DenseMatrix(golden[key + "/a"], p.FpFormat.F64)
    cfg = p.IterConfig(k=10, m=6, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.POLICY_PRESETS[pname], seed=9)
    rs = p.subspace_iter_svd(a, cfg)
    exact = np.linalg.svd(golden[key + "/a"], compute_uv=False)
    _criteria(rs.values, rs.residuals, golden[key + "/vals"], golden[key + "/res"], exact, 5, per_pair=True)


def test_ofrr_eig_known_answers(ofrr_gpu, golden):
    p = ofrr_gpu
    # Rayleigh quotient 2.0 for diag(3,1), u=[1,1] (tests/test_projection.py:71-75)
    rs = p.ofrr_eig(p.DenseMatrix(np.diag([3.0, 1.0]), p.FpFormat.F64),
                    p.DenseMatrix(np.array([[1.0], [1.0]]), p.FpFormat.F64), p.FULL_F64)
    assert rs.values[0] == pytest.approx(2.0, abs=1e-14)
    for pname in ("full-f64", "full-f32"):
        rs = p.ofrr_eig(p.DenseMatrix(golden[f"ofrreig/{pname}/a"], p.FpFormat.F64),
                        p.DenseMatrix(golden[f"ofrreig/{pname}/u"], p.POLICY_PRESETS[pname].storage),
                        p.POLICY_PRESETS[pname])
        # full-f32: the reference rounds every fp32 product and sum of A.U; the device uses
        # fp32 FMA in another order -> agreement at the fp32 level
        rt = 1e-10 if pname == "full-f64" else 2e-5
        np.testing.assert_allclose(rs.values, golden[f"ofrreig/{pname}/vals"], rtol=rt, atol=rt)
        np.testing.assert_allclose(rs.vectors.data, golden[f"ofrreig/{pname}/vecs"], rtol=1e3 * rt, atol=1e3 * rt)


def test_ofrr_eig_errors(ofrr_gpu):
    p = ofrr_gpu
    with pytest.raises(p.EmptyPencilError):       # tests/test_projection.py:96-99
        p.ofrr_eig(p.DenseMatrix(np.eye(3), p.FpFormat.F64), p.DenseMatrix(np.zeros((3, 2)), p.FpFormat.F64),
                   p.FULL_F64)
    with pytest.raises(p.OverflowDiagnostic):      # tests/test_projection.py:101-105
        p.ofrr_eig(p.DenseMatrix(np.full((2, 2), 6.0e4), p.FpFormat.F64),
                   p.DenseMatrix(np.full((2, 1), 6.0e4), p.FpFormat.F64), p.NATIVE_F16)


def test_ofrr_svd_golden(ofrr_gpu, golden):
    p = ofrr_gpu
    rs = p.ofrr_svd(p.DenseMatrix(golden["ofrrsvd/a"], p.FpFormat.F64),
                    p.DenseMatrix(golden["ofrrsvd/u"], p.FpFormat.F64),
                    p.DenseMatrix(golden["ofrrsvd/v"], p.FpFormat.F64), p.FULL_F64)
    np.testing.assert_allclose(rs.values, golden["ofrrsvd/vals"], rtol=1e-10)
    np.testing.assert_allclose(rs.vectors.data, golden["ofrrsvd/uu"], rtol=1e-7, atol=1e-8)
    np.testing.assert_allclose(rs.right_vectors.data, golden["ofrrsvd/vv"], rtol=1e-7, atol=1e-8)


@pytest.mark.parametrize("fmt", ["tc-bf16", "tc-f16", "full-f32", "tc-fp8"])
def test_driver_eig_vs_oracle_geometric(ofrr_gpu, oracle, fmt):
    """C1/C2-style problem at oracle-feasible size: geometric spectrum, n=1024 (WHT
    generator), top 10, k 20: same synthetic A, same X0, same policy."""
    p, o = ofrr_gpu, oracle
    n, top, k, m = 1024, 10, 20, 5
    pol = p.POLICY_PRESETS[fmt]
    lam = p.geometric_spectrum(n, top, k)
    A, f = p.synthetic_symmetric(lam, pol.storage, seed=SEED)
    a_host = o.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, int(pol.storage))
    cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr", policy=pol,
                       seed=SEED)
    rs = p.subspace_iter_eig(A, cfg)
    ref = o.subspace_iter_eig(a_host, k=k, m=m, iters=1, pol=o.as_pol(pol), seed=SEED)
    exact = np.sort(np.linalg.eigvalsh(a_host))[::-1]
    _criteria(rs.values, rs.residuals, ref.values, ref.residuals, exact, top, per_pair=fmt == "full-f32")


def test_driver_eig_c1_fp32(ofrr_gpu, oracle):
    """C1: 2000 x 2000 dense symmetric, geometric spectrum, top 10, k 20, fp32 basis /
    fp64 projection -- the reference's CPU configuration, run through the oracle."""
    p, o = ofrr_gpu, oracle
    n, top, k, m = 2000, 10, 20, 4
    a_host, lam = o.geometric_symmetric(n, top, k, seed=SEED, fmt=o.F32)
    cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.FULL_F32, seed=SEED)
    rs = p.subspace_iter_eig(p.DenseMatrix(a_host, p.FpFormat.F32), cfg)
    ref = o.subspace_iter_eig(a_host, k=k, m=m, iters=1, pol=o.FULL_F32, seed=SEED)
    exact = np.sort(np.linalg.eigvalsh(a_host))[::-1]
    _criteria(rs.values, rs.residuals, ref.values, ref.residuals, exact, top, per_pair=True)


def test_driver_eig_tolerance_stop(ofrr_gpu):
    """Extension: IterConfig(tol, top) stops at the first outer iteration whose FP64
    residuals of the top pairs are below tol."""
    p = ofrr_gpu
    n, top, k = 4096, 16, 32
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    st = p.RunStats()
    cfg = p.IterConfig(k=k, m=30, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.TC_BF16, seed=SEED, tol=2e-2, top=top)
    rs = p.subspace_iter_eig(A, cfg, stats=st)
    assert st.converged and st.iterations < 30
    assert np.max(rs.residuals[:top]) < 2e-2
    assert st.history[-1][1] < 2e-2


def test_driver_eig_fp32_basis_on_bf16_operator(ofrr_gpu, oracle):
    """full-f32 policy on a bf16-stored operator: the fp32 blocks run on the bf16 tensor
    cores (three-slice split); parity vs the oracle's full-f32 run on the same A."""
    p, o = ofrr_gpu, oracle
    n, top, k, m = 1024, 10, 20, 6
    lam = p.geometric_spectrum(n, top, k)
    A, f = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    a_host = o.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, o.BF16)
    cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.FULL_F32, seed=SEED)
    rs = p.subspace_iter_eig(A, cfg)
    ref = o.subspace_iter_eig(a_host, k=k, m=m, iters=1, pol=o.FULL_F32, seed=SEED)
    exact = np.sort(np.linalg.eigvalsh(a_host))[::-1]
    _criteria(rs.values, rs.residuals, ref.values, ref.residuals, exact, top, per_pair=True)
    assert np.max(rs.residuals[:top]) < 1e-4


def test_driver_eig_fp64_basis_on_bf16_operator(ofrr_gpu, oracle):
    """full-f64 policy on a bf16-stored operator: the fp64 blocks multiply A on the int8
    tensor cores (Ozaki digit planes, no fp64 copy of A); parity vs the oracle's full-f64
    run (FP64 products) on the same A, to 1e-8-class residuals."""
    import paper_2505_00281_b200.ops as ops
    p, o = ofrr_gpu, oracle
    n, top, k, m = 1024, 10, 20, 8
    lam = p.geometric_spectrum(n, top, k)
    A, f = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    a_host = o.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, o.BF16)
    cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.FULL_F64, seed=SEED)
    before = len(A._dev)
    rs = p.subspace_iter_eig(A, cfg)
    assert p.FpFormat.F64 not in A._dev and len(A._dev) == before      # no fp64 copy of A was made
    ref = o.subspace_iter_eig(a_host, k=k, m=m, iters=1, pol=o.FULL_F64, seed=SEED)
    exact = np.sort(np.linalg.eigvalsh(a_host))[::-1]
    _criteria(rs.values, rs.residuals, ref.values, ref.residuals, exact, top)
    assert np.max(rs.residuals[:top]) < 1e-8
    assert ops.OZAKI_FMTS


def test_driver_precision_ladder(ofrr_gpu):
    """IterConfig.ladder: fp32 basis on the bf16 tensor cores first, then the fp64 rung
    (int8 Ozaki products) from its restart block, to a 1e-9 FP64 residual."""
    p = ofrr_gpu
    n, top, k = 4096, 16, 32
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    cfg = p.IterConfig(k=k, m=40, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.FULL_F64, ladder=p.FULL_F32, ladder_switch=1e-3, seed=SEED, tol=1e-9, top=top)
    st = p.RunStats()
    rs = p.subspace_iter_eig(A, cfg, stats=st)
    assert st.converged and np.max(rs.residuals[:top]) < 1e-9
    assert rs.vectors.data.dtype == np.float64
    np.testing.assert_allclose(rs.values[:top], lam[:top], rtol=1e-2)   # A is bf16-rounded
    its = [i for i, _ in st.history]
    assert its == sorted(its) and st.iterations == its[-1]


def test_ozaki_gemm_vs_fp64(ofrr_gpu, oracle):
    """ofrr_ozaki_gemm: W = A X (fp64 X, bf16 A) to ~1e-14 of the FP64 product; column
    inf-norms and the fp32 second output."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(7)
    rows, cols, k = 777, 20000, 70
    a = o.round_to(rng.standard_normal((rows, cols)), 3)
    x = rng.standard_normal((cols, k))
    A = p.DenseMatrix(np.asfortranarray(a), p.FpFormat.F64).device_operator(p.FpFormat.BF16)
    X = ops.block_from_host(x, p.FpFormat.F64, torch.device("cuda"))
    W = ops.new_block(rows, k, p.FpFormat.F64, torch.device("cuda"))
    W2 = ops.new_block(rows, k, p.FpFormat.F32, torch.device("cuda"))
    colmax = torch.zeros(k, dtype=torch.float64, device="cuda")
    ops.gemm_av(A, X, W, colmax=colmax, W2=W2)
    ref = a @ x
    got = W.to_numpy_f64()
    bound = 1e-13 * (np.abs(a) @ np.abs(x))
    assert np.all(np.abs(got - ref) <= bound), np.max(np.abs(got - ref) / bound)
    np.testing.assert_array_equal(colmax.cpu().numpy(), np.max(np.abs(got), axis=0))
    np.testing.assert_array_equal(W2.to_numpy_f64(), o.round_to(got, 1))


@pytest.mark.parametrize("pname", ["tc-bf16", "tc-f16", "full-f32"])
def test_driver_svd_tensor_core_vs_oracle(ofrr_gpu, oracle, pname):
    """partial SVD on the tensor-core path (A V and A^T U both K-major: A^T resident):
    tall low-rank + noise matrix (C4-style, scaled down), vs the oracle on the same A."""
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(SEED)
    n1, n2, r, k, top, m = 3000, 512, 40, 24, 8, 5
    g1, _ = np.linalg.qr(rng.standard_normal((n1, r)))
    g2, _ = np.linalg.qr(rng.standard_normal((n2, r)))
    sig = 0.8 ** np.arange(r)
    a = (g1 * sig) @ g2.T + 1e-4 * rng.standard_normal((n1, n2)) / np.sqrt(n2)
    pol = p.POLICY_PRESETS[pname]
    store = pol.storage if pol.storage != p.FpFormat.F32 else p.FpFormat.BF16
    a = o.round_to(a, int(store))
    cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr", policy=pol,
                       seed=SEED)
    rs = p.subspace_iter_svd(p.DenseMatrix(a, store), cfg)
    ref = o.subspace_iter_svd(a, k=k, m=m, iters=1, pol=o.as_pol(pol), seed=SEED)
    exact = np.linalg.svd(a, compute_uv=False)
    _criteria(rs.values, rs.residuals, ref.values, ref.residuals, exact, top)


@pytest.mark.gpu
@pytest.mark.parametrize("pname", ["tc-bf16", "full-f32", "full-f64"])
def test_driver_reuse_av_vs_oracle(ofrr_gpu, oracle, pname):
    """IterConfig.reuse_av: the MatVec of the restart block comes from the projection's
    W = A U (A U Y = W Y, ofrr_reuse_power) -- one A pass per outer iteration after the
    first.  Parity with the oracle's reference schedule (north-star criteria) and the pass
    count."""
    p, o = ofrr_gpu, oracle
    n, top, k, m = 1024, 10, 20, 8
    lam = p.geometric_spectrum(n, top, k)
    A, f = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    a_host = o.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, o.BF16)
    pol = p.POLICY_PRESETS[pname]
    opol = {"tc-bf16": o.TC_BF16, "full-f32": o.FULL_F32, "full-f64": o.FULL_F64}[pname]
    cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=pol, seed=SEED, reuse_av=True)
    st = p.RunStats()
    rs = p.subspace_iter_eig(A, cfg, stats=st)
    assert st.a_passes == m + 1
    ref = o.subspace_iter_eig(a_host, k=k, m=m, iters=1, pol=opol, seed=SEED)
    exact = np.sort(np.linalg.eigvalsh(a_host))[::-1]
    _criteria(rs.values, rs.residuals, ref.values, ref.residuals, exact, top)
    if pname == "full-f64":
        assert np.max(rs.residuals[:top]) < 1e-8


@pytest.mark.gpu
def test_driver_reuse_av_ladder_to_tol(ofrr_gpu):
    """reuse_av with the precision ladder and a time-to-tolerance stop (the C3 north-star
    configuration at reduced n): converges to the FP64 tolerance with fewer A passes."""
    p = ofrr_gpu
    n, top, k = 4096, 16, 32
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    res = {}
    for reuse in (False, True):
        cfg = p.IterConfig(k=k, m=40, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                           policy=p.FULL_F64, ladder=p.FULL_F32, seed=SEED, tol=1e-9, top=top, reuse_av=reuse)
        st = p.RunStats()
        rs = p.subspace_iter_eig(A, cfg, stats=st)
        assert st.converged and np.max(rs.residuals[:top]) < 1e-9
        res[reuse] = (rs, st)
    np.testing.assert_allclose(res[True][0].values[:top], res[False][0].values[:top], rtol=1e-12)
    assert res[True][1].a_passes < res[False][1].a_passes


@pytest.mark.gpu
@pytest.mark.parametrize("pname,reuse", [("full-f32", False), ("full-f32", True), ("full-f64", True)])
def test_device_loop_matches_host_loop(ofrr_gpu, pname, reuse):
    """The outer loop as one CUDA graph with device-side control flow (csrc/loop.cu:
    conditional WHILE over the captured iteration, IF around the FP64 report): once the
    graphs exist (two earlier solves), a solve launches it once and must reproduce the host
    loop's iterations, values, vectors and residuals exactly."""
    import os
    p = ofrr_gpu
    n, top, k = 4096, 16, 32
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    tol = 1e-4 if pname == "full-f32" else 1e-9
    cfg = p.IterConfig(k=k, m=40, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.POLICY_PRESETS[pname], seed=SEED, tol=tol, top=top, reuse_av=reuse)
    runs = []
    for _ in range(4):
        st = p.RunStats()
        rs = p.subspace_iter_eig(A, cfg, stats=st)
        runs.append((rs, st))
    host_rs, host_st = runs[0]
    assert not host_st.device_loop and runs[-1][1].device_loop
    for rs, st in runs[1:]:
        assert st.converged and st.iterations == host_st.iterations and st.a_passes == host_st.a_passes
        np.testing.assert_array_equal(rs.values, host_rs.values)
        np.testing.assert_array_equal(rs.residuals, host_rs.residuals)
        np.testing.assert_array_equal(rs.vectors.data, host_rs.vectors.data)
        assert [i for i, _ in st.history] == [i for i, _ in host_st.history]
    assert np.max(runs[-1][0].residuals[:top]) < tol


def test_three_rung_ladder_to_fp64(ofrr_gpu):
    """IterConfig.ladder as a tuple: fp32 -> full-f64-lite (~30-bit products) -> full-f64, the
    lite rung handing its next iterate (W Y) over; converged to 1e-9 in FP64, the FP64 report
    taken from the final rung's FP64-accurate W, and the values as exact as the 2-rung ladder."""
    p = ofrr_gpu
    n, top, k = 2048, 16, 32
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    base = dict(k=k, m=40, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr", policy=p.FULL_F64,
                seed=SEED, tol=1e-9, top=top, reuse_av=True)
    st3, st2 = p.RunStats(), p.RunStats()
    rs3 = p.subspace_iter_eig(A, p.IterConfig(ladder=(p.FULL_F32, p.POLICY_PRESETS["full-f64-lite"]),
                                              ladder_switch=(1e-4, 1e-6), **base), stats=st3)
    rs2 = p.subspace_iter_eig(A, p.IterConfig(ladder=p.FULL_F32, ladder_switch=1e-4, **base), stats=st2)
    assert st3.converged and np.max(rs3.residuals[:top]) < 1e-9
    assert [r[0] for r in st3.rungs] == ["F32", "F64L", "F64"]
    np.testing.assert_allclose(rs3.values[:top], rs2.values[:top], rtol=1e-12)
    # the returned residuals are FP64 residuals of the returned vectors
    from paper_2505_00281_b200.projection import residual_report
    indep = residual_report(A, rs3).residuals
    np.testing.assert_allclose(rs3.residuals[:top], indep[:top], rtol=1e-3, atol=1e-13)


def test_fp8_rung_with_column_scaling(ofrr_gpu):
    """The FP8 (e4m3) basis: A and the basis blocks in e4m3 on the f8f6f4 tensor cores; the
    products stay in fp32 until the column scaling (power steps) or the Grams (projection),
    so A U never has to fit e4m3's 448 (C5: it used to overflow).  A clustered spectrum scaled
    to e4m3's range, top-16: no overflow, and the FP8 basis settles at its format's floor
    (e4m3 keeps 3 mantissa bits: residuals ~0.15-0.3, values to a few percent)."""
    p = ofrr_gpu
    n, top, k = 4096, 16, 32
    lam = p.clustered_spectrum(n, clusters=2, per=8)
    probe, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED)
    amax = float(probe.device_operator(p.FpFormat.BF16).t[:, :n].abs().max())
    lam = lam * 2.0 ** np.round(np.log2(2.0 / amax))
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.FP8_E4M3, seed=SEED)
    cfg = p.IterConfig(k=k, m=30, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr", policy=p.TC_FP8,
                       seed=SEED, tol=1e-1, top=top)
    st = p.RunStats()
    rs = p.subspace_iter_eig(A, cfg, stats=st)
    assert np.all(np.isfinite(rs.values[:top])) and np.all(np.isfinite(rs.residuals[:top]))
    assert np.max(rs.residuals[:top]) < 0.5
    assert min(w for _, w in st.history) < 0.3                   # it converged to the e4m3 floor
    err = np.abs(rs.values[:top] - lam[:top]) / lam[:top]
    assert np.max(err) < 0.1, err


@pytest.mark.gpu
def test_graph_cache_keyed_by_basis_and_projection(ofrr_gpu, monkeypatch):
    """Captured iteration graphs are reused only by solves whose body they captured: a solve
    with another basis builder / projection on the same operator and shapes must not replay a
    graph captured for the first one (results equal the graph-free run, bit for bit)."""
    p = ofrr_gpu
    n, k, top = 600, 16, 6
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.F32, seed=5)
    pol = p.POLICY_PRESETS["full-f32"]

    def run(meth, proj):
        cfg = p.IterConfig(k=k, m=3, iter=1, basis_method=p.BasisMethod(meth), projection=proj, policy=pol, seed=3)
        return p.subspace_iter_eig(A, cfg)

    monkeypatch.setenv("OFRR_CUDA_GRAPHS", "0")
    ref = run("cgs", "rr")
    monkeypatch.setenv("OFRR_CUDA_GRAPHS", "1")
    for _ in range(3):
        run("hess-l", "ofrr")                    # warms and captures graphs for these shapes
    for _ in range(3):
        got = run("cgs", "rr")
        np.testing.assert_array_equal(np.asarray(got.values), np.asarray(ref.values))
        np.testing.assert_array_equal(np.asarray(got.residuals), np.asarray(ref.residuals))


@pytest.mark.gpu
@pytest.mark.parametrize("switch,m", [((1e-3, 1e-6), 40), ((1e-30, 1e-30), 3)])
def test_ladder_device_rungs_equal_host_loop(ofrr_gpu, monkeypatch, switch, m):
    """Ladder rungs on the device-side loop (k_loop_decide_rung) give bit for bit the host
    loop's answer: a rung that finishes on the device, and a rung that exhausts m (the device
    stops for the host, which re-runs the rung from the same start block)."""
    from paper_2505_00281_b200 import driver
    p = ofrr_gpu
    n, k, top = 4096, 32, 8
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=21)
    cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.POLICY_PRESETS["full-f64"], seed=4, tol=1e-9, top=top,
                       ladder=(p.POLICY_PRESETS["full-f32-lite"], p.POLICY_PRESETS["full-f64-lite"]),
                       ladder_switch=switch, reuse_av=True)

    def solve():
        st = p.RunStats()
        return p.subspace_iter_eig(A, cfg, stats=st), st

    monkeypatch.setattr(driver, "DEVICE_LOOP", False)
    ref, st_ref = solve()
    monkeypatch.setattr(driver, "DEVICE_LOOP", True)
    for _ in range(3):                          # capture, then the device loops
        got, st = solve()
    np.testing.assert_array_equal(np.asarray(got.values), np.asarray(ref.values))
    np.testing.assert_array_equal(np.asarray(got.residuals), np.asarray(ref.residuals))
    assert st.iterations == st_ref.iterations and st.a_passes == st_ref.a_passes
    assert st.rungs == st_ref.rungs
