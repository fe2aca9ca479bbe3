"""GPU parity of every kernel on the OFRR hot path against the CPU oracle (which is
pinned to the reference by tests/test_oracle_golden.py).  Calls go through the C ABI
(libofrr_b200.so) via the package's typed ops layer."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

F16, F32, F64, BF16, FP8 = 0, 1, 2, 3, 4


def _op(p, a, fmt):
    """row-major device operator from a host float64 matrix (values representable)."""
    m = p.DenseMatrix(np.asfortranarray(a), p.FpFormat.F64)
    return m.device_operator(p.FpFormat(fmt))


def _blk(p, x, fmt):
    from paper_2505_00281_b200 import ops
    import torch
    return ops.block_from_host(x, p.FpFormat(fmt), torch.device("cuda"))


def _host(b, k=None):
    return b.to_numpy_f64(k)


def _ulp_close(got, ref, fmt_eps, frac=1e-2):
    """got == ref except for at most `frac` of entries that differ by one storage ulp."""
    d = np.abs(got - ref)
    bad = d > 0
    if not bad.any():
        return True
    tol = 2.0 * fmt_eps * np.maximum(np.abs(ref), 1e-30)
    return bad.mean() <= frac and np.all(d[bad] <= tol[bad])


@pytest.mark.parametrize("fmt", [BF16, F16])
@pytest.mark.parametrize("shape", [(256, 128, 32), (1000, 1000, 20), (517, 777, 64), (2048, 2048, 128),
                                   (300, 4096, 200), (1, 64, 1), (4000, 512, 256)])
def test_gemm_tc_fp32_out_vs_fp64(ofrr_gpu, oracle, fmt, shape):
    """K1 (tcgen05): fp32-accumulated A.X against the exact fp64 product."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rows, cols, k = shape
    rng = np.random.default_rng(rows * 7 + cols + k)
    a = o.round_to(rng.standard_normal((rows, cols)), fmt)
    x = o.round_to(rng.random((cols, k)), fmt)
    A = _op(p, a, fmt)
    X = _blk(p, x, fmt)
    W = ops.new_block(rows, k, p.FpFormat.F32, A.device)
    colmax = torch.zeros(k, dtype=torch.float64, device=A.device)
    ops.gemm_av(A, X, W, colmax=colmax)
    got = _host(W)
    exact = a @ x
    bound = 1e-5 * (np.abs(a) @ np.abs(x)) + 1e-30
    assert np.all(np.abs(got - exact) <= bound), np.max(np.abs(got - exact) / bound)
    np.testing.assert_array_equal(colmax.cpu().numpy(), np.max(np.abs(got), axis=0))


@pytest.mark.parametrize("fmt", [BF16, F16])
def test_gemm_tc_storage_out_vs_oracle(ofrr_gpu, oracle, fmt):
    """K1 rounded to the storage format vs the oracle's mixed_gemm (F32 products/sums):
    equal except for rare one-ulp ties decided by the fp32 summation order."""
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(11)
    rows, cols, k = 1500, 1300, 48
    a = o.round_to(rng.standard_normal((rows, cols)), fmt)
    x = o.round_to(rng.random((cols, k)), fmt)
    A = _op(p, a, fmt)
    W = ops.new_block(rows, k, p.FpFormat(fmt), A.device)
    ops.gemm_av(A, _blk(p, x, fmt), W)
    ref = o.mixed_gemm(a, x, F32, F32, fmt)
    got = _host(W)
    d = np.abs(got - ref)
    bad = d > 0
    msg = f"{bad.mean():.2e} of entries differ; max rel {np.max(d / np.maximum(np.abs(ref), 1e-30)):.2e}"
    # a differing entry is one storage ulp away, or within the fp32 summation-order
    # error (sums that cancel to near zero)
    allowed = 2.0 * o.EPS[fmt] * np.abs(ref) + 1e-5 * (np.abs(a) @ np.abs(x))
    assert bad.mean() <= 1e-2 and np.all(d <= allowed), msg


def test_gemm_fp8(ofrr_gpu, oracle):
    """K1 kind::f8f6f4 (e4m3) vs the exact product."""
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(3)
    rows, cols, k = 700, 1024, 64
    a = o.round_to(rng.standard_normal((rows, cols)), FP8)
    x = o.round_to(rng.random((cols, k)), FP8)
    A = _op(p, a, FP8)
    W = ops.new_block(rows, k, p.FpFormat.F32, A.device)
    ops.gemm_av(A, _blk(p, x, FP8), W)
    exact = a @ x
    assert np.all(np.abs(_host(W) - exact) <= 1e-5 * (np.abs(a) @ np.abs(x)) + 1e-30)


@pytest.mark.parametrize("fmt", [F32, F64])
def test_gemm_simt_vs_oracle(ofrr_gpu, oracle, fmt):
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(5)
    rows, cols, k = 333, 450, 20
    a = o.round_to(rng.standard_normal((rows, cols)), fmt)
    x = o.round_to(rng.random((cols, k)), fmt)
    A = _op(p, a, fmt)
    W = ops.new_block(rows, k, p.FpFormat(fmt), A.device)
    ops.gemm_av(A, _blk(p, x, fmt), W)
    ref = o.mixed_gemm(a, x, fmt, fmt, fmt)
    tol = 1e-5 if fmt == F32 else 1e-13
    np.testing.assert_allclose(_host(W), ref, rtol=tol, atol=tol * np.abs(ref).max())


@pytest.mark.parametrize("pname,pol", [("tc-bf16", (BF16, F32, F32)), ("tc-f16", (F16, F32, F32)),
                                       ("native-f16", (F16, F16, F16)), ("full-f32", (F32, F32, F32)),
                                       ("full-f64", (F64, F64, F64))])
def test_scale_columns_bitwise(ofrr_gpu, oracle, pname, pol):
    """K2 reproduces ofrr/precision.py:159-169 bit for bit."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    s, c, a_ = pol
    rng = np.random.default_rng(9)
    x = o.round_to(rng.standard_normal((1234, 7)) * 40, s)
    x[:, 3] = 0.0
    X = _blk(p, x, s)
    colmax = torch.tensor(np.max(np.abs(x), axis=0), dtype=torch.float64, device="cuda")
    ops.scale_columns(X, colmax, p.FpFormat(c))
    np.testing.assert_array_equal(_host(X), o.scale_columns_inf(x, o.Pol(s, c, a_)))


@pytest.mark.parametrize("pol", [(BF16, F32, F32), (F16, F32, F32), (F16, F16, F16), (F16, F16, F32),
                                 (F32, F32, F32), (F64, F64, F64), (FP8, F32, F32), (FP8, BF16, F32),
                                 (F32, F64, F64), (BF16, BF16, F32)])
@pytest.mark.parametrize("n,k", [(300, 12), (5000, 64), (20000, 40)])
def test_hessenberg_bitwise(ofrr_gpu, oracle, pol, n, k):
    """K3 reproduces ofrr/basis.py:151-196 bit for bit: Q, pivots, kept."""
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    s, c, a_ = pol
    rng = np.random.default_rng(n + k)
    x = o.round_to(rng.random((n, k)), s)
    h = ops.hessenberg(_blk(p, x, s), p.FpFormat(s), p.FpFormat(c), o.EPS[s])
    nk = int(h.n_kept.item())
    q, piv, kept = o.hessenberg_basis(x, o.Pol(s, c, a_))
    assert nk == q.shape[1]
    np.testing.assert_array_equal(h.pivots[:nk].cpu().numpy(), piv)
    np.testing.assert_array_equal(h.kept[:k].cpu().numpy().astype(bool), kept)
    np.testing.assert_array_equal(_host(h.Q, nk), q)


@pytest.mark.parametrize("pol", [(F32, F32, F32), (F64, F64, F64), (BF16, F32, F32), (F32, F64, F64)])
def test_hessenberg_c3_shape_bitwise(ofrr_gpu, oracle, pol):
    """K3 at the headline shape (65536 x 128: 443 rows per CTA, the fp32 rows in shared
    memory with 16-byte trailing updates, the fp64 rows in global memory with panels), a
    dependent column included: Q, pivots and kept bit for bit."""
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    s, c, a_ = pol
    n, k = 65536, 128
    rng = np.random.default_rng(65)
    x = o.round_to(rng.random((n, k)) - 0.25, s)
    x[:, 77] = o.round_to(0.5 * x[:, 3], s)
    h = ops.hessenberg(_blk(p, x, s), p.FpFormat(s), p.FpFormat(c), o.EPS[s])
    nk = int(h.n_kept.item())
    q, piv, kept = o.hessenberg_basis(x, o.Pol(s, c, a_))
    assert nk == q.shape[1] and nk < k
    np.testing.assert_array_equal(h.pivots[:nk].cpu().numpy(), piv)
    np.testing.assert_array_equal(h.kept[:k].cpu().numpy().astype(bool), kept)
    np.testing.assert_array_equal(_host(h.Q, nk), q)


@pytest.mark.parametrize("pol", [(BF16, F32, F32), (F32, F32, F32), (F64, F64, F64), (FP8, BF16, F32)])
@pytest.mark.parametrize("pb", [1, 8, 32])
def test_hessenberg_global_panels_bitwise(ofrr_gpu, oracle, pol, pb):
    """K3's global-memory mode (row blocks too large for shared memory, e.g. C3's fp64 rung)
    with panel-deferred trailing updates: still the reference's Q, pivots and kept mask bit
    for bit, including a dependent (dropped) column and a panel boundary inside the block."""
    import ctypes
    from paper_2505_00281_b200 import ops, _lib
    p, o = ofrr_gpu, oracle
    s, c, a_ = pol
    n, k = 6000, 45
    rng = np.random.default_rng(7)
    x = o.round_to(rng.random((n, k)) - 0.5, s)
    x[:, 9] = o.round_to(2.0 * x[:, 4], s)                 # dependent column -> skipped
    L = _lib.load()
    L.ofrr_debug_hess_mode.argtypes = [ctypes.c_int, ctypes.c_int]
    L.ofrr_debug_hess_mode(1, pb)
    try:
        h = ops.hessenberg(_blk(p, x, s), p.FpFormat(s), p.FpFormat(c), o.EPS[s])
        nk = int(h.n_kept.item())
        Q = _host(h.Q, nk)
    finally:
        L.ofrr_debug_hess_mode(0, -1)
    q, piv, kept = o.hessenberg_basis(x, o.Pol(s, c, a_))
    assert nk == q.shape[1]
    np.testing.assert_array_equal(h.pivots[:nk].cpu().numpy(), piv)
    np.testing.assert_array_equal(h.kept[:k].cpu().numpy().astype(bool), kept)
    np.testing.assert_array_equal(Q, q)


@pytest.mark.parametrize("case", ["f64_20x6", "f16_25x8", "mh_64x10", "f32_64x10", "tc16_300x12", "dep_6x3",
                                  "ties_8x3"])
def test_hessenberg_golden(ofrr_gpu, golden, case):
    """K3 against the reference's own outputs (tests/golden)."""
    from paper_2505_00281_b200 import ops
    p = ofrr_gpu
    key = f"hess/{case}/left"
    s, c, _ = (int(v) for v in golden[key + "/policy"])
    x = golden[key + "/x"]
    eps = {0: 2.0**-10, 1: 2.0**-23, 2: 2.0**-52}[s]
    h = ops.hessenberg(_blk(p, x, s), p.FpFormat(s), p.FpFormat(c), eps)
    nk = int(h.n_kept.item())
    np.testing.assert_array_equal(_host(h.Q, nk), golden[key + "/q"])
    np.testing.assert_array_equal(h.pivots[:nk].cpu().numpy(), golden[key + "/pivots"])
    np.testing.assert_array_equal(h.kept[: x.shape[1]].cpu().numpy().astype(bool), golden[key + "/kept"])


@pytest.mark.parametrize("fmt,out", [(BF16, F64), (F16, F32), (F32, F64), (F64, F64)])
@pytest.mark.parametrize("k", [70, 128])
def test_gram_vs_fp64(ofrr_gpu, oracle, fmt, out, k):
    """K4: U^T W and U^T U (fp64 sums of exact products), rounded to the projection format
    (k = 128: tile-aligned, the U^T U tiles below the diagonal mirrored)."""
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(fmt * 10 + out)
    n = 9000
    u = o.round_to(rng.standard_normal((n, k)), fmt)
    w = o.round_to(rng.standard_normal((n, k)), fmt)
    G1, G2 = ops.gram(_blk(p, u, fmt), _blk(p, w, fmt), p.FpFormat(out))
    g1 = G1.cpu().numpy().T
    g2 = G2.cpu().numpy().T
    tol = 1e-12 if out == F64 else 2e-7
    np.testing.assert_allclose(g1, o.round_to(u.T @ w, out), rtol=tol, atol=tol * np.abs(u.T @ w).max())
    np.testing.assert_allclose(g2, o.round_to(u.T @ u, out), rtol=tol, atol=tol * np.abs(u.T @ u).max())


@pytest.mark.parametrize("n", [1, 2, 5, 12, 40])
def test_sym_eig_golden(ofrr_gpu, golden, n):
    """K5 sym_eig vs the reference's Jacobi results (ordering and sign rule included)."""
    p = ofrr_gpu
    r = p.sym_eig(golden[f"symeig/{n}/s"])
    np.testing.assert_allclose(r.values, golden[f"symeig/{n}/vals"], rtol=1e-12, atol=1e-12 * n)
    np.testing.assert_allclose(r.vectors, golden[f"symeig/{n}/vecs"], atol=1e-9)


@pytest.mark.parametrize("n", ["2", "6", "15", "33", "rankdef"])
def test_gen_eig_golden(ofrr_gpu, golden, n):
    p = ofrr_gpu
    r = p.sym_def_gen_eig(golden[f"geneig/{n}/b"], golden[f"geneig/{n}/m"])
    np.testing.assert_allclose(r.values, golden[f"geneig/{n}/vals"], rtol=1e-10, atol=1e-11)
    np.testing.assert_allclose(r.vectors, golden[f"geneig/{n}/vecs"], rtol=1e-8, atol=1e-9)


@pytest.mark.parametrize("k", [64, 100, 128, 200, 400])
def test_gen_eig_large_vs_lapack(ofrr_gpu, k):
    """K5 at the basis widths of the BASELINE configs (k = 64 / 128; 200 / 400 for SVD)."""
    import scipy.linalg
    p = ofrr_gpu
    rng = np.random.default_rng(k)
    b = rng.standard_normal((k, k))
    b = (b + b.T) / 2
    r = rng.standard_normal((k, k))
    m = r.T @ r + 0.5 * np.eye(k)
    res = p.sym_def_gen_eig(b, m)
    ref = np.sort(scipy.linalg.eigh(b, m, eigvals_only=True))[::-1]
    np.testing.assert_allclose(res.values, ref, atol=1e-9 * np.abs(ref).max())
    g = res.vectors.T @ m @ res.vectors
    np.testing.assert_allclose(g, np.eye(k), atol=1e-8)


def test_svd_block_pencil_k400_vs_lapack(ofrr_gpu):
    """The C4 SVD pencil (k1 = k2 = 200 -> 400 x 400): [[0, G], [G', 0]] against
    diag(Mu, Mv), as ofrr_svd assembles it (ofrr/projection.py:99-133): the positive
    eigenvalues are the singular values of Lu^-1 G Lv^-T (Mu = Lu Lu', Mv = Lv Lv')."""
    import scipy.linalg
    p = ofrr_gpu
    rng = np.random.default_rng(400)
    k1 = k2 = 200
    g = rng.standard_normal((k1, k2)) * (0.9 ** np.arange(k2))[None, :]
    ru, rv = rng.standard_normal((k1, k1)), rng.standard_normal((k2, k2))
    mu, mv = ru.T @ ru / k1 + np.eye(k1), rv.T @ rv / k2 + np.eye(k2)
    b = np.zeros((k1 + k2, k1 + k2))
    b[:k1, k1:], b[k1:, :k1] = g, g.T
    m = scipy.linalg.block_diag(mu, mv)
    res = p.sym_def_gen_eig(b, m)
    lu, lv = np.linalg.cholesky(mu), np.linalg.cholesky(mv)
    sv = np.linalg.svd(np.linalg.solve(lu, np.linalg.solve(lv, g.T).T), compute_uv=False)
    np.testing.assert_allclose(res.values[:k2], sv, rtol=1e-9, atol=1e-12 * sv[0])
    np.testing.assert_allclose(res.values[k2:], -sv[::-1], rtol=1e-9, atol=1e-12 * sv[0])
    # +-sigma pairs of the smallest singular values (0.9^200 ~ 7e-10) are nearly degenerate
    # around 0: M-orthonormality there is ~eps ||B|| / gap
    y = res.vectors
    np.testing.assert_allclose(y.T @ m @ y, np.eye(k1 + k2), atol=1e-6)


def test_ritz_and_residual(ofrr_gpu, oracle):
    """K6 (U Y in fp64 + storage rounding) and K7 (FP64 residual) vs numpy."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(1)
    n, k = 3000, 40
    u = o.round_to(rng.standard_normal((n, k)), BF16)
    y = rng.standard_normal((k, k))
    U = _blk(p, u, BF16)
    Y = torch.tensor(np.ascontiguousarray(y.T), device="cuda")
    r_dev = torch.tensor([30], dtype=torch.int32, device="cuda")
    U64, X = ops.ritz(U, Y, k, r_dev, k, 1.0, want64=True, x_fmt=p.FpFormat.BF16)
    ut = u @ y[:, :30]
    np.testing.assert_allclose(_host(U64)[:, :30], ut, rtol=1e-12, atol=1e-12 * np.abs(ut).max())
    assert not _host(U64)[:, 30:].any()
    np.testing.assert_array_equal(_host(X)[:, :30], o.round_to(_host(U64)[:, :30], BF16))
    # residual
    a = rng.standard_normal((n, n))
    a = o.round_to((a + a.T) / 2, BF16)
    A = _op(p, a, BF16)
    lam = rng.standard_normal(30)
    res = ops.residual_eig(A, U64, torch.tensor(lam, device="cuda"), None, 30).cpu().numpy()
    ref = np.linalg.norm(a @ ut - ut * lam[None, :], axis=0) / np.abs(lam)
    np.testing.assert_allclose(res, ref, rtol=1e-10)


@pytest.mark.parametrize("n,k,r_max,rv,ufmt,wfmt", [(3001, 40, 30, 30, BF16, F32), (16384, 64, 32, 32, F32, F32),
                                                    (1000, 70, 65, 41, F32, F64), (33, 5, 3, 2, F16, F32)])
@pytest.mark.parametrize("mode", [0, 2])
def test_residual_estimate_vs_numpy(ofrr_gpu, oracle, n, k, r_max, rv, ufmt, wfmt, mode):
    """K7e: ||(W - lambda_j U) y_j|| / |lambda_j| (mode 0) / raw sums of squares (mode 2)
    over the first r = min(r_max, *r_dev) Ritz columns, zeros past r."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(n + k)
    u = o.round_to(rng.standard_normal((n, k)), ufmt)
    w = rng.standard_normal((n, k))
    w = w if wfmt == F64 else o.round_to(w, wfmt)
    y = rng.standard_normal((k, k))
    lam = rng.uniform(0.5, 2.0, k) * rng.choice([-1, 1], k)
    U, W = _blk(p, u, ufmt), _blk(p, w, wfmt)
    Y = torch.tensor(np.ascontiguousarray(y.T), device="cuda")
    r_dev = torch.tensor([rv], dtype=torch.int32, device="cuda")
    got = ops.residual_estimate(U, W, Y, k, torch.tensor(lam, device="cuda"), r_dev, r_max, mode=mode).cpu().numpy()
    d = w @ y[:, :rv] - (u @ y[:, :rv]) * lam[None, :rv]
    ss = np.sum(d * d, axis=0)
    ref = ss if mode == 2 else np.sqrt(ss) / np.abs(lam[:rv])
    np.testing.assert_allclose(got[:rv], ref, rtol=1e-11)
    assert not got[rv:].any()


@pytest.mark.parametrize("n,k,r_max,rv,t,ufmt,wfmt,xfmt", [(3001, 40, 40, 30, 24, BF16, F32, BF16),
                                                            (65536, 128, 128, 128, 64, F32, F32, F32),
                                                            (1000, 70, 65, 41, 65, F64, F64, F64),
                                                            (33, 5, 3, 2, 1, F16, F32, F16),
                                                            (777, 96, 96, 80, 0, F32, F32, F32)])
def test_restart_fused_vs_separate(ofrr_gpu, oracle, n, k, r_max, rv, t, ufmt, wfmt, xfmt):
    """K6f: Ritz block (fp64 and rounded), next power step W Y (rounded, column maxima,
    non-finite flags) bit for bit those of K6 (ritz / reuse_power); the residual estimate
    of the first t columns vs K7e and numpy."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(n + k + t)
    u = o.round_to(rng.standard_normal((n, k)), ufmt)
    w = rng.standard_normal((n, k)) * 3.0
    w = w if wfmt == F64 else o.round_to(w, wfmt)
    y = rng.standard_normal((k, k))
    lam = rng.uniform(0.5, 2.0, k) * rng.choice([-1, 1], k)
    U, W = _blk(p, u, ufmt), _blk(p, w, wfmt)
    Y = torch.tensor(np.ascontiguousarray(y.T), device="cuda")
    r_dev = torch.tensor([rv], dtype=torch.int32, device="cuda")
    vals = torch.tensor(lam, device="cuda")
    fl = torch.zeros(2, dtype=torch.int32, device="cuda")
    cm = torch.zeros(r_max, dtype=torch.float64, device="cuda")
    U64, Xu, Xw, est = ops.restart(U, W, Y, k, r_dev, r_max, want64=True, xu_fmt=p.FpFormat(xfmt), flags_u=fl[0:1],
                                   xw_fmt=p.FpFormat(xfmt), colmax=cm, flags_w=fl[1:2], vals=vals, t=t)
    R64, RX = ops.ritz(U, Y, k, r_dev, r_max, 1.0, want64=True, x_fmt=p.FpFormat(xfmt))
    cm2 = torch.zeros(r_max, dtype=torch.float64, device="cuda")
    RW = ops.reuse_power(W, Y, k, r_dev, r_max, p.FpFormat(xfmt), cm2)
    assert torch.equal(U64.t[:r_max, :n], R64.t[:r_max, :n])
    assert torch.equal(Xu.t[:r_max, :n], RX.t[:r_max, :n])
    assert torch.equal(Xw.t[:r_max, :n], RW.t[:r_max, :n])
    assert torch.equal(cm, cm2)
    assert not fl.any()
    if t == 0:
        assert est is None
        return
    ref_dev = ops.residual_estimate(U, W, Y, k, vals, r_dev, min(t, r_max)).cpu().numpy()
    got = est.cpu().numpy()
    tv = min(t, rv)
    d = w @ y[:, :tv] - (u @ y[:, :tv]) * lam[None, :tv]
    ref = np.sqrt(np.sum(d * d, axis=0)) / np.abs(lam[:tv])
    np.testing.assert_allclose(got[:tv], ref, rtol=1e-11)
    np.testing.assert_allclose(got[:tv], ref_dev[:tv], rtol=1e-13)
    assert not got[tv:].any()


@pytest.mark.parametrize("fmt,rows,cols,r,rv", [(BF16, 300, 20000, 64, 64), (BF16, 1000, 1000, 100, 90),
                                                (F16, 257, 3001, 7, 7), (FP8, 640, 5000, 33, 20),
                                                (BF16, 129, 16384, 32, 32)])
def test_residual_ozaki_vs_fp64(ofrr_gpu, oracle, fmt, rows, cols, r, rv):
    """K7 on the int8 tensor cores (Ozaki digit planes) vs numpy fp64: ||A x_j - s_j y_j|| /
    s_j for rectangular A (several K chunks, padded tiles, two column passes, r_dev < r)."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(rows + cols + r)
    a = o.round_to(rng.standard_normal((rows, cols)) * np.exp(rng.uniform(-3, 3, (rows, 1))), fmt)
    a = np.where(np.abs(a) > 400, 0.0, a)
    x = rng.standard_normal((cols, r))
    y = rng.standard_normal((rows, r))
    s = np.abs(rng.standard_normal(r)) + 0.1
    A = _op(p, a, fmt)
    X = _blk(p, x, F64)
    Yb = _blk(p, y, F64)
    res = torch.zeros(r, dtype=torch.float64, device="cuda")
    r_dev = torch.tensor([rv], dtype=torch.int32, device="cuda")
    ops.residual_pair(A, False, X, Yb, torch.tensor(s, device="cuda"), r_dev, r, res, accumulate_max=0)
    ref = np.linalg.norm(a @ x[:, :rv] - y[:, :rv] * s[None, :rv], axis=0) / s[:rv]
    got = res.cpu().numpy()
    np.testing.assert_allclose(got[:rv], ref, rtol=1e-11)
    assert not got[rv:].any()


def test_residual_ozaki_tiny_residuals(ofrr_gpu, oracle):
    """FP64-class accuracy where it matters: exact (fp64 eigh) eigenpairs of a bf16 matrix
    have residuals ~1e-15; the int8-digit product must not add more than ~1e-12."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(5)
    n = 1500
    a = rng.standard_normal((n, n))
    a = o.round_to((a + a.T) / 2, BF16)
    w, v = np.linalg.eigh(a)
    sel = np.argsort(-np.abs(w))[:48]
    lam, vec = w[sel], v[:, sel]
    A = _op(p, a, BF16)
    V = _blk(p, vec, F64)
    res = ops.residual_eig(A, V, torch.tensor(lam, device="cuda"), None, 48).cpu().numpy()
    ref = np.linalg.norm(a @ vec - vec * lam[None, :], axis=0) / np.abs(lam)
    assert np.all(ref < 1e-13)
    assert np.all(np.abs(res - ref) < 2e-12), np.max(np.abs(res - ref))


@pytest.mark.parametrize("n", [1024, 1000])
def test_generator_bitwise(ofrr_gpu, oracle, n):
    """K8 evaluates the synthetic matrix bit for bit like the host formula."""
    p, o = ofrr_gpu, oracle
    lam = p.geometric_spectrum(n, 10, 20)
    for fmt in (F64, BF16):
        m, f = p.synthetic_symmetric(lam, p.FpFormat(fmt), seed=5)
        got = m.data
        ref = o.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, fmt)
        np.testing.assert_array_equal(got, ref)
    # the spectrum is the prescribed one
    ev = np.sort(np.linalg.eigvalsh(o.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, F64)))[::-1]
    np.testing.assert_allclose(ev[:50], lam[:50], atol=1e-13)


@pytest.mark.parametrize("shape", [(2048, 2048, 64), (1000, 3000, 20), (4096, 1024, 85), (1024, 2048, 128), (700, 640, 200),
                                   (640, 512, 128), (100, 300, 90)])
def test_gemm_split_fp32_block_vs_fp64(ofrr_gpu, oracle, shape):
    """K1 split mode: bf16 A times an fp32 block via three bf16 slices is fp32-accurate."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rows, cols, k = shape
    rng = np.random.default_rng(rows + k)
    a = o.round_to(rng.standard_normal((rows, cols)), BF16)
    x = o.round_to(rng.standard_normal((cols, k)), F32)
    A = _op(p, a, BF16)
    X = _blk(p, x, F32)
    W = ops.new_block(rows, k, p.FpFormat.F32, A.device)
    colmax = torch.zeros(k, dtype=torch.float64, device=A.device)
    ops.gemm_av(A, X, W, colmax=colmax)
    got = _host(W)
    exact = a @ x
    bound = 2e-6 * (np.abs(a) @ np.abs(x)) + 1e-30
    assert np.all(np.abs(got - exact) <= bound), np.max(np.abs(got - exact) / bound)
    np.testing.assert_array_equal(colmax.cpu().numpy(), np.max(np.abs(got), axis=0))


@pytest.mark.parametrize("n,k,fmt", [(1000, 20, F64), (16384, 64, BF16), (333, 7, F16), (5000, 33, F32)])
def test_start_block_matches_numpy(ofrr_gpu, oracle, n, k, fmt):
    """X0 on the device == numpy default_rng(seed).random((n, k)) rounded (ofrr/driver.py:97-99)."""
    import torch
    from paper_2505_00281_b200 import ops
    for seed in (0, 2, 20240901):
        X = ops.start_block(seed, n, k, ofrr_gpu.FpFormat(fmt), torch.device("cuda"))
        ref = oracle.round_to(np.random.default_rng(seed).random((n, k)), fmt)
        np.testing.assert_array_equal(_host(X), ref)


def _exact_rows_dot(a, x):
    """A X with every product and sum exact (A entries and X entries are floats; the sum of
    exact products is formed in fp64 twice-compensated: a 2Sum/2Prod dot, error << 1 ulp)."""
    import math
    out = np.empty((a.shape[0], x.shape[1]))
    for j in range(x.shape[1]):
        for i in range(a.shape[0]):
            out[i, j] = math.fsum(a[i] * x[:, j])      # exact rounding of the exact sum of exact products
    return out


@pytest.mark.parametrize("case", ["heads", "tails", "full"])
def test_ozaki_heads_and_tails(ofrr_gpu, oracle, case):
    """K7z's 3-digit heads of A + exact fp64 tails (oz.cu, k_oz_rowscale) against exact products.

    heads: entries within 2^15 of their row maximum -> no tails (pure 15-digit-product path);
    tails: a few entries per row far below the maximum -> listed tails, still the head path;
    full:  rows with more tails than the per-row list holds -> all six digit planes.
    Every case must be FP64-accurate: |W - AX| <= 2^-44 |A||X| + 4 ulp (the digit products with
    p + q >= 6 are dropped: ~2^-46 per term, as in the six-digit scheme)."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng({"heads": 1, "tails": 2, "full": 3}[case])
    rows, cols, k = 300, 3000, 40
    a = rng.uniform(0.5, 1.0, (rows, cols)) * rng.choice([-1.0, 1.0], (rows, cols))
    if case == "tails":
        for i in range(rows):                        # 0..5 tiny entries per row
            j = rng.choice(cols, size=i % 6, replace=False)
            a[i, j] *= 2.0 ** rng.uniform(-40, -16, j.size)
    elif case == "full":
        a *= 2.0 ** rng.uniform(-30, 0, (rows, cols))   # wide range: most entries have tails
    a = o.round_to(a * np.exp(rng.uniform(-2, 2, (rows, 1))), BF16)
    x = rng.standard_normal((cols, k))
    A = _op(p, a, BF16)
    oz = ops.OzakiOperator(A)
    full, tails = oz.info()
    assert full == (case == "full"), (full, tails)
    if case == "heads":
        assert tails == 0
    if case == "tails":
        assert tails > 0
    X = _blk(p, x, F64)
    W = ops.new_block(rows, k, p.FpFormat.F64, torch.device("cuda"))
    ops.gemm_av(A, X, W, oz=oz)
    got = W.to_numpy_f64()
    ref = _exact_rows_dot(a, x)
    bound = 2.0 ** -44 * (np.abs(a) @ np.abs(x)) + 4 * np.spacing(np.abs(ref))
    if case == "full":
        # six digits on the 46-bit window below each row's maximum: the truncated digit
        # products weigh ~2^-40 of max|a_i.| sum|x| (the round-1 scheme's accuracy)
        bound = 2.0 ** -40 * np.max(np.abs(a), axis=1)[:, None] * np.sum(np.abs(x), axis=0)[None, :]
    assert np.all(np.abs(got - ref) <= bound), np.max(np.abs(got - ref) / bound)


@pytest.mark.parametrize("fmt", [BF16, F16])
def test_ozaki_tmem_kernel_large(ofrr_gpu, oracle, monkeypatch, fmt):
    """The heads kernel with the digit planes in TMEM (k_ozk_ts) at a size where every CTA runs
    ~50 k-blocks (all rings wrap many times): bitwise equal to the shared-memory kernel
    (k_ozk_gemm, same integer digit products and the same fp64 level sums), bitwise repeatable,
    and within 2^-44 |A||X| of an FP64 product."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(5)
    rows, cols, k = 4000, 16000, 64
    a = o.round_to(rng.standard_normal((rows, cols)) * np.exp(rng.uniform(-3, 3, (rows, 1))), fmt)
    x = rng.standard_normal((cols, k))
    A = _op(p, a, fmt)
    oz = ops.OzakiOperator(A)
    assert oz.info()[0] == 0
    X = _blk(p, x, F64)
    outs = []
    for flag in ("1", "1", "1", "0"):
        monkeypatch.setenv("OFRR_OZK_TMEM_A", flag)
        W = ops.new_block(rows, k, p.FpFormat.F64, torch.device("cuda"))
        ops.gemm_av(A, X, W, oz=oz)
        torch.cuda.synchronize()
        outs.append(W.to_numpy_f64())
    for w in outs[1:]:
        np.testing.assert_array_equal(outs[0], w)
    ref = (torch.as_tensor(a, device="cuda") @ torch.as_tensor(x, device="cuda")).cpu().numpy()
    mag = np.abs(a) @ np.abs(x)
    assert np.all(np.abs(outs[0] - ref) <= (2.0 ** -44 + cols * 2.0 ** -53) * mag)
    # the lite tier (shared-memory kernel, 128-column passes): repeatable, ~2^-30
    lite = []
    for _ in range(2):
        W = ops.new_block(rows, k, p.FpFormat.F64, torch.device("cuda"))
        ops.gemm_av(A, X, W, oz=oz, levels=4)
        torch.cuda.synchronize()
        lite.append(W.to_numpy_f64())
    np.testing.assert_array_equal(lite[0], lite[1])
    assert np.all(np.abs(lite[0] - ref) <= 2.0 ** -26 * mag)


def test_ozaki_lite_levels(ofrr_gpu, oracle):
    """ofrr_ozaki_gemm_levels(levels=4): the digit products with p + q < 4 (128-column passes),
    ~2^-30 of |A||X| per term; levels=6 stays FP64-accurate on the same inputs."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(44)
    rows, cols, k = 500, 4000, 100
    a = o.round_to(rng.standard_normal((rows, cols)), BF16)
    x = rng.standard_normal((cols, k))
    A = _op(p, a, BF16)
    oz = ops.OzakiOperator(A)
    X = _blk(p, x, F64)
    ref = _exact_rows_dot(a, x)
    mag = np.abs(a) @ np.abs(x)
    for levels, rel in ((3, 2.0 ** -18), (4, 2.0 ** -26), (5, 2.0 ** -34), (6, 2.0 ** -44)):
        W = ops.new_block(rows, k, p.FpFormat.F64, torch.device("cuda"))
        ops.gemm_av(A, X, W, oz=oz, levels=levels)
        err = np.abs(W.to_numpy_f64() - ref)
        assert np.all(err <= rel * mag + 4 * np.spacing(np.abs(ref))), (levels, np.max(err / mag))
    assert np.max(err / mag) < 2.0 ** -44


def test_gemm_split_two_slices(ofrr_gpu, oracle):
    """fp32 block on the bf16 tensor cores with 2 slices (the full-f32-lite rung): the block
    carried to a 16-bit significand (x_hi + x_mid), exact products, fp32 sums."""
    import torch
    from paper_2505_00281_b200 import ops
    p, o = ofrr_gpu, oracle
    rng = np.random.default_rng(12)
    rows, cols, k = 700, 3000, 96
    a = o.round_to(rng.standard_normal((rows, cols)), BF16)
    x = o.round_to(rng.standard_normal((cols, k)), F32)
    A = _op(p, a, BF16)
    X = _blk(p, x, F32)
    hi = o.round_to(x, BF16)
    x2 = hi + o.round_to(x - hi, BF16)                  # what two slices carry
    mag = np.abs(a) @ np.abs(x)
    for levels, xr, rel in ((4, x2, 2.0 ** -20), (6, x, 2.0 ** -20)):
        W = ops.new_block(rows, k, p.FpFormat.F32, torch.device("cuda"))
        ops.gemm_av(A, X, W, levels=levels)
        assert np.all(np.abs(W.to_numpy_f64() - a @ xr) <= rel * mag), levels
    assert np.max(np.abs(a @ x2 - a @ x) / mag) > 2.0 ** -24      # the two variants differ
