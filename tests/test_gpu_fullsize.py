"""Full-size independent validation of the benched configurations (last
bullet): the answers of the C2 and C3 bench solves are checked by test-only FP64 computations
that share nothing with the product's kernels.

* C2 (16384^2, top-32, k=64, full-f32 basis, tol 1e-2): all eigenvalues of the bf16-rounded A
  by ``torch.linalg.eigvalsh`` in FP64 (cuSOLVER), residuals by a plain FP64 ``A @ V``.
  Per pair: |theta_i - lambda_i| <= ||A v_i - theta_i v_i|| / ||v_i|| (the residual bound for
  a symmetric matrix), the reported residuals equal the independent ones to 1e-6 relative,
  and every residual of the top 32 is below tol.
* C3 (65536^2, top-64, k=128, the headline ladder to 1e-8): residuals by a row-blocked FP64
  product (A's bf16 rows widened exactly), per pair below 1e-8.  Values against the prescribed
  spectrum lambda_i = rho^i of the exact matrix A0 (A = round_bf16(A0)): by Weyl,
  |lambda_i(A) - rho^i| <= ||A - A0||_2, estimated by block power iteration on A - A0 (A0 x is
  applied exactly from its factors, matrix.py: s * FWHT(lam_p * FWHT(s * x)) / n plus the
  rank-2r term), times a safety factor of 2.  With ||A - A0||_2 ~ 1e-5 against consecutive gaps
  of ~3.5e-3, the check pins the returned pairs as the TOP 64, which a small residual alone
  does not.
"""
import numpy as np
import pytest
import torch

SEED = 20240901


def _fwht(x: torch.Tensor) -> torch.Tensor:
    """Unnormalised Walsh-Hadamard transform along dim 0 (Sylvester order, matrix._fwht)."""
    n = x.shape[0]
    y = x.reshape(n, -1)
    h = 1
    while h < n:
        y = y.reshape(n // (2 * h), 2, h, -1)
        y = torch.stack((y[:, 0] + y[:, 1], y[:, 0] - y[:, 1]), dim=1)
        h *= 2
    return y.reshape(x.shape)


def _exact_apply(f, x: torch.Tensor) -> torch.Tensor:
    """A0 x for the synthetic factors (FP64, no n x n matrix)."""
    dev = x.device
    s = torch.as_tensor(f.s, dtype=torch.float64, device=dev)[:, None]
    c = torch.as_tensor(f.c, dtype=torch.float64, device=dev)
    lam_p = _fwht(c[:, None])                         # FWHT(FWHT(lam_p) / n) = lam_p
    base = s * (_fwht(lam_p * _fwht(s * x)) / f.n)
    W = torch.as_tensor(f.Wf, dtype=torch.float64, device=dev)
    M = torch.as_tensor(f.Mf, dtype=torch.float64, device=dev)
    return base + W @ (M.T @ x) + M @ (W.T @ x)


def _apply_f64(A_op, x: torch.Tensor, block: int = 4096) -> torch.Tensor:
    """A x in FP64 from the device operator's rows (bf16 -> fp64 is exact)."""
    n = A_op.cols
    out = torch.empty((A_op.rows, x.shape[1]), dtype=torch.float64, device=x.device)
    for r0 in range(0, A_op.rows, block):
        r1 = min(A_op.rows, r0 + block)
        out[r0:r1] = A_op.t[r0:r1, :n].to(torch.float64) @ x
    return out


def _solve(p, cfg_name):
    import bench
    cfg = bench.CONFIGS[cfg_name]
    n, top, k = cfg["n"], cfg["top"], cfg["k"]
    lam = p.geometric_spectrum(n, top, k)
    A, f = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=SEED)
    icfg = bench.make_iter_config(p, cfg)
    st = p.RunStats()
    rs = p.subspace_iter_eig(A, icfg, stats=st)
    return cfg, A, f, lam, rs, st


def _independent_residuals(A_op, rs, top):
    dev = A_op.t.device
    V = torch.as_tensor(np.ascontiguousarray(rs.vectors.data[:, :top]), dtype=torch.float64, device=dev)
    th = torch.as_tensor(rs.values[:top], dtype=torch.float64, device=dev)
    R = _apply_f64(A_op, V) - V * th[None, :]
    rnorm = torch.linalg.vector_norm(R, dim=0)
    vnorm = torch.linalg.vector_norm(V, dim=0)
    return (rnorm / th.abs()).cpu().numpy(), rnorm.cpu().numpy(), vnorm.cpu().numpy()


@pytest.mark.gpu
def test_c2_bench_answer_independent_fp64(ofrr_gpu):
    p = ofrr_gpu
    cfg, A, f, lam, rs, st = _solve(p, "c2")
    top, tol = cfg["top"], cfg["tol"]
    assert st.converged
    op = A.device_operator(p.FpFormat.BF16)
    res, rnorm, vnorm = _independent_residuals(op, rs, top)
    # the product's FP64 residual report vs the independent FP64 product, per pair
    np.testing.assert_allclose(rs.residuals[:top], res, rtol=1e-6, atol=0)
    assert np.all(res < tol), res
    # every eigenvalue of the bf16 matrix (FP64, cuSOLVER)
    A64 = op.t[:, :cfg["n"]].to(torch.float64)
    ev = torch.linalg.eigvalsh(A64).flip(0)[:top].cpu().numpy()
    del A64
    bound = rnorm / vnorm * (1 + 1e-9) + 1e-13
    err = np.abs(rs.values[:top] - ev)
    assert np.all(err <= bound), (err, bound)
    # and the accuracy the values actually reach: quadratic in the residual down to the floor of
    # the full-f32 policy (W = A U summed in fp32: the Rayleigh quotient carries ~2^-23 sqrt(n)
    # relative noise, measured 7.7e-6 here)
    fp32_floor = 2.0 ** -23 * 128
    assert np.all(err / np.abs(ev) <= np.maximum(res ** 2 * 100, fp32_floor)), (err / np.abs(ev), res)


@pytest.mark.gpu
def test_c3_headline_answer_independent_fp64(ofrr_gpu):
    p = ofrr_gpu
    import bench
    cfg, A, f, lam, rs, st = _solve(p, bench.DEFAULT_CONFIG)          # the headline as benched
    top, tol, n = cfg["top"], cfg["tol"], cfg["n"]
    assert st.converged
    op = A.device_operator(p.FpFormat.BF16)
    res, rnorm, vnorm = _independent_residuals(op, rs, top)
    # both FP64-accurate: they agree to the FP64 floor of a 65536-term residual (~1e-13 relative
    # to |lambda|) -- the solve often ends far below tol, where that floor dominates
    np.testing.assert_allclose(rs.residuals[:top], res, rtol=1e-3, atol=2e-12)
    assert np.all(res < tol), res
    # ||A - A0||_2 by block power iteration (A0 exact from its factors)
    g = torch.Generator(device=op.t.device)
    g.manual_seed(7)
    X = torch.randn((n, 4), generator=g, dtype=torch.float64, device=op.t.device)
    est = 0.0
    for _ in range(12):
        X, _ = torch.linalg.qr(X)
        Y = _apply_f64(op, X) - _exact_apply(f, X)
        est = float(torch.linalg.matrix_norm(Y, ord=2))
        X = Y
    assert 0 < est < 1e-3, est
    exact = lam[:top]
    err = np.abs(rs.values[:top] - exact)
    bound = 2.0 * est + rnorm / vnorm
    assert np.all(err <= bound), (err.max(), bound.min())
    gaps = -np.diff(lam[:top + 1])
    assert np.all(bound < gaps / 2), "the bound must separate consecutive eigenvalues"
