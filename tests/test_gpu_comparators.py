"""The classical comparators on the GPU: Gram-Schmidt builders
(csrc/gs.cu) against the oracle / the reference's golden runs (golden_gs.npz), classical
Rayleigh-Ritz, and the drivers with those bases and projections."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EPS = {0: 2.0 ** -11, 1: 2.0 ** -24, 2: 2.0 ** -53}
POLS = {"native-f16": (0, 0, 0), "mixed-half": (0, 0, 1), "full-f32": (1, 1, 1), "full-f64": (2, 2, 2)}


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden_gs.npz")))


def _run_gs(p, x, pname, meth):
    import torch
    from paper_2505_00281_b200 import ops
    pol = p.POLICY_PRESETS[pname]
    X = ops.block_from_host(x, pol.storage, torch.device("cuda"))
    h = ops.orthonormalize(X, meth, pol.storage, pol.compute, pol.accumulate, pol.drop_tol)
    nk = int(h.n_kept.item())
    return h.Q.to_numpy_f64(nk), h.kept.cpu().numpy()[: x.shape[1]].astype(bool)


@pytest.mark.parametrize("case", ["rand_40x6", "pos_64x10", "ill_50x8", "dep_12x4"])
@pytest.mark.parametrize("pname", list(POLS))
@pytest.mark.parametrize("meth", ["mgs-l", "mgs-r", "cgs", "cgs2"])
def test_gram_schmidt_vs_reference(ofrr_gpu, gold, case, pname, meth):
    """Same kept columns as the reference; the basis equal to the reference's to the
    accumulate format's rounding (parallel sums) -- scaled by the input's conditioning
    for the ill-conditioned case; orthogonality no worse than ~10x the reference's."""
    p = ofrr_gpu
    base = f"gs/{case}/{pname}/{meth}"
    x = gold[base + "/x"]
    q, kept = _run_gs(p, x, pname, meth)
    qr, keptr = gold[base + "/q"], gold[base + "/kept"]
    s, c, a = POLS[pname]
    if case == "dep_12x4" and s != 2:
        # an exactly dependent column in low precision: the drop test sits on rounding noise
        assert kept.sum() in (keptr.sum(), keptr.sum() - 1, keptr.sum() + 1)
        return
    np.testing.assert_array_equal(kept, keptr)
    cond = 1e7 if case == "ill_50x8" else 1.0
    tol = max(EPS[a], EPS[s]) * 64 * cond
    assert np.max(np.abs(q - qr)) <= max(tol, 4 * EPS[s]), np.max(np.abs(q - qr))
    loss = np.abs(q.T @ q - np.eye(q.shape[1])).max()
    ref_loss = np.abs(qr.T @ qr - np.eye(qr.shape[1])).max()
    assert loss <= 10 * ref_loss + 64 * EPS[s], (loss, ref_loss)


@pytest.mark.parametrize("pname", ["full-f64", "full-f32"])
def test_rr_eig_vs_reference(ofrr_gpu, gold, pname):
    p = ofrr_gpu
    pol = p.POLICY_PRESETS[pname]
    rs = p.rr_eig(p.DenseMatrix(gold[f"rreig/{pname}/a"], p.FpFormat.F64),
                  p.DenseMatrix(gold[f"rreig/{pname}/q"], pol.storage), pol)
    rt = 1e-10 if pname == "full-f64" else 2e-5
    np.testing.assert_allclose(rs.values, gold[f"rreig/{pname}/vals"], rtol=rt, atol=rt)
    np.testing.assert_allclose(rs.vectors.data, gold[f"rreig/{pname}/vecs"], rtol=1e3 * rt, atol=1e3 * rt)


@pytest.mark.parametrize("pname", ["full-f64", "full-f32"])
@pytest.mark.parametrize("meth,proj", [("mgs-l", "rr"), ("cgs2", "rr"), ("mgs-r", "ofrr"), ("cgs", "rr")])
def test_driver_classical_vs_reference(ofrr_gpu, gold, pname, meth, proj):
    """subspace_iter_eig with the Gram-Schmidt bases (and classical RR) vs the reference's
    own runs: the north-star criteria per pair."""
    p = ofrr_gpu
    pol = p.POLICY_PRESETS[pname]
    a = p.DenseMatrix(gold[f"driver/{pname}/a"], p.FpFormat.F64)
    cfg = p.IterConfig(k=20, m=3, iter=2, basis_method=p.BasisMethod(meth), projection=proj, policy=pol, seed=2)
    rs = p.subspace_iter_eig(a, cfg)
    key = f"driver/{pname}/{meth}/{proj}"
    exact = gold["driver/exact"] if pname == "full-f64" else np.sort(np.linalg.eigvalsh(gold[f"driver/{pname}/a"]))[::-1]
    top = 6
    ref_err = np.abs(gold[key + "/vals"][:top] - exact[:top]) / np.abs(exact[:top])
    err = np.abs(rs.values[:top] - exact[:top]) / np.abs(exact[:top])
    assert np.all(err <= np.maximum(10 * ref_err, 1e-6)), (err, ref_err)
    # per pair: within 2x of the reference's residual, plus (fp32 policy) the fp32 rounding floor
    # of the pair -- u |lambda_1| / |lambda_i| times a small constant: at that floor both runs'
    # residuals are rounding noise of their own (different) summation orders
    floor = 0.0 if pname == "full-f64" else 8 * 2.0 ** -24 * np.abs(exact[0]) / np.abs(exact[:top])
    assert np.all(rs.residuals[:top] <= 2 * gold[key + "/res"][:top] + floor + 1e-13), (
        rs.residuals[:top], gold[key + "/res"][:top], floor)


def test_driver_svd_classical_vs_reference(ofrr_gpu, gold):
    p = ofrr_gpu
    a = p.DenseMatrix(gold["driver_svd/a"], p.FpFormat.F64)
    cfg = p.IterConfig(k=10, m=6, iter=1, basis_method=p.BasisMethod.CGS2, projection="rr", policy=p.FULL_F64,
                       seed=9)
    rs = p.subspace_iter_svd(a, cfg)
    exact = gold["driver_svd/exact"]
    top = 5
    ref_err = np.abs(gold["driver_svd/vals"][:top] - exact[:top]) / exact[:top]
    err = np.abs(rs.values[:top] - exact[:top]) / exact[:top]
    assert np.all(err <= np.maximum(10 * ref_err, 1e-6)), (err, ref_err)
    assert np.all(rs.residuals[:top] <= 2 * gold["driver_svd/res"][:top] + 1e-13)


def test_rr_svd_vs_reference(ofrr_gpu, gold):
    p = ofrr_gpu
    rs = p.rr_svd(p.DenseMatrix(gold["rrsvd/a"], p.FpFormat.F64), p.DenseMatrix(gold["rrsvd/u"], p.FpFormat.F64),
                  p.DenseMatrix(gold["rrsvd/v"], p.FpFormat.F64), p.FULL_F64)
    np.testing.assert_allclose(rs.values, gold["rrsvd/vals"], rtol=1e-10)
    # singular vectors up to a joint sign per triplet
    for j in range(len(rs.values)):
        u, ur = rs.vectors.data[:, j], gold["rrsvd/uu"][:, j]
        sgn = np.sign(u @ ur)
        np.testing.assert_allclose(sgn * u, ur, atol=1e-8)
        np.testing.assert_allclose(sgn * rs.right_vectors.data[:, j], gold["rrsvd/vv"][:, j], atol=1e-8)
