"""Golden vectors for the classical comparators: the reference's own
Gram-Schmidt builders (ofrr/basis.py:65-148), classical Rayleigh-Ritz (ofrr/projection.py:
64-96) and the drivers with those bases, on small seeded inputs -> tests/golden/golden_gs.npz.
Runs the REFERENCE package read-only (pure-numpy backend); only this script touches
/root/reference.

    OFRR_PURE_PYTHON=1 python tests/golden/make_golden_gs.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("OFRR_PURE_PYTHON", "1")
sys.path.insert(0, REF)

from ofrr.basis import BasisMethod, orthonormalize  # noqa: E402
from ofrr.driver import IterConfig, subspace_iter_eig, subspace_iter_svd  # noqa: E402
from ofrr.matrix import DenseMatrix, KernelConfig, gaussian_kernel, sample_uniform_square  # noqa: E402
from ofrr.precision import FULL_F32, FULL_F64, MIXED_HALF, NATIVE_F16, FpFormat, round_to  # noqa: E402
from ofrr.projection import rr_eig, rr_svd  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_gs.npz")
POL = {"native-f16": NATIVE_F16, "mixed-half": MIXED_HALF, "full-f32": FULL_F32, "full-f64": FULL_F64}
METHODS = ("mgs-l", "mgs-r", "cgs", "cgs2")


def main():
    g = {}
    rng = np.random.default_rng(20250501)
    cases = {
        "rand_40x6": rng.standard_normal((40, 6)),
        "pos_64x10": rng.random((64, 10)),
        "dep_12x4": np.column_stack([np.arange(12.0), 2 * np.arange(12.0), np.ones(12), rng.standard_normal(12)]),
        "ill_50x8": rng.standard_normal((50, 8)) @ np.diag(10.0 ** -np.arange(8)),
    }
    for cname, xv in cases.items():
        for pname, pol in POL.items():
            x = DenseMatrix(np.asfortranarray(round_to(xv, pol.storage)), pol.storage)
            for meth in METHODS:
                key = f"gs/{cname}/{pname}/{meth}"
                try:
                    fac = orthonormalize(x, BasisMethod(meth), pol)
                    g[key + "/q"], g[key + "/kept"] = fac.q.data, fac.kept
                except Exception as e:                            # EmptyBasisError
                    g[key + "/error"] = np.array(type(e).__name__)
                g[key + "/x"] = x.data
    s = rng.standard_normal((30, 30))
    s = (s + s.T) / 2
    for pname in ("full-f64", "full-f32"):
        pol = POL[pname]
        a = DenseMatrix(round_to(s, pol.storage), FpFormat.F64)
        q = orthonormalize(DenseMatrix(round_to(rng.standard_normal((30, 5)), pol.storage), pol.storage),
                           BasisMethod.CGS2, pol).q
        rs = rr_eig(a, q, pol)
        g[f"rreig/{pname}/a"], g[f"rreig/{pname}/q"] = a.data, q.data
        g[f"rreig/{pname}/vals"], g[f"rreig/{pname}/vecs"] = rs.values, rs.vectors.data
    pts = sample_uniform_square(120, float(np.sqrt(120)), 42)
    kern = gaussian_kernel(KernelConfig(1.0, 10.0, 0.01, pts), FpFormat.F64)
    g["driver/exact"] = np.sort(np.linalg.eigvalsh(kern.data))[::-1]
    for pname in ("full-f64", "full-f32"):
        pol = POL[pname]
        a = DenseMatrix(round_to(kern.data, pol.storage), FpFormat.F64)
        g[f"driver/{pname}/a"] = a.data
        for meth, proj in (("mgs-l", "rr"), ("cgs2", "rr"), ("mgs-r", "ofrr"), ("cgs", "rr")):
            cfg = IterConfig(k=20, m=3, iter=2, basis_method=BasisMethod(meth), projection=proj, policy=pol, seed=2)
            rs = subspace_iter_eig(a, cfg)
            key = f"driver/{pname}/{meth}/{proj}"
            g[key + "/vals"], g[key + "/vecs"], g[key + "/res"] = rs.values, rs.vectors.data, rs.residuals
    pts1 = sample_uniform_square(100, 10.0, 7)
    pts2 = sample_uniform_square(40, 10.0, 8)
    cross = gaussian_kernel(KernelConfig(0.2, 10.0, 0.0, pts1, cross_points=pts2), FpFormat.F64)
    cfg = IterConfig(k=10, m=6, iter=1, basis_method=BasisMethod.CGS2, projection="rr", policy=FULL_F64, seed=9)
    rs = subspace_iter_svd(cross, cfg)
    g["driver_svd/a"] = cross.data
    g["driver_svd/vals"], g["driver_svd/res"] = rs.values, rs.residuals
    g["driver_svd/exact"] = np.linalg.svd(cross.data, compute_uv=False)
    a = rng.standard_normal((12, 9))
    u = orthonormalize(DenseMatrix(rng.standard_normal((12, 4)), FpFormat.F64), BasisMethod.CGS2, FULL_F64).q
    v = orthonormalize(DenseMatrix(rng.standard_normal((9, 4)), FpFormat.F64), BasisMethod.CGS2, FULL_F64).q
    rs = rr_svd(DenseMatrix(a, FpFormat.F64), u, v, FULL_F64)
    g["rrsvd/a"], g["rrsvd/u"], g["rrsvd/v"] = a, u.data, v.data
    g["rrsvd/vals"], g["rrsvd/uu"], g["rrsvd/vv"] = rs.values, rs.vectors.data, rs.right_vectors.data
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1024:.1f} KiB")


if __name__ == "__main__":
    main()
