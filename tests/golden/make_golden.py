"""Generate the golden vectors that pin the oracle (and, through it, the GPU path).

Runs the REFERENCE package itself (imported read-only from /root/reference/pkg/src,
pure-numpy kernel backend, which its own tests pin bit-identical to the compiled one:
tests/test_kernels_backends.py:21-85) on small seeded inputs and stores inputs and
outputs in tests/golden/golden.npz.  Only this script touches /root/reference; the
committed .npz travels to the GPU box.

    OFRR_PURE_PYTHON=1 python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("OFRR_PURE_PYTHON", "1")
sys.path.insert(0, REF)

import ofrr  # noqa: E402
from ofrr.basis import BasisMethod, hessenberg_basis  # noqa: E402
from ofrr.driver import IterConfig, subspace_iter_eig, subspace_iter_svd  # noqa: E402
from ofrr.matrix import DenseMatrix, KernelConfig, gaussian_kernel, sample_uniform_square  # noqa: E402
from ofrr.precision import (FULL_F32, FULL_F64, MIXED_HALF, NATIVE_F16, FpFormat, PrecisionPolicy,  # noqa: E402
                            mixed_gemm, round_to, scale_columns_inf)
from ofrr.projection import ofrr_eig, ofrr_svd  # noqa: E402
from ofrr.smallsolve import sym_def_gen_eig, sym_eig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
SEED = 20240901
POL = {"native-f16": NATIVE_F16, "mixed-half": MIXED_HALF, "full-f32": FULL_F32, "full-f64": FULL_F64,
       "tc-f16": PrecisionPolicy(FpFormat.F16, FpFormat.F32, FpFormat.F32)}


def main():
    g = {}
    rng = np.random.default_rng(SEED)
    # --- mixed_gemm (ofrr/precision.py:122-135) --------------------------------------
    for name, pol in POL.items():
        for (m, k, n) in ((7, 5, 4), (40, 33, 6)):
            a = round_to(rng.standard_normal((m, k)) * 3, pol.storage)
            b = round_to(rng.standard_normal((k, n)) * 3, pol.storage)
            key = f"gemm/{name}/{m}x{k}x{n}"
            g[key + "/a"], g[key + "/b"] = a, b
            for out in (FpFormat.F16, FpFormat.F32, FpFormat.F64):
                g[key + f"/out{int(out)}"] = mixed_gemm(a, b, pol, out)
    # --- scale_columns_inf (ofrr/precision.py:159-169) ------------------------------
    x = rng.standard_normal((30, 4)) * 50
    x[:, 2] = 0.0
    g["scale/x"] = x
    for name, pol in POL.items():
        g[f"scale/{name}"] = scale_columns_inf(round_to(x, pol.storage), pol)
    # --- hessenberg_basis (ofrr/basis.py:151-196) -----------------------------------
    hcases = {
        "f64_20x6": (rng.standard_normal((20, 6)), "full-f64"),
        "f16_25x8": (rng.standard_normal((25, 8)), "native-f16"),
        "mh_64x10": (rng.standard_normal((64, 10)), "mixed-half"),
        "f32_64x10": (rng.random((64, 10)), "full-f32"),
        "tc16_300x12": (rng.random((300, 12)), "tc-f16"),
        "dep_6x3": (np.column_stack([np.ones(6), np.ones(6), np.arange(6, dtype=float)]), "full-f64"),
        "ties_8x3": (np.ones((8, 3)) * np.array([1.0, 2.0, 3.0]) + np.eye(8, 3), "full-f64"),
    }
    for name, (xv, pname) in hcases.items():
        pol = POL[pname]
        xm = DenseMatrix(np.asfortranarray(round_to(xv, pol.storage)), pol.storage)
        for layout in ("left", "right"):
            fac = hessenberg_basis(xm, layout, pol)
            key = f"hess/{name}/{layout}"
            g[key + "/x"] = xm.data
            g[key + "/q"] = fac.q.data
            g[key + "/pivots"] = fac.pivots
            g[key + "/kept"] = fac.kept
            g[key + "/policy"] = np.array([int(pol.storage), int(pol.compute), int(pol.accumulate)])
    # --- small solves (ofrr/smallsolve.py) ------------------------------------------
    for n in (1, 2, 5, 12, 40):
        s = rng.standard_normal((n, n))
        s = (s + s.T) / 2
        r = sym_eig(s)
        g[f"symeig/{n}/s"], g[f"symeig/{n}/vals"], g[f"symeig/{n}/vecs"] = s, r.values, r.vectors
    for n in (2, 6, 15, 33):
        b = rng.standard_normal((n, n))
        b = (b + b.T) / 2
        rr = rng.standard_normal((n, n))
        mm = rr.T @ rr + 0.5 * np.eye(n)
        r = sym_def_gen_eig(b, mm)
        g[f"geneig/{n}/b"], g[f"geneig/{n}/m"] = b, mm
        g[f"geneig/{n}/vals"], g[f"geneig/{n}/vecs"] = r.values, r.vectors
    # rank-deficient M (tests/test_smallsolve.py:84-93)
    n = 6
    rr = rng.standard_normal((n, n - 1))
    mm = rr @ rr.T
    b = rng.standard_normal((n, n))
    b = (b + b.T) / 2
    r = sym_def_gen_eig(b, mm)
    g["geneig/rankdef/b"], g["geneig/rankdef/m"] = b, mm
    g["geneig/rankdef/vals"], g["geneig/rankdef/vecs"] = r.values, r.vectors
    # --- ofrr_eig (ofrr/projection.py:75-87) ----------------------------------------
    s = rng.standard_normal((30, 30))
    s = (s + s.T) / 2
    u = rng.standard_normal((30, 5))
    for pname in ("full-f64", "full-f32"):
        pol = POL[pname]
        a = DenseMatrix(round_to(s, pol.storage), FpFormat.F64)
        uu = DenseMatrix(round_to(u, pol.storage), pol.storage)
        rs = ofrr_eig(a, uu, pol)
        g[f"ofrreig/{pname}/a"], g[f"ofrreig/{pname}/u"] = a.data, uu.data
        g[f"ofrreig/{pname}/vals"], g[f"ofrreig/{pname}/vecs"] = rs.values, rs.vectors.data
    # --- drivers (ofrr/driver.py) ----------------------------------------------------
    pts = sample_uniform_square(120, float(np.sqrt(120)), 42)
    kern = gaussian_kernel(KernelConfig(1.0, 10.0, 0.01, pts), FpFormat.F64)
    for pname in ("full-f64", "full-f32", "tc-f16"):
        pol = POL[pname]
        a = DenseMatrix(round_to(kern.data, pol.storage), FpFormat.F64)
        for method in ("hess-l", "hess-r"):
            cfg = IterConfig(k=20, m=3, iter=2, basis_method=BasisMethod(method), projection="ofrr",
                             policy=pol, seed=2)
            rs = subspace_iter_eig(a, cfg)
            key = f"driver_eig/{pname}/{method}"
            g[key + "/a"] = a.data
            g[key + "/vals"], g[key + "/vecs"], g[key + "/res"] = rs.values, rs.vectors.data, rs.residuals
    g["driver_eig/exact"] = np.sort(np.linalg.eigvalsh(kern.data))[::-1]
    pts1 = sample_uniform_square(100, 10.0, 7)
    pts2 = sample_uniform_square(40, 10.0, 8)
    cross = gaussian_kernel(KernelConfig(0.2, 10.0, 0.0, pts1, cross_points=pts2), FpFormat.F64)
    for pname in ("full-f64", "full-f32"):
        pol = POL[pname]
        a = DenseMatrix(round_to(cross.data, pol.storage), FpFormat.F64)
        cfg = IterConfig(k=10, m=6, iter=1, basis_method=BasisMethod.HESS_LEFT, projection="ofrr", policy=pol,
                         seed=9)
        rs = subspace_iter_svd(a, cfg)
        key = f"driver_svd/{pname}"
        g[key + "/a"] = a.data
        g[key + "/vals"], g[key + "/u"], g[key + "/v"], g[key + "/res"] = (
            rs.values, rs.vectors.data, rs.right_vectors.data, rs.residuals)
    g["driver_svd/exact"] = np.linalg.svd(cross.data, compute_uv=False)
    # ofrr_svd on a random case (ofrr/projection.py:99-133)
    a = rng.standard_normal((12, 9))
    u = rng.standard_normal((12, 4))
    v = rng.standard_normal((9, 4))
    rs = ofrr_svd(DenseMatrix(a, FpFormat.F64), DenseMatrix(u, FpFormat.F64), DenseMatrix(v, FpFormat.F64), FULL_F64)
    g["ofrrsvd/a"], g["ofrrsvd/u"], g["ofrrsvd/v"] = a, u, v
    g["ofrrsvd/vals"], g["ofrrsvd/uu"], g["ofrrsvd/vv"] = rs.values, rs.vectors.data, rs.right_vectors.data
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1024:.1f} KiB, "
          f"reference backend = {ofrr.active_backend}")


if __name__ == "__main__":
    main()
