"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and against the reference's own known answers.
CPU only (no GPU)."""

import math

import numpy as np
import pytest

POLS = {"native-f16": (0, 0, 0), "mixed-half": (0, 0, 1), "full-f32": (1, 1, 1), "full-f64": (2, 2, 2),
        "tc-f16": (0, 1, 1)}


def pol(o, name):
    s, c, a = POLS[name]
    return o.Pol(s, c, a)


def test_round_known_answers(oracle):
    o = oracle
    # tests/test_precision.py:55-69
    assert o.round_to(np.array([1.0 + 2.0**-11]), o.F16)[0] == 1.0
    assert o.round_to(np.array([7.0e4]), o.F16)[0] == np.inf
    assert o.round_to(np.array([-7.0e4]), o.F16)[0] == -np.inf
    assert o.round_to(np.array([65504.0]), o.F16)[0] == 65504.0
    assert o.round_to(np.array([2.0**-24]), o.F16)[0] == 2.0**-24
    assert o.round_to(np.array([2.0**-26]), o.F16)[0] == 0.0


@pytest.mark.parametrize("fmt", ["f16", "f32", "bf16"])
def test_round_matches_bit_simulation(oracle, fmt):
    """Integer-mantissa simulation in the style of the reference's fp_oracle.py:22-36."""
    o = oracle
    p, emin, mx = {"f16": (11, -14, 65504.0), "f32": (24, -126, float.fromhex("0x1.fffffep+127")),
                   "bf16": (8, -126, float.fromhex("0x1.fep127"))}[fmt]
    code = {"f16": o.F16, "f32": o.F32, "bf16": o.BF16}[fmt]

    def sim(x):
        if x == 0.0 or math.isnan(x) or math.isinf(x):
            return x
        mag = abs(x)
        _, e = math.frexp(mag)
        q = max(e - p, emin - p + 1)
        r = math.ldexp(float(round(math.ldexp(mag, -q))), q)
        if r > mx:
            r = math.inf
        return -r if x < 0 else r

    rng = np.random.default_rng(7)
    lo = -140 if fmt != "f16" else -30
    x = np.sign(rng.standard_normal(4000)) * 2.0 ** rng.uniform(lo, 20 if fmt == "f16" else 120, 4000)
    got = o.round_to(x, code)
    for xi, gi in zip(x, got):
        assert gi == sim(float(np.float32(xi))) or gi == sim(xi), xi


def test_mixed_dot_known_answers(oracle):
    o = oracle
    x = np.ones(2049)
    assert o.mixed_dot(x, x, o.F16, o.F16) == 2048.0     # tests/test_precision.py:97-99
    assert o.mixed_dot(x, x, o.F16, o.F32) == 2049.0     # :101-103


@pytest.mark.parametrize("name", list(POLS))
def test_gemm_matches_reference_bitwise(oracle, golden, name):
    o = oracle
    p = pol(o, name)
    for shape in ("7x5x4", "40x33x6"):
        key = f"gemm/{name}/{shape}"
        a, b = golden[key + "/a"], golden[key + "/b"]
        for out in (o.F16, o.F32, o.F64):
            got = o.mixed_gemm(a, b, p.compute, p.accumulate, out)
            np.testing.assert_array_equal(got, golden[key + f"/out{out}"])


@pytest.mark.parametrize("name", list(POLS))
def test_scale_columns_bitwise(oracle, golden, name):
    o = oracle
    p = pol(o, name)
    x = o.round_to(golden["scale/x"], p.storage)
    np.testing.assert_array_equal(o.scale_columns_inf(x, p), golden[f"scale/{name}"])


@pytest.mark.parametrize("case", ["f64_20x6", "f16_25x8", "mh_64x10", "f32_64x10", "tc16_300x12", "dep_6x3",
                                  "ties_8x3"])
def test_hessenberg_bitwise(oracle, golden, case):
    o = oracle
    for layout in ("left", "right"):
        key = f"hess/{case}/{layout}"
        s, c, a = golden[key + "/policy"]
        q, piv, kept = o.hessenberg_basis(golden[key + "/x"], o.Pol(int(s), int(c), int(a)))
        np.testing.assert_array_equal(q, golden[key + "/q"])
        np.testing.assert_array_equal(piv, golden[key + "/pivots"])
        np.testing.assert_array_equal(kept, golden[key + "/kept"])


def test_hessenberg_is_gepp(oracle):
    """tests/test_basis.py:100-113: Hessenberg basis = P'L of row-pivoted LU."""
    import scipy.linalg
    o = oracle
    rng = np.random.default_rng(5)
    for _ in range(10):
        n = int(rng.integers(4, 40))
        k = int(rng.integers(2, min(n, 16) + 1))
        a = rng.standard_normal((n, k))
        q, piv, _ = o.hessenberg_basis(a, o.FULL_F64)
        p, l, _ = scipy.linalg.lu(a)
        pl = p @ l
        np.testing.assert_allclose(q, pl[:, : q.shape[1]], atol=1e-12)
        np.testing.assert_array_equal(piv, np.argmax(p, axis=0)[: piv.size])


@pytest.mark.parametrize("n", [1, 2, 5, 12, 40])
def test_sym_eig_matches_reference(oracle, golden, n):
    o = oracle
    vals, vecs = o.sym_eig(golden[f"symeig/{n}/s"])
    np.testing.assert_array_equal(vals, golden[f"symeig/{n}/vals"])
    np.testing.assert_array_equal(vecs, golden[f"symeig/{n}/vecs"])


@pytest.mark.parametrize("n", ["2", "6", "15", "33", "rankdef"])
def test_gen_eig_matches_reference(oracle, golden, n):
    o = oracle
    vals, vecs = o.sym_def_gen_eig(golden[f"geneig/{n}/b"], golden[f"geneig/{n}/m"])
    np.testing.assert_allclose(vals, golden[f"geneig/{n}/vals"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(vecs, golden[f"geneig/{n}/vecs"], rtol=1e-10, atol=1e-11)


@pytest.mark.parametrize("pname", ["full-f64", "full-f32"])
def test_ofrr_eig_matches_reference(oracle, golden, pname):
    o = oracle
    rs = o.ofrr_eig(golden[f"ofrreig/{pname}/a"], golden[f"ofrreig/{pname}/u"], pol(o, pname))
    np.testing.assert_allclose(rs.values, golden[f"ofrreig/{pname}/vals"], rtol=1e-12)
    np.testing.assert_allclose(rs.vectors, golden[f"ofrreig/{pname}/vecs"], rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("pname", ["full-f64", "full-f32", "tc-f16"])
def test_driver_eig_matches_reference(oracle, golden, pname):
    o = oracle
    key = f"driver_eig/{pname}/hess-l"
    rs = o.subspace_iter_eig(golden[key + "/a"], k=20, m=3, iters=2, pol=pol(o, pname), seed=2)
    np.testing.assert_allclose(rs.values, golden[key + "/vals"], rtol=1e-12)
    np.testing.assert_allclose(rs.residuals, golden[key + "/res"], rtol=1e-6, atol=1e-14)
    # hess-l and hess-r are the same algorithm (tests/test_basis.py:92-98)
    np.testing.assert_array_equal(golden[key + "/vals"], golden[f"driver_eig/{pname}/hess-r/vals"])


def test_driver_eig_fp64_accuracy(golden):
    """tests/test_driver.py:63-70: OFRR-Hess converges to 1e-10 on the kernel matrix."""
    ref = golden["driver_eig/exact"]
    vals = golden["driver_eig/full-f64/hess-l/vals"]
    assert np.all(np.abs(vals[:6] - ref[:6]) / ref[:6] < 1e-10)


@pytest.mark.parametrize("pname", ["full-f64", "full-f32"])
def test_driver_svd_matches_reference(oracle, golden, pname):
    o = oracle
    key = f"driver_svd/{pname}"
    rs = o.subspace_iter_svd(golden[key + "/a"], k=10, m=6, iters=1, pol=pol(o, pname), seed=9)
    np.testing.assert_allclose(rs.values, golden[key + "/vals"], rtol=1e-11)
    np.testing.assert_allclose(rs.residuals, golden[key + "/res"], rtol=1e-5, atol=1e-12)


def test_ofrr_svd_matches_reference(oracle, golden):
    o = oracle
    rs = o.ofrr_svd(golden["ofrrsvd/a"], golden["ofrrsvd/u"], golden["ofrrsvd/v"], o.FULL_F64)
    np.testing.assert_allclose(rs.values, golden["ofrrsvd/vals"], rtol=1e-12)
    np.testing.assert_allclose(rs.vectors, golden["ofrrsvd/uu"], rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(rs.right_vectors, golden["ofrrsvd/vv"], rtol=1e-9, atol=1e-10)


def test_rayleigh_quotient_known_answer(oracle):
    """tests/test_projection.py:71-75."""
    o = oracle
    rs = o.ofrr_eig(np.diag([3.0, 1.0]), np.array([[1.0], [1.0]]), o.FULL_F64)
    assert rs.values[0] == pytest.approx(2.0, abs=1e-14)
