"""Pin the oracle's restatement of the classical comparators against
the reference itself (tests/golden/make_golden_gs.py -> golden_gs.npz): the Gram-Schmidt
builders (ofrr/basis.py:65-148) and classical Rayleigh-Ritz (ofrr/projection.py:64-72)
bit for bit, the drivers with those bases to 1e-12.  CPU only."""

import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
POLS = {"native-f16": (0, 0, 0), "mixed-half": (0, 0, 1), "full-f32": (1, 1, 1), "full-f64": (2, 2, 2)}


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden_gs.npz")))


def _pol(o, name):
    return o.Pol(*POLS[name])


GS_KEYS = [f"{c}/{p}/{m}" for c in ("rand_40x6", "pos_64x10", "dep_12x4", "ill_50x8")
           for p in POLS for m in ("mgs-l", "mgs-r", "cgs", "cgs2")]


@pytest.mark.parametrize("key", GS_KEYS)
def test_orthonormalize_bitwise(oracle, gold, key):
    case, pname, meth = key.split("/")
    base = f"gs/{key}"
    q, kept = oracle.orthonormalize(gold[base + "/x"], meth, _pol(oracle, pname))
    np.testing.assert_array_equal(kept, gold[base + "/kept"])
    np.testing.assert_array_equal(q, gold[base + "/q"])


@pytest.mark.parametrize("pname", ["full-f64", "full-f32"])
def test_rr_eig_bitwise(oracle, gold, pname):
    r = oracle.rr_eig(gold[f"rreig/{pname}/a"], gold[f"rreig/{pname}/q"], _pol(oracle, pname))
    np.testing.assert_array_equal(r.values, gold[f"rreig/{pname}/vals"])
    np.testing.assert_array_equal(r.vectors, gold[f"rreig/{pname}/vecs"])


@pytest.mark.parametrize("pname", ["full-f64", "full-f32"])
@pytest.mark.parametrize("meth,proj", [("mgs-l", "rr"), ("cgs2", "rr"), ("mgs-r", "ofrr"), ("cgs", "rr")])
def test_driver_with_gs_bases(oracle, gold, pname, meth, proj):
    a = gold[f"driver/{pname}/a"]
    rs = oracle.subspace_iter_eig(a, k=20, m=3, iters=2, pol=_pol(oracle, pname), seed=2, method=meth,
                                  projection=proj)
    key = f"driver/{pname}/{meth}/{proj}"
    np.testing.assert_allclose(rs.values, gold[key + "/vals"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(rs.residuals, gold[key + "/res"], rtol=1e-6, atol=1e-13)
