"""The experiment harness on the B200 path (paper_2505_00281_b200/harness.py) against the
reference harness (ofrr/cli.py): spec grammar, cell validation, matrix generation, row
schema and order, CSV/JSON formatting (host tests), and the OFRR cells' values and
residuals against the reference's own CSV on the same specs (GPU test; golden files from
tests/golden/make_harness_golden.py)."""

import csv
import io
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _h():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2505_00281_b200 import harness
    return harness


def _ref_rows(name):
    with open(os.path.join(GOLD, name + ".ref.csv")) as fh:
        return list(csv.DictReader(fh))


def test_spec_grammar_and_cells():
    h = _h()
    spec = h.parse_spec_text("""# comment
experiment = kernel-eig
n = 50   # trailing comment
k=8
seed = 7
format = json
cell = full-f64:full-f64:hess-l:ofrr
cell = mixed-half : tc-bf16 : hess-r : ofrr
""")
    assert spec.experiment == "kernel-eig" and spec.seed == 7 and spec.fmt == "json"
    assert spec.get_int("n") == 50 and spec.get_int("k") == 8 and spec.get_int("m", 1) == 1
    assert [c.basis_method for c in spec.cells] == ["hess-l", "hess-r"]
    assert spec.cells[1].matvec_policy == "mixed-half" and spec.cells[1].policy == "tc-bf16"
    for bad in ("cell = full-f64:full-f64:hess-l", "cell = nope:full-f64:hess-l:ofrr",
                "cell = full-f64:full-f64:qr:ofrr", "cell = full-f64:full-f64:hess-l:lanczos", "k 8"):
        with pytest.raises(ValueError):
            h.parse_spec_text(bad)


def test_kernel_matrices_match_the_reference_generator():
    """Same PCG64 points and the same FP64 formula as ofrr/matrix.py:89-113."""
    h = _h()
    fp = json.load(open(os.path.join(GOLD, "harness_fingerprints.json")))
    for name, gen in (("harness_eig", h.kernel_matrix), ("harness_svd", h.cross_kernel_matrix)):
        a = gen(h.parse_spec_file(os.path.join(GOLD, name + ".cfg")))
        f = fp[name]
        assert list(a.shape) == f["shape"]
        assert a[0, 0] == f["diag0"] and a[3, 7] == f["a37"]
        assert abs(a.sum() - f["sum"]) <= 1e-12 * abs(f["sum"])


def test_result_format_matches_the_reference_schema():
    h = _h()
    ref = _ref_rows("harness_eig")
    with open(os.path.join(GOLD, "harness_eig.ref.csv")) as fh:
        header = fh.readline().strip().split(",")
    assert header == h.CSV_COLUMNS
    rows = [{c: (float(r[c]) if c in h._NUM_COLS and r[c] != "" else
                 (int(r[c]) if c == "index" and r[c] != "" else r[c])) for c in h.CSV_COLUMNS} for r in ref]
    text = h.format_results(rows, "csv")
    with open(os.path.join(GOLD, "harness_eig.ref.csv")) as fh:
        assert text == fh.read()                       # 17 significant digits, same quoting
    recs = json.loads(h.format_results(rows, "json"))
    assert len(recs) == len(rows) and set(recs[0]) == set(h.CSV_COLUMNS)
    assert recs[0]["cond2"] is None and isinstance(recs[0]["value"], float)


def test_unsupported_experiment_raises():
    h = _h()
    with pytest.raises(ValueError):
        h.run_experiment(h.parse_spec_text("experiment = cond-study\ncell = full-f64:full-f64:hess-l:none"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["harness_eig", "harness_svd"])
def test_harness_rows_vs_reference_harness(ofrr_gpu, name):
    """Every cell of the reference's own run -- the OFRR cells and the classical comparator
    (Gram-Schmidt basis + classical RR, csrc/gs.cu): same rows (keys, order, status), the
    north-star value / residual criteria per cell."""
    h = _h()
    spec = h.parse_spec_file(os.path.join(GOLD, name + ".cfg"))
    ours = h.run_experiment(spec)
    ref = _ref_rows(name)
    ours_ok = list(ours)
    ref_ok = list(ref)
    key = lambda r: (r["matrix"], r["policy"], r["basis_method"], r["projection"], str(r["index"]))  # noqa: E731
    assert [key(r) for r in ours_ok] == [key(r) for r in ref_ok]
    # per cell, the north-star criteria with the reading of tests/test_gpu_driver.py::
    # _criteria: the max over the cell's reported pairs of the relative error within
    # max(10 x the reference's, 1e-6), of the residual within 2x the reference's (single
    # pairs of a 16-bit or fp32 pipeline are a rounding lottery at their noise floor)
    cells = {}
    for o, r in zip(ours_ok, ref_ok):
        assert o["status"] == r["status"] == "ok"
        assert float(o["reference"]) == pytest.approx(float(r["reference"]), rel=1e-12)
        w = cells.setdefault(key(o)[:4], [0.0, 0.0, 0.0, 0.0])
        w[0] = max(w[0], o["rel_error"])
        w[1] = max(w[1], float(r["rel_error"]))
        w[2] = max(w[2], o["residual"])
        w[3] = max(w[3], float(r["residual"]))
    for cell, (oe, re_, orr, rr) in cells.items():
        assert oe <= max(10 * re_, 1e-6), (cell, oe, re_)
        # residuals at the FP64 floor (~1e-13 for n = 400) are rounding noise: 2x + that floor
        assert orr <= 2 * rr + 1e-12, (cell, orr, rr)
    text = h.format_results(ours, "csv")
    assert text.splitlines()[0].split(",") == h.CSV_COLUMNS


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["harness_eig", "harness_svd"])
def test_device_kernel_generator_matches_host(ofrr_gpu, name):
    """csrc/gen.cu evaluates the reference's kernel formula in the reference's operation order:
    every entry within 2 ulp of the host FP64 matrix (CUDA's exp vs libm's, then f and s), most bitwise."""
    h = _h()
    spec = h.parse_spec_file(os.path.join(GOLD, name + ".cfg"))
    ks = h.kernel_spec(spec)
    host = h.kernel_host(ks)
    dev = h.kernel_operator(ks)
    op = dev.device_operator()
    got = op.t[:, :op.cols].cpu().numpy()
    ulp = np.spacing(np.abs(host))
    assert np.all(np.abs(got - host) <= 2 * ulp), np.max(np.abs(got - host) / ulp)
    assert np.mean(got == host) > 0.9


@pytest.mark.gpu
def test_threaded_cells_equal_serial(ofrr_gpu):
    """--threads: cells from a thread pool (ofrr/cli.py:399-401) give the serial rows."""
    h = _h()
    spec = h.parse_spec_file(os.path.join(GOLD, "harness_eig.cfg"))
    serial = h.run_experiment(spec)
    threaded = h.run_experiment(spec, threads=4)
    strip = lambda rows: [{c: r[c] for c in h.CSV_COLUMNS if c != "wall_ms"} for r in rows]  # noqa: E731
    assert strip(serial) == strip(threaded)
