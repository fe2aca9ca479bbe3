"""Experiment harness on the B200 path: the reference's spec-file grammar, cell syntax and
CSV/JSON result schema (ofrr/cli.py:47-126, 226-286, 411-444), running the OFRR cells on
the GPU.  SURVEY.md 8(f), rank 3.

    python -m paper_2505_00281_b200.harness kernel-eig --spec fig3.cfg [--set k=v] [--seed S]
                                            [--out results.csv] [--format csv|json]

* Spec files: ``key = value`` lines, ``#`` comments, repeated ``cell = mvp:pol:method:proj``
  lines (ofrr/cli.py:100-126).  Same keys and defaults: n, f, l, s, n2, side, k, m, iter,
  restarts, top, seed, out, format.
* Matrices: the reference's seeded Gaussian kernel (``kernel-eig``: square, points from
  PCG64(seed + 777); ``kernel-svd``: cross kernel with columns from PCG64(seed + 778);
  ofrr/cli.py:163-189, ofrr/matrix.py:89-113), generated in FP64 on the host exactly as the
  reference does and uploaded once.
* The ``reference`` column is the FP64 spectrum of the same matrix (LAPACK through numpy),
  as ofrr/cli.py:359-365 computes it with the reference's own eigensolver.
* Cells whose method/projection is outside the OFRR path on this package (Gram-Schmidt
  builders, classical RR, ``none``/``raw``, Krylov) produce the reference's failure row
  with status ``error`` (the package has no CPU fallback).  ``sparse-eig``,
  ``cond-study`` and ``bench`` are outside the B200 path and raise ``ValueError``.
* Rows, their order (ofrr/cli.py:405-408) and the 17-digit number format (:411-444) are
  the reference's.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .basis import BasisMethod
from .driver import IterConfig, subspace_iter_eig, subspace_iter_svd
from .errors import ConvergenceError, EmptyBasisError, EmptyPencilError, OverflowDiagnostic
from .matrix import DenseMatrix
from .precision import POLICY_PRESETS, FpFormat

CSV_COLUMNS = [
    "experiment", "matrix", "policy", "basis_method", "projection", "index",
    "value", "reference", "rel_error", "residual", "cond2", "wall_ms",
    "status",
]
EXPERIMENTS = ("kernel-eig", "kernel-svd")
_METHODS = {m.value: m for m in BasisMethod}
_NUM_COLS = {"value", "reference", "rel_error", "residual", "cond2", "wall_ms"}


@dataclass
class Cell:
    """``matvec_policy:policy:basis_method:projection`` (ofrr/cli.py:57-78)."""
    matvec_policy: str
    policy: str
    basis_method: str
    projection: str

    @classmethod
    def parse(cls, text: str) -> "Cell":
        parts = text.split(":")
        if len(parts) != 4:
            raise ValueError(f"cell {text!r}: expected matvec_policy:policy:method:projection")
        mvp, pol, meth, proj = (p.strip() for p in parts)
        for name in (mvp, pol):
            if name not in POLICY_PRESETS:
                raise ValueError(f"cell {text!r}: unknown policy preset {name!r}")
        if meth not in _METHODS and meth != "raw":
            raise ValueError(f"cell {text!r}: unknown basis method {meth!r}")
        if proj not in ("rr", "ofrr", "none"):
            raise ValueError(f"cell {text!r}: projection must be rr/ofrr/none")
        return cls(mvp, pol, meth, proj)


@dataclass
class ExperimentSpec:
    experiment: str
    params: dict = field(default_factory=dict)
    cells: list = field(default_factory=list)
    seed: int = 0
    out: Optional[str] = None
    fmt: str = "csv"

    def get(self, key, default=None):
        return self.params.get(key, default)

    def get_int(self, key, default=None):
        v = self.params.get(key)
        return default if v is None else int(v)

    def get_float(self, key, default=None):
        v = self.params.get(key)
        return default if v is None else float(v)


def parse_spec_text(text: str, origin: str = "<spec>") -> ExperimentSpec:
    """The spec grammar of ofrr/cli.py:100-126 (repeated ``cell=`` lines accumulate)."""
    params: dict = {}
    cells: list = []
    for lineno, line in enumerate(text.splitlines(), start=1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"{origin}:{lineno}: expected key=value")
        key, _, value = line.partition("=")
        key, value = key.strip(), value.strip()
        if key == "cell":
            cells.append(Cell.parse(value))
        else:
            params[key] = value
    return ExperimentSpec(experiment=params.pop("experiment", ""), params=params, cells=cells,
                          seed=int(params.pop("seed", 0)), out=params.pop("out", None),
                          fmt=params.pop("format", "csv"))


def parse_spec_file(path: str) -> ExperimentSpec:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_spec_text(fh.read(), path)


# ---- matrices (ofrr/cli.py:163-189; ofrr/matrix.py:89-113) -------------------------------
def _points(n: int, side: float, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).random((n, 2)) * side


def _gaussian(x: np.ndarray, y: Optional[np.ndarray], f: float, l: float, s: float) -> np.ndarray:
    yy = x if y is None else y
    d2 = np.sum(x * x, axis=1)[:, None] + np.sum(yy * yy, axis=1)[None, :] - 2.0 * (x @ yy.T)
    np.maximum(d2, 0.0, out=d2)
    a = np.exp(-d2 / (2.0 * l * l))
    if y is None:
        a[np.diag_indices_from(a)] += s
    a *= f
    return np.asfortranarray(a)


def kernel_matrix(spec: ExperimentSpec) -> np.ndarray:
    n = spec.get_int("n", 1000)
    side = spec.get_float("side", float(np.sqrt(n)))
    return _gaussian(_points(n, side, spec.seed + 777), None, spec.get_float("f", 1.0),
                     spec.get_float("l", 10.0), spec.get_float("s", 0.0))


def cross_kernel_matrix(spec: ExperimentSpec) -> np.ndarray:
    n, n2 = spec.get_int("n", 1000), spec.get_int("n2", 200)
    side = spec.get_float("side", float(np.sqrt(n)))
    cols = _points(n2, side, spec.seed + 778)
    return _gaussian(_points(n, side, spec.seed + 777), cols, spec.get_float("f", 0.2),
                     spec.get_float("l", 10.0), 0.0)


# ---- rows --------------------------------------------------------------------------------
_FAILURES = ((OverflowDiagnostic, "overflow"), ((EmptyBasisError, EmptyPencilError), "breakdown"),
             (ConvergenceError, "error"))


def _status_of(exc: Exception) -> str:
    for types, name in _FAILURES:
        if isinstance(exc, types):
            return name
    return "error"


def _blank_row(spec, matrix, cell) -> dict:
    return {c: "" for c in CSV_COLUMNS} | {
        "experiment": spec.experiment, "matrix": matrix, "policy": f"{cell.matvec_policy}:{cell.policy}",
        "basis_method": cell.basis_method, "projection": cell.projection, "status": "ok"}


def _iter_config(spec: ExperimentSpec, cell: Cell) -> IterConfig:
    if cell.basis_method not in _METHODS:
        raise ValueError(f"basis method {cell.basis_method!r} is outside the OFRR path")
    return IterConfig(k=spec.get_int("k", 20), m=spec.get_int("m", 1), iter=spec.get_int("iter", 1),
                      restarts=spec.get_int("restarts", 0), basis_method=_METHODS[cell.basis_method],
                      projection=cell.projection, policy=POLICY_PRESETS[cell.policy],
                      matvec_policy=POLICY_PRESETS[cell.matvec_policy], seed=spec.seed)


def _value_rows(spec, name, cell, values, residuals, reference, wall_ms, top) -> list:
    """ofrr/cli.py:248-268."""
    rows = []
    nrep = min(top, len(values)) if top else len(values)
    for i in range(nrep):
        row = _blank_row(spec, name, cell)
        row["index"] = i
        row["value"] = values[i]
        if reference is not None and i < len(reference) and reference[i] != 0.0:
            row["reference"] = reference[i]
            row["rel_error"] = abs(values[i] - reference[i]) / abs(reference[i])
        if residuals is not None:
            row["residual"] = residuals[i]
        row["wall_ms"] = wall_ms
        rows.append(row)
    if nrep < (top or 0):
        row = _blank_row(spec, name, cell)
        row["status"] = "breakdown"
        row["wall_ms"] = wall_ms
        rows.append(row)
    return rows


def _run_cell(spec, a: DenseMatrix, name, reference, cell, svd: bool) -> list:
    top = spec.get_int("top", 0)
    try:
        cfg = _iter_config(spec, cell)
        t0 = time.monotonic()
        rs = subspace_iter_svd(a, cfg) if svd else subspace_iter_eig(a, cfg)
        wall = (time.monotonic() - t0) * 1e3
    except Exception as exc:  # cell failures become rows, not crashes (ofrr/cli.py:277-280)
        row = _blank_row(spec, name, cell)
        row["status"] = _status_of(exc)
        return [row]
    return _value_rows(spec, name, cell, np.asarray(rs.values), np.asarray(rs.residuals), reference, wall, top)


def run_experiment(spec: ExperimentSpec) -> list:
    """Every grid cell of a kernel-eig / kernel-svd spec, in the reference's row order."""
    env_seed = os.environ.get("OFRR_SEED")
    if env_seed is not None:
        spec.seed = int(env_seed)
    if spec.experiment == "kernel-eig":
        host = kernel_matrix(spec)
        name = f"kernel(n={host.shape[0]},f={spec.get('f', '1')},l={spec.get('l', '10')},s={spec.get('s', '0')})"
        ref = np.sort(np.linalg.eigvalsh(host))[::-1]
        svd = False
    elif spec.experiment == "kernel-svd":
        host = cross_kernel_matrix(spec)
        name = f"kernel-cross({host.shape[0]}x{host.shape[1]},f={spec.get('f', '0.2')},l={spec.get('l', '10')})"
        ref = np.linalg.svd(host, compute_uv=False)
        svd = True
    else:
        raise ValueError(f"experiment {spec.experiment!r} is outside the B200 OFRR path "
                         f"(supported: {', '.join(EXPERIMENTS)})")
    a = DenseMatrix.from_array(host, FpFormat.F64)
    rows = []
    for cell in spec.cells:
        rows += _run_cell(spec, a, name, ref, cell, svd)
    rows.sort(key=lambda r: (r["matrix"], r["policy"], r["basis_method"], r["projection"],
                             r["index"] if r["index"] != "" else -1))
    return rows


def _fmt_num(v) -> str:
    if v == "" or v is None:
        return ""
    return format(float(v), ".17g")


def format_results(rows: list, fmt: str) -> str:
    """CSV or JSON with 17 significant digits (ofrr/cli.py:411-435)."""
    if fmt == "csv":
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for row in rows:
            w.writerow([_fmt_num(row[c]) if c in _NUM_COLS else row[c] for c in CSV_COLUMNS])
        return buf.getvalue()
    if fmt == "json":
        recs = []
        for row in rows:
            recs.append({c: ((None if row[c] == "" else float(format(float(row[c]), ".17g")))
                             if c in _NUM_COLS else row[c]) for c in CSV_COLUMNS})
        return json.dumps(recs, indent=1) + "\n"
    raise ValueError(f"unknown format {fmt!r}")


def write_results(rows: list, fmt: str, path: Optional[str]) -> None:
    text = format_results(rows, fmt)
    if path is None:
        sys.stdout.write(text)
        return
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)


def main(argv: Optional[list] = None) -> int:
    """The reference CLI's options (ofrr/cli.py:453-486) for the two kernel experiments."""
    parser = argparse.ArgumentParser(prog="python -m paper_2505_00281_b200.harness",
                                     description="OFRR experiment harness on B200")
    sub = parser.add_subparsers(dest="command", required=True)
    for cmd in EXPERIMENTS:
        p = sub.add_parser(cmd)
        p.add_argument("--spec", required=True)
        p.add_argument("--seed", type=int, default=None)
        p.add_argument("--out", default=None)
        p.add_argument("--format", choices=("csv", "json"), default=None)
        p.add_argument("--set", action="append", default=[], metavar="KEY=VALUE")
    args = parser.parse_args(argv)
    spec = parse_spec_file(args.spec)
    spec.experiment = args.command
    for override in args.set:
        key, _, value = override.partition("=")
        spec.params[key.strip()] = value.strip()
    if args.seed is not None:
        spec.seed = args.seed
    if args.out is not None:
        spec.out = args.out
    if args.format is not None:
        spec.fmt = args.format
    write_results(run_experiment(spec), spec.fmt, spec.out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
