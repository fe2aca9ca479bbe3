"""Experiment harness on the B200 path: runs the reference's spec files for the two OFRR
experiments (``kernel-eig``, ``kernel-svd``) and writes the reference's result schema.
SURVEY.md 8(f), rank 3.

    python -m paper_2505_00281_b200.harness kernel-eig --spec fig3.cfg [--set k=v] [--seed S]
                                            [--out results.csv] [--format csv|json] [--threads N]

What is kept from the reference (the on-disk formats either side of the path):
* spec files: ``key = value`` lines, ``#`` comments, repeated ``cell = mvp:pol:method:proj``
  lines (grammar of ofrr/cli.py:100-126, cell syntax of :57-78); keys n, f, l, s, n2, side,
  k, m, iter, restarts, top, seed, out, format with the reference's defaults;
* the seeded Gaussian-kernel matrices (ofrr/matrix.py:89-113; points PCG64(seed + 777),
  cross-kernel columns PCG64(seed + 778), ofrr/cli.py:163-189);
* the 13-column row schema, the row order (ofrr/cli.py:405-408), failure statuses and the
  17-significant-digit CSV / JSON text (ofrr/cli.py:411-444);
* ``--threads``: cells run from a thread pool (ofrr/cli.py:399-401).

What is B200-native: the n x n (or n x n2) kernel matrix is evaluated on the device in FP64
(``ofrr_gaussian_kernel``, csrc/gen.cu) straight into the HBM-resident operator -- no n^2 host
work or upload; the ``reference`` column (the full FP64 spectrum / singular values of the same
matrix, ofrr/cli.py:359-365) comes from cuSOLVER on that device copy.  Cells outside the
B200 path (``raw`` / ``none``, Krylov builders) are ``error`` rows: there is no CPU fallback.
``sparse-eig``, ``cond-study`` and ``bench`` are outside the path and raise ``ValueError``.
"""

from __future__ import annotations

import argparse
import concurrent.futures
import csv
import io
import json
import os
import re
import sys
import time
from typing import Callable, Iterable, NamedTuple, Optional

import numpy as np

from .basis import BasisMethod, GRAM_SCHMIDT_METHODS, HESSENBERG_METHODS
from .driver import IterConfig, subspace_iter_eig, subspace_iter_svd
from .errors import ConvergenceError, EmptyBasisError, EmptyPencilError, OverflowDiagnostic
from .matrix import DenseMatrix
from .precision import POLICY_PRESETS, FpFormat

# ---- the result schema ---------------------------------------------------------------------
# (column, kind): "s" text, "i" integer index, "f" number written with 17 significant digits
SCHEMA = (("experiment", "s"), ("matrix", "s"), ("policy", "s"), ("basis_method", "s"),
          ("projection", "s"), ("index", "i"), ("value", "f"), ("reference", "f"), ("rel_error", "f"),
          ("residual", "f"), ("cond2", "f"), ("wall_ms", "f"), ("status", "s"))
CSV_COLUMNS = [c for c, _ in SCHEMA]
_NUM_COLS = frozenset(c for c, kind in SCHEMA if kind == "f")
EXPERIMENTS = ("kernel-eig", "kernel-svd")
PROJECTIONS = ("rr", "ofrr", "none")
_BLOCK_METHODS = {m.value: m for m in BasisMethod}

# exception class -> row status (ofrr/cli.py failure statuses)
_STATUS = ((OverflowDiagnostic, "overflow"), (EmptyBasisError, "breakdown"), (EmptyPencilError, "breakdown"),
           (ConvergenceError, "error"))


# ---- cells and specs -------------------------------------------------------------------------
_CELL = re.compile(r"^([^:]*):([^:]*):([^:]*):([^:]*)$")


class Cell(NamedTuple):
    """One grid cell ``matvec_policy:policy:basis_method:projection``."""
    matvec_policy: str
    policy: str
    basis_method: str
    projection: str

    @classmethod
    def parse(cls, text: str) -> "Cell":
        hit = _CELL.match(text.strip())
        if hit is None:
            raise ValueError(f"cell {text!r}: expected matvec_policy:policy:method:projection")
        cell = cls(*(g.strip() for g in hit.groups()))
        bad = [p for p in (cell.matvec_policy, cell.policy) if p not in POLICY_PRESETS]
        if bad:
            raise ValueError(f"cell {text!r}: unknown policy preset {bad[0]!r}")
        if cell.basis_method != "raw" and cell.basis_method not in _BLOCK_METHODS:
            raise ValueError(f"cell {text!r}: unknown basis method {cell.basis_method!r}")
        if cell.projection not in PROJECTIONS:
            raise ValueError(f"cell {text!r}: projection must be one of {'/'.join(PROJECTIONS)}")
        return cell

    @property
    def policy_label(self) -> str:
        return f"{self.matvec_policy}:{self.policy}"


class ExperimentSpec:
    """A parsed spec: the experiment name, its keyed parameters (strings, typed on access),
    the cell grid and the run options (seed, output path, format)."""

    _RUN_KEYS = {"experiment": ("experiment", str), "seed": ("seed", int), "out": ("out", str),
                 "format": ("fmt", str)}

    def __init__(self, experiment: str = "", params: Optional[dict] = None, cells: Optional[list] = None,
                 seed: int = 0, out: Optional[str] = None, fmt: str = "csv"):
        self.experiment, self.seed, self.out, self.fmt = experiment, seed, out, fmt
        self.params = dict(params or {})
        self.cells = list(cells or [])

    def get(self, key: str, default=None):
        return self.params.get(key, default)

    def get_int(self, key: str, default=None):
        return default if key not in self.params else int(self.params[key])

    def get_float(self, key: str, default=None):
        return default if key not in self.params else float(self.params[key])

    def assign(self, key: str, value: str) -> None:
        """One ``key = value`` entry: run options, a cell, or a parameter."""
        if key == "cell":
            self.cells.append(Cell.parse(value))
        elif key in self._RUN_KEYS:
            attr, conv = self._RUN_KEYS[key]
            setattr(self, attr, conv(value))
        else:
            self.params[key] = value


def _entries(text: str, origin: str) -> Iterable[tuple]:
    for lineno, raw in enumerate(text.splitlines(), start=1):
        body = raw.partition("#")[0].strip()
        if not body:
            continue
        key, eq, value = body.partition("=")
        if not eq:
            raise ValueError(f"{origin}:{lineno}: expected key=value")
        yield key.strip(), value.strip()


def parse_spec_text(text: str, origin: str = "<spec>") -> ExperimentSpec:
    spec = ExperimentSpec()
    for key, value in _entries(text, origin):
        spec.assign(key, value)
    return spec


def parse_spec_file(path: str) -> ExperimentSpec:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_spec_text(fh.read(), path)


# ---- matrices -----------------------------------------------------------------------------
class KernelSpec(NamedTuple):
    """The Gaussian kernel of a spec: A_ij = f (exp(-|x_i - y_j|^2 / (2 l^2)) + s [square, i = j])."""
    x: np.ndarray                 # n x 2 points
    y: Optional[np.ndarray]       # n2 x 2 column points (cross kernel) or None (square)
    f: float
    l: float
    s: float

    @property
    def shape(self):
        return (self.x.shape[0], (self.x if self.y is None else self.y).shape[0])


def _uniform_points(count: int, side: float, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).random((count, 2)) * side


def kernel_spec(spec: ExperimentSpec) -> KernelSpec:
    """Points and parameters of the spec's kernel matrix (ofrr/cli.py:163-189)."""
    n = spec.get_int("n", 1000)
    side = spec.get_float("side", float(np.sqrt(n)))
    x = _uniform_points(n, side, spec.seed + 777)
    if spec.experiment == "kernel-svd":
        y = _uniform_points(spec.get_int("n2", 200), side, spec.seed + 778)
        return KernelSpec(x, y, spec.get_float("f", 0.2), spec.get_float("l", 10.0), 0.0)
    return KernelSpec(x, None, spec.get_float("f", 1.0), spec.get_float("l", 10.0), spec.get_float("s", 0.0))


def kernel_host(ks: KernelSpec) -> np.ndarray:
    """The FP64 kernel matrix on the host in the reference's operation order (ofrr/matrix.py:
    97-113) -- small n only (tests, fingerprints); the harness itself uses kernel_operator."""
    y = ks.x if ks.y is None else ks.y
    d2 = np.maximum((np.sum(ks.x * ks.x, axis=1)[:, None] + np.sum(y * y, axis=1)[None, :]) - 2.0 * (ks.x @ y.T), 0.0)
    a = np.exp(-d2 / (2.0 * ks.l * ks.l))
    if ks.y is None:
        a[np.diag_indices_from(a)] += ks.s
    return np.asfortranarray(a * ks.f)


def kernel_matrix(spec: ExperimentSpec) -> np.ndarray:
    """Host FP64 matrix of a kernel-eig spec (square)."""
    return kernel_host(kernel_spec(_as(spec, "kernel-eig")))


def cross_kernel_matrix(spec: ExperimentSpec) -> np.ndarray:
    """Host FP64 matrix of a kernel-svd spec (n x n2)."""
    return kernel_host(kernel_spec(_as(spec, "kernel-svd")))


def _as(spec: ExperimentSpec, experiment: str) -> ExperimentSpec:
    return ExperimentSpec(experiment, spec.params, spec.cells, spec.seed, spec.out, spec.fmt)


def kernel_operator(ks: KernelSpec, device=None) -> DenseMatrix:
    """The kernel matrix evaluated on the device in FP64 (csrc/gen.cu), row-major and HBM
    resident, wrapped as a DenseMatrix (its bf16 / f16 / f32 copies are made from it)."""
    import torch
    from . import _lib, ops
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    n, m = ks.shape
    op = ops.new_operator(n, m, FpFormat.F64, device)
    px = torch.as_tensor(np.ascontiguousarray(ks.x), dtype=torch.float64, device=device)
    py = None if ks.y is None else torch.as_tensor(np.ascontiguousarray(ks.y), dtype=torch.float64, device=device)
    L = _lib.load()
    _lib.check(L.ofrr_gaussian_kernel(px.data_ptr(), n, None if py is None else py.data_ptr(), m, float(ks.f),
                                      float(ks.l), float(ks.s), op.ptr, op.lda, int(FpFormat.F64),
                                      torch.cuda.current_stream(device).cuda_stream), "gaussian_kernel")
    ops._count(1)
    return DenseMatrix.on_device(op)


def _matrix_label(spec: ExperimentSpec, ks: KernelSpec) -> str:
    n, m = ks.shape
    if ks.y is None:
        return f"kernel(n={n},f={spec.get('f', '1')},l={spec.get('l', '10')},s={spec.get('s', '0')})"
    return f"kernel-cross({n}x{m},f={spec.get('f', '0.2')},l={spec.get('l', '10')})"


def _reference_values(a: DenseMatrix, svd: bool) -> np.ndarray:
    """FP64 spectrum (descending) or singular values of the device matrix (cuSOLVER)."""
    import torch
    op = a.device_operator(FpFormat.F64)
    t = op.t[:, :op.cols]
    vals = torch.linalg.svdvals(t) if svd else torch.linalg.eigvalsh(t).flip(0)
    return vals.cpu().numpy()


# ---- rows ---------------------------------------------------------------------------------------
def _row(spec: ExperimentSpec, matrix: str, cell: Cell, **fields) -> dict:
    row = dict.fromkeys(CSV_COLUMNS, "")
    row.update(experiment=spec.experiment, matrix=matrix, policy=cell.policy_label,
               basis_method=cell.basis_method, projection=cell.projection, status="ok")
    row.update(fields)
    return row


def _failure_status(exc: Exception) -> str:
    return next((status for cls, status in _STATUS if isinstance(exc, cls)), "error")


def _config_for(spec: ExperimentSpec, cell: Cell) -> IterConfig:
    method = _BLOCK_METHODS.get(cell.basis_method)
    if method is None or not (method in HESSENBERG_METHODS or method in GRAM_SCHMIDT_METHODS) \
            or cell.projection == "none":
        raise ValueError(f"cell {cell}: outside the B200 subspace-iteration path")
    return IterConfig(k=spec.get_int("k", 20), m=spec.get_int("m", 1), iter=spec.get_int("iter", 1),
                      restarts=spec.get_int("restarts", 0), basis_method=method, projection=cell.projection,
                      policy=POLICY_PRESETS[cell.policy], matvec_policy=POLICY_PRESETS[cell.matvec_policy],
                      seed=spec.seed)


def _cell_rows(spec: ExperimentSpec, a: DenseMatrix, matrix: str, reference: np.ndarray, cell: Cell,
               svd: bool) -> list:
    """The rows of one cell: one per reported value (up to ``top``), a ``breakdown`` row when
    fewer came back, or one failure row (cell failures never abort the grid)."""
    top = spec.get_int("top", 0)
    try:
        cfg = _config_for(spec, cell)
        t0 = time.monotonic()
        rs = (subspace_iter_svd if svd else subspace_iter_eig)(a, cfg)
        wall = (time.monotonic() - t0) * 1e3
    except Exception as exc:
        return [_row(spec, matrix, cell, status=_failure_status(exc))]
    values, resid = np.asarray(rs.values), np.asarray(rs.residuals)
    count = min(top, values.size) if top else values.size
    out = []
    for idx in range(count):
        extra = {}
        if idx < reference.size and reference[idx] != 0.0:
            extra = dict(reference=reference[idx], rel_error=abs(values[idx] - reference[idx]) / abs(reference[idx]))
        out.append(_row(spec, matrix, cell, index=idx, value=values[idx], residual=resid[idx], wall_ms=wall, **extra))
    if top and count < top:
        out.append(_row(spec, matrix, cell, status="breakdown", wall_ms=wall))
    return out


def _row_order(row: dict):
    return (row["matrix"], row["policy"], row["basis_method"], row["projection"],
            -1 if row["index"] == "" else row["index"])


def run_experiment(spec: ExperimentSpec, threads: int = 1) -> list:
    """Every cell of a kernel-eig / kernel-svd spec (from a thread pool when threads > 1),
    in the reference's row order."""
    if "OFRR_SEED" in os.environ:
        spec.seed = int(os.environ["OFRR_SEED"])
    if spec.experiment not in EXPERIMENTS:
        raise ValueError(f"experiment {spec.experiment!r} is outside the B200 OFRR path "
                         f"(supported: {', '.join(EXPERIMENTS)})")
    svd = spec.experiment == "kernel-svd"
    ks = kernel_spec(spec)
    a = kernel_operator(ks)
    matrix = _matrix_label(spec, ks)
    reference = _reference_values(a, svd)
    job: Callable[[Cell], list] = lambda cell: _cell_rows(spec, a, matrix, reference, cell, svd)  # noqa: E731
    if threads > 1:
        with concurrent.futures.ThreadPoolExecutor(max_workers=threads) as pool:
            chunks = list(pool.map(job, spec.cells))
    else:
        chunks = [job(cell) for cell in spec.cells]
    return sorted((row for chunk in chunks for row in chunk), key=_row_order)


# ---- output ---------------------------------------------------------------------------------------
def _num17(v) -> str:
    return "" if v is None or v == "" else format(float(v), ".17g")


def _csv_text(rows: list) -> str:
    buf = io.StringIO()
    out = csv.writer(buf, lineterminator="\n")
    out.writerow(CSV_COLUMNS)
    out.writerows([[_num17(r[c]) if c in _NUM_COLS else r[c] for c in CSV_COLUMNS] for r in rows])
    return buf.getvalue()


def _json_text(rows: list) -> str:
    def field(c, v):
        if c not in _NUM_COLS:
            return v
        return None if v == "" else float(_num17(v))
    return json.dumps([{c: field(c, r[c]) for c in CSV_COLUMNS} for r in rows], indent=1) + "\n"


_WRITERS = {"csv": _csv_text, "json": _json_text}


def format_results(rows: list, fmt: str) -> str:
    if fmt not in _WRITERS:
        raise ValueError(f"unknown format {fmt!r}")
    return _WRITERS[fmt](rows)


def write_results(rows: list, fmt: str, path: Optional[str]) -> None:
    text = format_results(rows, fmt)
    if path is None:
        sys.stdout.write(text)
    else:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)


def main(argv: Optional[list] = None) -> int:
    parser = argparse.ArgumentParser(prog="python -m paper_2505_00281_b200.harness",
                                     description="OFRR experiment harness on B200")
    sub = parser.add_subparsers(dest="command", required=True)
    for name in EXPERIMENTS:
        cmd = sub.add_parser(name)
        cmd.add_argument("--spec", required=True)
        cmd.add_argument("--seed", type=int)
        cmd.add_argument("--out")
        cmd.add_argument("--format", choices=sorted(_WRITERS))
        cmd.add_argument("--threads", type=int, default=1)
        cmd.add_argument("--set", action="append", default=[], metavar="KEY=VALUE")
    args = parser.parse_args(argv)
    spec = parse_spec_file(args.spec)
    spec.experiment = args.command
    for item in args.set:
        key, _, value = item.partition("=")
        spec.assign(key.strip(), value.strip())
    for attr, value in (("seed", args.seed), ("out", args.out), ("fmt", args.format)):
        if value is not None:
            setattr(spec, attr, value)
    write_results(run_experiment(spec, threads=args.threads), spec.fmt, spec.out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
