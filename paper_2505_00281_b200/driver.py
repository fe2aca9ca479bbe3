"""Outer iterations of OFRR on the device: subspace iteration for eigenpairs and
alternating subspace iteration for the partial SVD.

Same entry points, options and results as ofrr/driver.py:40-173
(``IterConfig``, ``subspace_iter_eig``, ``subspace_iter_svd``), restricted to the
B200 path's basis/projection pair (hess-l / hess-r + "ofrr"; anything else raises
ValueError -- there is no CPU fallback).  Extension fields on IterConfig:
``tol`` / ``top`` turn the fixed ``m`` outer iterations into "stop once the FP64
residuals of the leading ``top`` pairs are below ``tol``" (``m`` is then the cap);
their defaults keep the reference's fixed-m behaviour.

Multi-GPU: when torch.distributed is initialised (one process per GPU), A is
row-partitioned (rank p owns rows [p*rp, (p+1)*rp)); each power step all-gathers the
n x k block and all-reduces the k column maxima, each projection all-reduces the k x k
partial Gram U_p^T W_p (fp64).  The Hessenberg basis, the pencil solve and the Ritz
recovery are redundant on every rank (deterministic, so every rank holds identical
results).  See DESIGN.md section "Multi-GPU".
"""

from __future__ import annotations

import math
import threading
import time
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import ops as _ops
from .basis import BasisMethod, GRAM_SCHMIDT_METHODS, HESSENBERG_METHODS, KRYLOV_METHODS
from .comm import Comm
from .errors import ConvergenceError, EmptyBasisError, EmptyPencilError, OverflowDiagnostic
from .matrix import DenseMatrix
from .precision import FpFormat, PrecisionPolicy, projection_policy, round_to
from .projection import POSITIVE_EIG_TOL, RitzSet


@dataclass(frozen=True)
class IterConfig:
    """ofrr/driver.py:40-62, plus the time-to-tolerance extension (tol, top)."""
    k: int
    m: int = 1
    iter: int = 1
    restarts: int = 0
    basis_method: BasisMethod = BasisMethod.MGS_LEFT
    projection: str = "rr"  # "rr" | "ofrr"
    policy: PrecisionPolicy = None
    matvec_policy: Optional[PrecisionPolicy] = None  # defaults to policy
    seed: int = 0
    tol: Optional[float] = None   # extension: stop when max residual over `top` < tol
    top: Optional[int] = None     # extension: number of leading pairs checked
    ladder: Optional[PrecisionPolicy] = None   # extension: cheaper policy run first (see below); or a
    #                               tuple of policies, cheapest first (one rung each)
    ladder_switch: float = 1e-3   # ... until its residual estimate falls below this (or stalls); a tuple
    #                               with one threshold per rung when ladder is a tuple
    reuse_av: bool = False        # extension: next power step from the projection, A U Y = W Y (one
    #                               A pass per outer iteration instead of iter + 1; see EigEngine)

    def __post_init__(self):
        if self.k < 1 or self.m < 1 or self.iter < 1 or self.restarts < 0:
            raise ValueError("k, m, iter must be >= 1 and restarts >= 0")
        if self.projection not in ("rr", "ofrr"):
            raise ValueError("projection must be 'rr' or 'ofrr'")
        if self.policy is None:
            raise ValueError("policy is required")
        if self.top is not None and not (1 <= self.top <= self.k):
            raise ValueError("top must be in [1, k]")
        if self.ladder is not None and self.tol is None:
            raise ValueError("a precision ladder needs tol (it switches on the residual estimate)")
        if isinstance(self.ladder, (tuple, list)):
            sw = self.ladder_switch
            if not isinstance(sw, (tuple, list)) or len(sw) != len(self.ladder):
                raise ValueError("a multi-rung ladder needs one ladder_switch per rung")

    @property
    def mv_policy(self) -> PrecisionPolicy:
        return self.matvec_policy or self.policy


def operator_for(a: DenseMatrix, block_fmt: FpFormat):
    """The device copy of A that multiplies blocks stored in ``block_fmt``.

    An F32 block against an operator held exactly in bf16 runs on the bf16 tensor cores
    (the block split into three bf16 slices, ops.gemm_av): fp32-accurate products at bf16
    HBM traffic, instead of a second fp32 copy of A on the CUDA cores."""
    block_fmt = FpFormat(block_fmt)
    if block_fmt == FpFormat.F32 and (a.fmt == FpFormat.BF16 or FpFormat.BF16 in getattr(a, "_dev", {})):
        op = a.device_operator(FpFormat.BF16)
        if a.exact_in(FpFormat.BF16):
            return op
    if block_fmt == FpFormat.F64:
        # an fp64 block against an operator held exactly in 16/8 bits: FP64-accurate int8
        # tensor-core products (ops.ozaki_gemm) -- no fp64 copy of A (4x the bytes)
        for low in (FpFormat.BF16, FpFormat.F16, FpFormat.FP8_E4M3):
            if a.fmt == low or low in getattr(a, "_dev", {}):
                op = a.device_operator(low)
                if a.exact_in(low):
                    return op
    return a.device_operator(block_fmt)


def _require_ofrr_path(cfg: IterConfig, what: str) -> None:
    """Block basis methods only: Hessenberg (the OFRR path) or Gram-Schmidt (the classical
    comparators), with projection 'ofrr' or 'rr' (ofrr/driver.py:52-58)."""
    if cfg.basis_method in KRYLOV_METHODS:
        raise ValueError(f"{what} needs a block basis method")
    if cfg.basis_method not in HESSENBERG_METHODS and cfg.basis_method not in GRAM_SCHMIDT_METHODS:
        raise ValueError(f"{cfg.basis_method.value!r} is not a block basis method")


@dataclass
class RunStats:
    """Per-run diagnostics (iterations done, residual history, phase timings)."""
    iterations: int = 0
    history: list = field(default_factory=list)   # (iteration, max residual over top)
    converged: bool = False
    a_passes: int = 0
    device_loop: bool = False     # the outer loop ran as one graph with device-side control flow
    rungs: list = field(default_factory=list)   # (basis storage format, iterations, A passes) per ladder rung


# status-vector slots (one int32[8] device vector, read once per sync point)
S_MV_FLAGS, S_NKEPT, S_EIG_STATUS, S_NOUT, S_GRAM_FLAGS, S_RESTART_FLAGS, S_NKEPT2 = 0, 1, 2, 3, 4, 5, 6


# CUDA graphs of the outer iteration, keyed by everything the captured launches depend on
# (device pointers of A, shapes, formats, policies).  A graph reads A through its pointer,
# so a new operator at the same address replays correctly.
_GRAPH_MAX = 8
_GRAPHS = OrderedDict()
# Concurrent callers (the reference CLI runs cells from a thread pool, ofrr/cli.py:399-401):
# solves on the device are serialised by this lock, which also guards the graph caches, the
# launch accounting and the Ozaki workspaces; a solve runs on the calling thread's current
# stream.
_SOLVE_LOCK = threading.RLock()
DEVICE_LOOP = True      # the whole solve as one graph launch (csrc/loop.cu) once its graphs exist
# the first iteration of a rung that starts from the previous rung's next iterate (stepped) takes
# its block product with 5 Ozaki levels (~2^-38 of |A||x|) instead of 6 when the rung's products
# are FP64-accurate: that iteration never produces the FP64 report (a convergence there goes to
# the host loop, which then takes the report from a separate FP64 product)
LEAD_LEVELS = int(__import__("os").environ.get("OFRR_LEAD_LEVELS", "5"))
# a lite fp64 rung (4 levels, ~2^-30) entered from an fp32 rung's Ritz block (not stepped):
# that block is only fp32-accurate, so its first power step takes 3 levels (6 products, ~2^-22)
FIRST_POWER_LEVELS = int(__import__("os").environ.get("OFRR_FIRST_POWER_LEVELS", "3"))
# ... and so does that iteration's projection product (its W feeds a Rayleigh-Ritz step whose
# subspace carries the ~2^-22 power step anyway, and the next power step W Y): 3 levels
FIRST_PROJ_LEVELS = int(__import__("os").environ.get("OFRR_FIRST_PROJ_LEVELS", "3"))
# a fresh solve's first power step multiplies the random start block: one bf16 slice of it is
# as good a start as three (the fp32 rung's later products keep their slices)
START_SLICES_LEVELS = int(__import__("os").environ.get("OFRR_START_LEVELS", "2"))
# ... and that first iteration's projection (residuals there are ~1e-1: a 2^-8 product is plenty)
START_PROJ_LEVELS = int(__import__("os").environ.get("OFRR_START_PROJ_LEVELS", "2"))
HANDOVER_STEPPED = __import__("os").environ.get("OFRR_HANDOVER_STEPPED") == "1"   # ladder: start every rung from the previous rung's W Y (experiments; see _subspace_iter_eig)
_WARM = set()
_NO_GRAPH = set()


class _IterGraph:
    def __init__(self, graph, Xs, outs, rec, prof_group):
        self.graph, self.Xs, self.outs, self.rec, self.prof_group = graph, Xs, outs, rec, prof_group
        self.report = None      # _ReportGraph of the final Ritz vectors + FP64 residuals


class _NoPhase:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_NO_PHASE = _NoPhase()


def _ph(name: str):
    """A named host phase (torch.profiler record_function range, e.g. scripts/timeline.py);
    free when no profiler is running."""
    import torch
    if torch._C._autograd._profiler_enabled():
        return torch.autograd.profiler.record_function("ofrr." + name)
    return _NO_PHASE


def _loop_debug(*msg) -> None:
    import os
    if os.environ.get("OFRR_LOOP_DEBUG"):
        print("[device loop]", *msg, flush=True)


class _LoopExec:
    """An instantiated device-loop graph (cudaGraphExec_t), destroyed with its owner."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            from . import _lib
            _lib.load().ofrr_loop_destroy(self.handle)
        except Exception:
            pass


class _ReportGraph:
    def __init__(self, graph, U64, res, rec):
        self.graph, self.U64, self.res, self.rec = graph, U64, res, rec


def _prof_collect(out) -> None:
    """Harvest K1 kernel timings (bench.py) after the iteration's synchronisation."""
    from . import _lib
    L = _lib.load()
    if L.ofrr_prof_gemm_active():
        g = out.get("prof_group", -1)
        if g is not None and g >= 0:
            L.ofrr_prof_gemm_collect_group(g)
        L.ofrr_prof_gemm_collect()


def _fetch_status(st, comm: Comm):
    if comm.distributed:
        comm.all_reduce_max_(st)
    return st.cpu().numpy()


def _raise_for(s, stage: str, eig: bool = True):
    if s[S_MV_FLAGS] & 1:
        raise OverflowDiagnostic("non-finite entries after MatVec")
    if eig:
        if s[S_GRAM_FLAGS] & 1:
            raise OverflowDiagnostic("non-finite entries in projected matrix")
        if s[S_EIG_STATUS] == 6:
            raise ConvergenceError("Jacobi eigendecomposition did not converge", float("nan"))
        if s[S_EIG_STATUS] == 5 or s[S_NOUT] == 0:
            raise EmptyPencilError("mass matrix retained no eigenvalues")
        if s[S_RESTART_FLAGS] & 1:
            raise OverflowDiagnostic(f"non-finite entries after {stage}")


class EigEngine:
    """Device state of one subspace_iter_eig run (single GPU or row-partitioned)."""

    def __init__(self, a: DenseMatrix, cfg: IterConfig, comm: Optional[Comm] = None, n_global: Optional[int] = None,
                 ops=None, report_scales: bool = True, prepared=None):
        self.ops = ops or _ops
        self.comm = comm or Comm.world()
        self.cfg = cfg
        self.pol = cfg.policy
        self.mv = cfg.mv_policy
        self.a = a
        self.n = int(n_global if n_global is not None else a.cols)
        self.A_mv = operator_for(a, self.mv.storage)
        self.A_pol = self.A_mv if self.pol.storage == self.mv.storage else operator_for(a, self.pol.storage)
        self.device = self.A_mv.device
        self.r0, self.r1 = self.comm.row_range(self.n)
        if self.comm.distributed and self.A_mv.rows != self.r1 - self.r0:
            raise ValueError(f"rank {self.comm.rank}: local A has {self.A_mv.rows} rows, expected "
                             f"{self.r1 - self.r0} (rows {self.r0}..{self.r1} of {self.n})")
        _, self.proj_out = projection_policy(self.pol)
        self.stats = RunStats()
        self._last_w2 = None    # the latest projection's W = A U in its accumulation format
        self._last_w2_levels = 6
        self._oz = {}           # prepared Ozaki digit planes per operator (this run)
        if prepared is not None:
            # an operator prepared on a side stream while the previous ladder rung ran
            oz, ev = prepared
            self._oz[id(oz.A)] = oz
            import torch
            torch.cuda.current_stream(oz.A.device).wait_event(ev)
        # the FP64 report's operator scales only depend on A: refreshed on a side stream while
        # the pencil solve occupies one SM (off the critical path), see _body
        self._res_oz = None
        self._refresh_now = True    # first iteration of a run: refresh the report's row scales
        # (a ladder rung that hands over to the next never reports: no early scale refresh;
        # if it ends the run after all, the report prepares its operator then)
        if (report_scales and self.ops is _ops and not self.comm.distributed
                and FpFormat.F64 not in (self.mv.storage, self.pol.storage) and hasattr(a, "residual_operator")):
            A_res = a.residual_operator(self.A_mv.fmt)
            if A_res.fmt in _ops.OZAKI_FMTS:
                self._res_oz = _ops.OzakiOperator(A_res, prepare=False)
                self._oz[id(A_res)] = self._res_oz

    def _ozaki(self, A):
        """Prepared int8 digit planes of a 16/8-bit operator (once per run), or None."""
        if self.ops is not _ops or A.fmt not in _ops.OZAKI_FMTS:
            return None
        oz = self._oz.get(id(A))
        if oz is None:
            oz = self.ops.OzakiOperator(A)
            self._oz[id(A)] = oz
        return oz

    def _block_oz(self, A, X):
        """The Ozaki operator when an fp64 block meets a 16/8-bit operator."""
        return self._ozaki(A) if X.fmt == FpFormat.F64 else None

    # ---- blocks ---------------------------------------------------------------------
    def start_block(self, out=None):
        """X0 = PCG64(seed) U(0,1), rounded to the MatVec storage (ofrr/driver.py:97-99)."""
        if out is None:
            return self.ops.start_block(self.cfg.seed, self.n, self.cfg.k, self.mv.storage, self.device)
        return self.ops.start_block(self.cfg.seed, self.n, self.cfg.k, self.mv.storage, self.device, out=out)

    def power(self, X, st, steps: Optional[int] = None, levels: Optional[int] = None):
        """cfg.iter MatVecs with inf-norm column scaling (ofrr/driver.py:102-105)."""
        import torch
        ops, comm = self.ops, self.comm
        k = X.k
        levels = self.mv.product_levels if levels is None else levels
        fp8 = self.mv.storage == FpFormat.FP8_E4M3
        for _ in range(self.cfg.iter if steps is None else steps):
            colmax = torch.zeros(k, dtype=torch.float64, device=self.device)
            # e4m3 storage (max 448): the product stays in fp32 until the column scaling, then
            # is rounded once into e4m3 (per-column scaling; see _to_fp8)
            W = ops.new_block(self.A_mv.rows, k, FpFormat.F32 if fp8 else self.mv.storage, self.device)
            ops.gemm_av(self.A_mv, X, W, colmax=colmax, flags=st[S_MV_FLAGS:S_MV_FLAGS + 1],
                        **({"oz": self._block_oz(self.A_mv, X), "levels": levels}
                           if self.ops is _ops else {}))
            self.stats.a_passes += 1
            comm.all_reduce_max_(colmax)
            ops.scale_columns(W, colmax, self.mv.compute)
            if fp8:
                W = self._to_fp8(W, st)
            if comm.distributed:
                Xn = ops.new_block(self.n, k, self.mv.storage, self.device)
                comm.all_gather_rows(W.t, Xn.t, self.n, k)
                X = Xn
            else:
                X = W
        return X

    def _to_fp8(self, W, st):
        """An inf-norm-scaled fp32 block rounded once into e4m3 (the FP8 rung's storage)."""
        X8 = self.ops.new_block(W.n, W.k, FpFormat.FP8_E4M3, self.device)
        self.ops.convert(W, X8, flags=st[S_MV_FLAGS:S_MV_FLAGS + 1])
        return X8

    def power_from(self, W, eig, kp: int, st, made=None):
        """A-pass reuse (cfg.reuse_av): the restart block is Ut = U Y, so its MatVec is
        A Ut = (A U) Y = W Y with W the projection's block product (kept in its accumulation
        format): X = round(W Y) to the MatVec storage, inf-norm scaled (ofrr/driver.py:
        102-105), then the remaining cfg.iter - 1 MatVecs with A.  Same iterate as the
        reference's A round(Ut) up to the rounding of Ut and the accumulation error of W."""
        import torch
        ops, comm = self.ops, self.comm
        fp8 = self.mv.storage == FpFormat.FP8_E4M3
        if made is not None:                      # W Y and its column norms from K6f (project)
            X, colmax = made
        else:
            colmax = torch.zeros(kp, dtype=torch.float64, device=self.device)
            X = ops.reuse_power(W, eig.vectors, kp, eig.n_out, kp, FpFormat.F32 if fp8 else self.mv.storage, colmax,
                                flags=st[S_MV_FLAGS:S_MV_FLAGS + 1])
        comm.all_reduce_max_(colmax)
        ops.scale_columns(X, colmax, self.mv.compute)
        if fp8:
            X = self._to_fp8(X, st)
        if comm.distributed:
            Xn = ops.new_block(self.n, kp, self.mv.storage, self.device)
            comm.all_gather_rows(X.t, Xn.t, self.n, kp)
            X = Xn
        if self.cfg.iter > 1:
            X = self.power(X, st, steps=self.cfg.iter - 1)
        return X

    def basis(self, X, st):
        """Hessenberg basis (K3), or a Gram-Schmidt comparator (csrc/gs.cu); redundant on
        every rank."""
        if self.cfg.basis_method in GRAM_SCHMIDT_METHODS:
            h = self.ops.orthonormalize(X, self.cfg.basis_method.value, self.pol.storage, self.pol.compute,
                                        self.pol.accumulate, self.pol.drop_tol)
        else:
            if self.ops is _ops:                 # the kept count straight into the status word
                return self.ops.hessenberg(X, self.pol.storage, self.pol.compute, self.pol.drop_tol,
                                           n_kept_out=st[S_NKEPT:S_NKEPT + 1])
            h = self.ops.hessenberg(X, self.pol.storage, self.pol.compute, self.pol.drop_tol)
        st[S_NKEPT:S_NKEPT + 1].copy_(h.n_kept)
        return h

    def _proj_levels_for(self, lead: bool) -> int:
        lv = self.pol.product_levels
        return LEAD_LEVELS if (lead and lv == 6 and LEAD_LEVELS in (5, 6)) else lv

    def _proj_levels(self) -> int:
        """Ozaki levels of this iteration's projection product (see LEAD_LEVELS)."""
        lv = self.pol.product_levels
        if getattr(self, "_entry_iter", False) and lv == 4 and self.pol.storage == FpFormat.F64:
            return FIRST_PROJ_LEVELS if FIRST_PROJ_LEVELS in (3, 4) else lv
        if getattr(self, "_entry_iter", False) and lv == 4 and self.pol.storage == FpFormat.F32:
            return START_PROJ_LEVELS if START_PROJ_LEVELS in (2, 4) else lv
        return LEAD_LEVELS if (getattr(self, "_lead", False) and lv == 6 and LEAD_LEVELS in (5, 6)) else lv

    def project(self, U, st, want64: bool, top_check: Optional[int] = None, reuse: bool = False):
        """ofrr_eig (ofrr/projection.py:75-87) + restart block (ofrr/driver.py:109).

        With ``top_check`` the block product also keeps W = A U in its accumulation
        format (fp32 on the tensor cores) and the residual estimate of the leading
        pairs is formed from it (K7e) -- no extra pass over A."""
        ops, comm = self.ops, self.comm
        kp = U.k
        fp8 = self.pol.storage == FpFormat.FP8_E4M3
        W2 = None
        if fp8:
            # e4m3 storage: W = A U stays in its fp32 accumulation format (A U exceeds e4m3's
            # 448 long before the basis does), the Grams are formed from U widened to fp32
            # (exact) and that W
            W = ops.new_block(self.A_pol.rows, kp, FpFormat.F32, self.device)
            ops.gemm_av(self.A_pol, U, W, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1],
                        **({"levels": self.pol.product_levels} if self.ops is _ops else {}))
            W2 = W if (top_check is not None or reuse) else None
            U8 = U
            U = ops.new_block(U8.n, kp, FpFormat.F32, self.device)
            ops.convert(U8, U)
        else:
            W = ops.new_block(self.A_pol.rows, kp, self.pol.storage, self.device)
            if top_check is not None or reuse:
                acc = FpFormat.F64 if FpFormat.F64 in (self.A_pol.fmt, U.fmt) else FpFormat.F32
                W2 = ops.new_block(self.A_pol.rows, kp, acc, self.device)
            ops.gemm_av(self.A_pol, U, W, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1], W2=W2,
                        **({"oz": self._block_oz(self.A_pol, U), "levels": self._proj_levels()}
                           if self.ops is _ops else {}))
        self.stats.a_passes += 1
        self._last_w2 = W2
        self._last_w2_levels = self._proj_levels() if W2 is not None and W2.fmt == FpFormat.F64 else 6
        Ul = _row_slice(U, self.r0, self.r1) if comm.distributed else U
        classical = self.cfg.projection == "rr"       # rr_eig (ofrr/projection.py:64-72): no mass matrix
        if comm.distributed:
            B, _ = ops.gram(Ul, W, self.proj_out, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1], want_m=False)
            comm.all_reduce_sum_(B)
            M = None if classical else ops.gram(U, None, self.proj_out, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1])[1]
        else:
            B, M = ops.gram(U, W, self.proj_out, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1], want_m=not classical)
        side = self._fork_res_scales()
        if classical or ops is not _ops:
            eig = ops.sym_eig(B, kp) if classical else ops.sym_def_gen_eig(B, M, kp)
            st[S_EIG_STATUS:S_EIG_STATUS + 1].copy_(eig.status)
            st[S_NOUT:S_NOUT + 1].copy_(eig.n_out)
        else:                                    # status and count straight into the status word
            eig = ops.sym_def_gen_eig(B, M, kp, n_out_out=st[S_NOUT:S_NOUT + 1],
                                      status_out=st[S_EIG_STATUS:S_EIG_STATUS + 1])
        if (not comm.distributed and hasattr(ops, "restart") and W2 is not None and W2.n == U.n and kp <= 256
                and (reuse or top_check is not None)):
            # K6f: Ritz block, next power step and residual estimate in one pass over (U, W2)
            import torch
            mv8 = self.mv.storage == FpFormat.FP8_E4M3
            colmax = torch.zeros(kp, dtype=torch.float64, device=self.device) if reuse else None
            U64, Xn, Xw, est = ops.restart(
                U, W2 if (reuse or top_check is not None) else None, eig.vectors, kp, eig.n_out, kp, want64=want64,
                xu_fmt=self.mv.storage, flags_u=st[S_RESTART_FLAGS:S_RESTART_FLAGS + 1],
                xw_fmt=(FpFormat.F32 if mv8 else self.mv.storage) if reuse else None, colmax=colmax,
                flags_w=st[S_MV_FLAGS:S_MV_FLAGS + 1], vals=eig.values if top_check is not None else None,
                t=min(top_check, kp) if top_check is not None else 0, mode=0)
            Xp = self.power_from(W2, eig, kp, st, made=(Xw, colmax)) if reuse else None
            self._join(side)
            if reuse:
                return eig, U64, Xn, est, Xp
            return eig, U64, Xn, est
        U64, Xn = ops.ritz(U, eig.vectors, kp, eig.n_out, kp, 1.0, want64=want64, x_fmt=self.mv.storage,
                           flags=st[S_RESTART_FLAGS:S_RESTART_FLAGS + 1])
        est = None
        if W2 is not None and top_check is not None:
            t = min(top_check, kp)
            est = ops.residual_estimate(Ul, W2, eig.vectors, kp, eig.values, eig.n_out, t,
                                        mode=2 if comm.distributed else 0)
            if comm.distributed:
                comm.all_reduce_sum_(est)                      # sums of squares over the row blocks
                est = _relative(est, eig.values, t)
        Xp = self.power_from(W2, eig, kp, st) if reuse else None
        self._join(side)
        if reuse:
            return eig, U64, Xn, est, Xp
        return eig, U64, Xn, est

    def _fork_res_scales(self):
        """Launch the row-scale pass of the FP64 report's operator on a side stream (it
        overlaps the single-SM pencil solve) -- in the first iteration of a run only (its own
        CUDA graph); returns the stream to join, or None."""
        if self._res_oz is None or not self._refresh_now:
            return None
        import torch
        main = torch.cuda.current_stream(self.device)
        side = torch.cuda.Stream(self.device) if not hasattr(self, "_side") else self._side
        self._side = side
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self._res_oz.refresh()
        return side

    def _join(self, side) -> None:
        if side is not None:
            import torch
            torch.cuda.current_stream(self.device).wait_stream(side)

    def residuals(self, U64, vals, r_dev, r):
        """FP64 ||A u - lambda u|| / |lambda| for the first r pairs (K7)."""
        import torch
        ops, comm = self.ops, self.comm
        A = self.a.residual_operator(self.A_mv.fmt) if hasattr(self.a, "residual_operator") else self.A_mv
        oz = self._ozaki(A)
        if not comm.distributed:
            if oz is not None:
                res = torch.zeros(max(r, 1), dtype=torch.float64, device=self.device)
                return ops.ozaki_residual(oz, U64, U64, vals, r_dev, r, res, 0)
            return ops.residual_eig(A, U64, vals, r_dev, r)
        res = torch.zeros(r, dtype=torch.float64, device=self.device)
        Yl = _row_slice(U64, self.r0, self.r1)
        if oz is not None:
            ops.ozaki_residual(oz, U64.narrow(r), Yl.narrow(r), vals, r_dev, r, res, 2)
        else:
            ops.residual_pair(A, False, U64.narrow(r), Yl.narrow(r), vals, r_dev, r, res, accumulate_max=2)
        comm.all_reduce_sum_(res)                              # sums of squares over the row blocks
        return _relative(res, vals, r)

    def finish_residuals(self, res, vals_np):
        return res.cpu().numpy()

    # ---- the outer loop -----------------------------------------------------------------
    def run(self, X0=None, stop_estimate: Optional[float] = None, stepped: bool = False):
        """The outer loop (ofrr/driver.py:101-111).  With cfg.tol the loop stops at the
        first iteration whose leading `top` residuals pass: the cheap estimate (K7e)
        nominates, the FP64 residual report (K7) confirms; the returned residuals are
        always the FP64 ones.

        Ladder rung (``stop_estimate``): return the restart block (no report) as soon as
        the estimate falls below ``stop_estimate`` or stalls; ``X0`` starts from a block.
        With A-pass reuse the rung hands over the NEXT iterate (its MatVec W Y, already made)
        in ``self.handover`` and the next rung starts with ``stepped=True``: its first
        iteration skips the power step (one FP64-accurate A pass fewer per ladder solve)."""
        self.stepped = bool(stepped)
        self._entered_from_block = X0 is not None and not self.stepped   # (FIRST_POWER_LEVELS)
        cfg = self.cfg
        tol, top = cfg.tol, (cfg.top or cfg.k)
        check = tol is not None
        fresh = X0 is None
        if fresh:
            X = None                                  # made below (into the loop graph's input when it runs)
        elif X0.fmt != self.mv.storage:
            X = self.ops.new_block(X0.n, X0.k, self.mv.storage, self.device)
            self.ops.convert(X0, X)                               # exact widening (f32 -> f64)
        else:
            X = X0
        eig = U64 = U = None
        r = 0
        rs = vals = None
        use_graph = self._graph_capable()
        prev_est = None
        if (X.fmt if X is not None else self.mv.storage) == FpFormat.F64:
            with _ph("ozaki_prepare"):
                self._ozaki(self.A_mv)               # FP64 blocks: slice A once per run, eagerly
        if self.mv.storage != self.pol.storage:
            self._ozaki(self.A_pol) if self.pol.storage == FpFormat.F64 else None
        if use_graph and DEVICE_LOOP and check and stop_estimate is None and (fresh or X.k == cfg.k) and cfg.m >= 2:
            with _ph("device_loop"):
                rs = self._device_loop(X, top)
            if rs is not None:
                return rs
        if (use_graph and DEVICE_LOOP and check and stop_estimate is not None and (fresh or X.k == cfg.k)
                and cfg.m >= 2 and not self.comm.distributed):
            with _ph("device_rung"):
                Xr = self._device_rung(X, top, stop_estimate)
            if Xr is not None:
                return Xr
        if X is None:
            X = self.start_block()
        for it in range(cfg.m):
            last = it == cfg.m - 1
            self._refresh_now = it == 0      # A's report scales: once per run (A may change between runs)
            # one iteration: power step(s), Hessenberg basis, projection with every column
            # (the basis keeps all k in the common case; dropped columns of Q are zero),
            # residual estimate -- replayed as one CUDA graph when possible.  One host sync.
            first = it == 0 and not self.stepped
            lead = it == 0 and self.stepped
            with _ph("graph_step"):
                out = self._graph_step(X, check, top, first, lead) if use_graph and X.k == cfg.k else None
            if out is None:
                with _ph("eager_body"):
                    out = self._body(X, check, top, first, lead)
                if use_graph:
                    _WARM.add(self._graph_key(check, top, first, lead))
            st, h, U, eig, Xn, est = out["st"], out["h"], out["U"], out["eig"], out["Xn"], out["est"]
            kp = U.k
            with _ph("iteration_sync"):
                s, vals_all, est_np = self._unpack(out, st, eig, est)      # the iteration's one sync
            if s[S_MV_FLAGS] & 1:
                raise OverflowDiagnostic("non-finite entries after MatVec")
            if s[S_NKEPT] == 0:
                raise EmptyBasisError("all columns skipped in Hessenberg process")
            if s[S_NKEPT] < kp:                                    # rare: redo with the kept width
                kp = int(s[S_NKEPT])
                U = h.Q.narrow(kp)
                st[S_EIG_STATUS:].zero_()                     # gram/pencil/restart slots
                res = self.project(U, st, want64=False, top_check=(top if check else None), reuse=cfg.reuse_av)
                eig, _, Xn, est = res[:4]
                out = dict(out, Xnext=res[4] if cfg.reuse_av else None, W2=self._last_w2, graph=None,
                           w2_levels=self._last_w2_levels)
                s, vals_all, est_np = self._fetch(st, eig.values, est)
            _raise_for(s, "projection")
            r = int(s[S_NOUT])
            vals = vals_all[:r]
            X = Xn.narrow(r)
            Xrestart = X                                           # the reference's restart block
            if cfg.reuse_av:
                X = out["Xnext"].narrow(r)                         # its MatVec, already made
            U64 = None
            self.stats.iterations = it + 1
            if check:
                e = self._finish(est_np, vals)
                worst = float(np.max(e[: min(top, r)])) if r >= top else float("inf")
                # the estimate comes from W in the accumulation format: near its own noise
                # floor it can stall above a tolerance the FP64 residuals already meet, so a
                # stalled estimate within 16x of tol is confirmed in FP64 as well
                stalled = prev_est is not None and worst > 0.5 * prev_est and worst < 16.0 * tol
                if stop_estimate is not None:
                    rung_done = worst < stop_estimate or (prev_est is not None and worst > 0.5 * prev_est)
                    prev_est = worst
                    self.stats.history.append((it + 1, worst))
                    if rung_done and not last:
                        self.handover = X if cfg.reuse_av else None    # the next iterate, power step made
                        return Xrestart                            # next rung starts from here
                    continue
                prev_est = worst
                if worst < tol or stalled or last:
                    with _ph("final_report"):
                        rs = self._final_report(out, U, eig, kp, r, vals, check, top)   # FP64 confirmation
                    worst = float(np.max(rs.residuals[: min(top, r)])) if r >= top else float("inf")
                    self.stats.history.append((it + 1, worst))
                    if worst < tol:
                        self.stats.converged = True
                        break
                else:
                    self.stats.history.append((it + 1, worst))
        if rs is None:
            rs = self._final_report(out, U, eig, U.k, r, vals, check, top)
        return rs

    def _device_loop(self, X, top: int):
        """The whole outer loop as one CUDA graph with device-side control flow (csrc/loop.cu):
        the first iteration's graph, then the steady iteration graph inside a conditional
        WHILE node, the FP64 report inside a conditional IF node -- the host launches once
        and reads the control block once.  Needs the three graphs captured by earlier solves
        of the same shapes; returns None when they are missing or the device stopped for a
        case the host loop handles (errors, a narrowed basis), and the caller then runs the
        host loop from the same start block (deterministic: same result)."""
        import ctypes
        import time
        import torch
        from . import _lib
        t0 = time.perf_counter()
        cfg = self.cfg
        L = _lib.load()
        self._refresh_now = True
        kf = self._graph_key(True, top, not self.stepped, self.stepped)
        self._refresh_now = False
        ks = self._graph_key(True, top, False)
        gf, gs = _GRAPHS.get(kf), _GRAPHS.get(ks)
        if gf is None or gs is None or gs.report is None or gf.outs.get("est") is None:
            _loop_debug("graphs missing", gf is None, gs is None, gs is not None and gs.report is None)
            return None
        _GRAPHS.move_to_end(kf)
        _GRAPHS.move_to_end(ks)
        # the exec clones gf's and gs's nodes (raw pointers into their buffers): the cache entry
        # holds gf itself, and an entry built from another gf (evicted and recaptured) is stale
        lk = (cfg.m, top, float(cfg.tol))
        loops = gs.__dict__.setdefault("loops", {})
        ent = loops.get(lk)
        if ent is not None and ent[0] is not gf:
            loops.pop(lk)
            ent = None
        lp = ent[1] if ent is not None else None
        if ent is None:
            ctl = torch.zeros(int(L.ofrr_loop_ctl_bytes()), dtype=torch.uint8, device=self.device)
            if gf is gs:
                src = dst = None
                nbytes = 0
            else:
                src_blk = gf.outs["Xnext"] if cfg.reuse_av else gf.Xs
                src, dst = src_blk.t.data_ptr(), gs.Xs.t.data_ptr()
                nbytes = gs.Xs.t.numel() * gs.Xs.t.element_size()
                if src_blk.t.numel() != gs.Xs.t.numel():
                    return None
            ex = ctypes.c_void_p()
            rc = L.ofrr_loop_build(gf.graph.raw_cuda_graph(), gs.graph.raw_cuda_graph(),
                                   gs.report.graph.raw_cuda_graph(), gf.outs["st"].data_ptr(),
                                   gf.outs["est"].data_ptr(), gs.outs["st"].data_ptr(), gs.outs["est"].data_ptr(),
                                   gs.report.res.data_ptr(), src, dst, nbytes, ctl.data_ptr(), cfg.m, top, cfg.k,
                                   float(cfg.tol), ctypes.byref(ex))
            if rc != 0:
                _loop_debug("build failed", _lib.last_error())   # the host loop takes over
                loops[lk] = (gf, None)
                return None
            lp = (_LoopExec(ex.value), ctl)
            loops[lk] = (gf, lp)
        elif lp is None:
            return None
        ex, ctl = lp
        t1 = time.perf_counter()
        if X is None and (gf.Xs.n, gf.Xs.k, FpFormat(gf.Xs.fmt)) == (self.n, cfg.k, FpFormat(self.mv.storage)):
            self.start_block(out=gf.Xs)                # straight into the loop graph's input
        elif X is None:
            gf.Xs.t.copy_(self.start_block().t)
        elif X.t.data_ptr() != gf.Xs.t.data_ptr():
            gf.Xs.t.copy_(X.t)
        t2 = time.perf_counter()
        with _ph("loop_launch"):
            _lib.check(L.ofrr_loop_launch(ex.handle, ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)),
                       "loop_launch")
        t3 = time.perf_counter()
        # the solve's one synchronisation: control block, values and FP64 residuals in one
        # pinned buffer
        k = cfg.k
        nb = ctl.numel()
        stage = gs.__dict__.get("stage")
        if stage is None:
            stage = gs.stage = torch.empty(nb + 8 * (2 * k), dtype=torch.uint8, pin_memory=True)
        stage[:nb].copy_(ctl, non_blocking=True)
        stage[nb:nb + 8 * k].view(torch.float64).copy_(gs.outs["pack"][8:8 + k], non_blocking=True)
        stage[nb + 8 * k:].view(torch.float64).copy_(gs.report.res[:k], non_blocking=True)
        rg = gs.report
        U64t = rg.U64.t.clone()                        # the returned vectors outlive the next replay
        with _ph("loop_sync"):
            torch.cuda.current_stream(self.device).synchronize()
        host = stage
        t4 = time.perf_counter()
        head = host[:16].view(torch.int32).numpy()
        state, its = int(head[0]), int(head[1])
        if state not in (1, 2):
            _loop_debug("device stopped for the host", state, its)
            return None
        hist = host[24:nb].view(torch.float64).numpy()
        nh = (hist.size) // 2
        est_h, fp64_h = hist[:nh], hist[nh:]
        _loop_debug("est", est_h[:its].tolist(), "fp64", fp64_h[:its].tolist())
        vals = host[nb:nb + 8 * k].view(torch.float64).numpy().copy()
        res = host[nb + 8 * k:].view(torch.float64).numpy().copy()
        self.stats.iterations = its
        self.stats.a_passes += gf.a_passes + (its - 1) * gs.a_passes
        for i in range(min(its, nh)):
            self.stats.history.append((i + 1, float(fp64_h[i]) if fp64_h[i] >= 0 else float(est_h[i])))
        self.stats.converged = state == 1
        self.stats.device_loop = True
        # launch / GEMM-log accounting of what ran on the device (bench.py gpu_launches, roofline)
        nrep = int(np.sum(fp64_h[:min(its, nh)] >= 0))
        gf.rec.replayed()
        for _ in range(its - 1):
            gs.rec.replayed()
        for _ in range(nrep):
            rg.rec.replayed()
        self.ops._count(1 + its + nrep)                      # init, decide per iteration, confirm per report
        U64c = self.ops.DevBlock(U64t, rg.U64.n, k, rg.U64.fmt)
        out = RitzSet(np.array(vals), DenseMatrix.from_block(U64c), "eig", residuals=res)
        t5 = time.perf_counter()
        _loop_debug(f"host us: keys {1e6 * (t1 - t0):.0f} copy {1e6 * (t2 - t1):.0f} launch {1e6 * (t3 - t2):.0f} "
                    f"sync {1e6 * (t4 - t3):.0f} post {1e6 * (t5 - t4):.0f}")
        return out

    def _device_rung(self, X, top: int, sw: float):
        """A ladder rung's outer loop as one CUDA graph (csrc/loop.cu loop_build_rung): the
        first and steady iteration graphs, the rung's stop test on the device (the host loop's
        `rung_done`, same thresholds), one launch and one read.  Returns the restart block
        (and sets self.handover) when the rung finished; None when the graphs are missing or
        the device stopped for a case the host loop handles -- the caller then runs the host
        loop from the same start block (the graphs' input copies leave X untouched)."""
        import ctypes
        import torch
        from . import _lib
        cfg = self.cfg
        L = _lib.load()
        self._refresh_now = True
        kf = self._graph_key(True, top, not self.stepped, self.stepped)
        self._refresh_now = False
        ks = self._graph_key(True, top, False)
        gf, gs = _GRAPHS.get(kf), _GRAPHS.get(ks)
        if gf is None or gs is None or gf.outs.get("est") is None or gs.outs.get("est") is None:
            return None
        _GRAPHS.move_to_end(kf)
        _GRAPHS.move_to_end(ks)
        lk = ("rung", cfg.m, top, float(sw))
        loops = gs.__dict__.setdefault("loops", {})
        ent = loops.get(lk)
        if ent is not None and ent[0] is not gf:
            loops.pop(lk)
            ent = None
        lp = ent[1] if ent is not None else None
        if ent is None:
            ctl = torch.zeros(int(L.ofrr_loop_ctl_bytes()), dtype=torch.uint8, device=self.device)
            if gf is gs:
                src = dst = None
                nbytes = 0
            else:
                src_blk = gf.outs["Xnext"] if cfg.reuse_av else gf.Xs
                src, dst = src_blk.t.data_ptr(), gs.Xs.t.data_ptr()
                nbytes = gs.Xs.t.numel() * gs.Xs.t.element_size()
                if src_blk.t.numel() != gs.Xs.t.numel():
                    return None
            ex = ctypes.c_void_p()
            rc = L.ofrr_loop_build_rung(gf.graph.raw_cuda_graph(), gs.graph.raw_cuda_graph(), gf.outs["st"].data_ptr(),
                                        gf.outs["est"].data_ptr(), gs.outs["st"].data_ptr(), gs.outs["est"].data_ptr(),
                                        src, dst, nbytes, ctl.data_ptr(), cfg.m, top, cfg.k, float(sw),
                                        ctypes.byref(ex))
            if rc != 0:
                _loop_debug("rung build failed", _lib.last_error())
                loops[lk] = (gf, None)
                return None
            lp = (_LoopExec(ex.value), ctl)
            loops[lk] = (gf, lp)
        elif lp is None:
            return None
        ex, ctl = lp
        if X is None and (gf.Xs.n, gf.Xs.k, FpFormat(gf.Xs.fmt)) == (self.n, cfg.k, FpFormat(self.mv.storage)):
            self.start_block(out=gf.Xs)
        elif X is None:
            gf.Xs.t.copy_(self.start_block().t)
        elif X.t.data_ptr() != gf.Xs.t.data_ptr():
            gf.Xs.t.copy_(X.t)
        _lib.check(L.ofrr_loop_launch(ex.handle, ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)),
                   "loop_launch")
        nb = ctl.numel()
        stage = gs.__dict__.get("stage_rung")
        if stage is None:
            stage = gs.stage_rung = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        stage.copy_(ctl, non_blocking=True)
        with _ph("rung_sync"):
            torch.cuda.current_stream(self.device).synchronize()
        head = stage[:16].view(torch.int32).numpy()
        state, its = int(head[0]), int(head[1])
        if state != 4:
            _loop_debug("rung: device stopped for the host", state, its)
            return None
        hist = stage[24:nb].view(torch.float64).numpy()
        est_h = hist[:hist.size // 2]
        self.stats.iterations = its
        self.stats.a_passes += gf.a_passes + (its - 1) * gs.a_passes
        for i in range(min(its, est_h.size)):
            self.stats.history.append((i + 1, float(est_h[i])))
        gf.rec.replayed()
        for _ in range(its - 1):
            gs.rec.replayed()
        self.ops._count(1 + its)                                 # init, decide per iteration
        self.stats.device_loop = True
        out = gf.outs if its == 1 else gs.outs
        r = cfg.k                                                # the device stops for the host otherwise
        self.handover = out["Xnext"].narrow(r) if cfg.reuse_av else None
        return out["Xn"].narrow(r)

    def _final_report(self, out, U, eig, kp, r, vals, check, top) -> RitzSet:
        """Ritz vectors in fp64 and the FP64 residual report -- replayed as a CUDA graph when
        the iteration came from one (full width), eager otherwise."""
        import torch
        g = out.get("graph")
        if g is not None and kp == U.k == r == self.cfg.k:
            rg = g.report
            if rg is None:
                rg = self._capture_report(g, U, eig, kp, r)
            if rg is not None:
                rg.graph.replay()
                rg.rec.replayed()
                res = rg.res.cpu().numpy()[:r]
                U64 = rg.U64
                U64c = self.ops.DevBlock(U64.t.clone(), U64.n, r, U64.fmt)   # outlive the next replay
                return RitzSet(np.array(vals[:r]), DenseMatrix.from_block(U64c), "eig", residuals=res)
        W2 = out.get("W2")
        if self._w2_is_fp64(W2, U, out.get("w2_levels", 6)):
            U64, res = self._report_from_w(U, W2, eig, kp, r)
            rs = RitzSet(np.array(vals[:r]), DenseMatrix.from_block(U64.narrow(r)), "eig")
            return RitzSet(rs.values, rs.vectors, "eig", residuals=res.cpu().numpy()[:r])
        U64, _ = self.ops.ritz(U, eig.vectors, kp, eig.n_out, kp, 1.0, want64=True)
        return self.report(U64, eig, r, vals)

    def _report_from_w(self, U, W2, eig, kp: int, r: int):
        """fp64 Ritz vectors U Y and their FP64 residuals from an FP64-accurate W2 = A U: one
        K6f pass (U64 + the residual sums) on one process, K6 + K7e otherwise."""
        if not self.comm.distributed and hasattr(self.ops, "restart") and kp <= 256 and W2.n == U.n:
            U64, _, _, res = self.ops.restart(U, W2, eig.vectors, kp, eig.n_out, kp, want64=True,
                                             vals=eig.values, t=r, mode=0)
            return U64, res
        U64, _ = self.ops.ritz(U, eig.vectors, kp, eig.n_out, kp, 1.0, want64=True)
        return U64, self.residuals_from_w(U, W2, eig, r)

    def _w2_is_fp64(self, W2, U, levels: int = 6) -> bool:
        """W2 = A U is an FP64-accurate product (fp64 block, full-accuracy K7z or fp64 FMA)."""
        return (W2 is not None and W2.fmt == FpFormat.F64 and W2.k >= U.k and self.pol.product_levels == 6
                and levels == 6)

    def residuals_from_w(self, U, W2, eig, r: int):
        """FP64 residuals ||A u_j - lambda_j u_j|| / |lambda_j| of the Ritz vectors u_j = U y_j
        when the projection's W2 = A U is itself an FP64-accurate product (fp64 blocks: K7z on
        a 16/8-bit operator, fp64 FMA otherwise): A u_j = W2 y_j, so the report is
        ||(W2 - lambda_j U) y_j|| / |lambda_j| in fp64 (K7e with fp64 operands) -- no further
        pass over A.  Row-partitioned: sums of squares all-reduced, finished on the device."""
        ops, comm = self.ops, self.comm
        Ul = _row_slice(U, self.r0, self.r1) if comm.distributed else U
        res = ops.residual_estimate(Ul, W2, eig.vectors, U.k, eig.values, eig.n_out, r,
                                    mode=2 if comm.distributed else 0)
        if comm.distributed:
            comm.all_reduce_sum_(res)
            res = _relative(res, eig.values, r)
        return res

    def _capture_report(self, g, U, eig, kp, r):
        import torch
        rec = self.ops.Recorder()
        graph = torch.cuda.CUDAGraph(keep_graph=True)
        torch.cuda.synchronize(self.device)
        try:
            with rec:
                with torch.cuda.graph(graph):
                    W2 = g.outs.get("W2")
                    if self._w2_is_fp64(W2, U, g.outs.get("w2_levels", 6)):
                        U64, res = self._report_from_w(U, W2, eig, kp, r)
                    else:
                        U64, _ = self.ops.ritz(U, eig.vectors, kp, eig.n_out, kp, 1.0, want64=True)
                        res = self.residuals(U64, eig.values, eig.n_out, r)
        except Exception:
            g.report = None
            return None
        g.report = _ReportGraph(graph, U64, res, rec)
        return g.report

    # ---- one outer iteration: eager body, or a replayed CUDA graph of it -----------------
    def _body(self, X, check: bool, top: int, first: bool = True, lead: bool = False) -> dict:
        """One outer iteration.  With cfg.reuse_av the input of every iteration but the
        first is already the power-stepped block (the previous projection made it)."""
        import torch
        st = torch.zeros(8, dtype=torch.int32, device=self.device)
        reuse = self.cfg.reuse_av
        lv = None
        if (first and self.mv.storage == FpFormat.F64 and self.mv.product_levels == 4 and X.fmt == FpFormat.F64
                and FIRST_POWER_LEVELS in (3, 4) and self.ops is _ops and X.k == self.cfg.k
                and getattr(self, "_entered_from_block", False)):
            lv = FIRST_POWER_LEVELS
        elif (first and self.mv.storage == FpFormat.F32 and self.mv.product_levels == 4   # the lite fp32 rung
              and self.A_mv.fmt == FpFormat.BF16 and self.ops is _ops
              and not self.stepped and not getattr(self, "_entered_from_block", False)
              and START_SLICES_LEVELS in (2, 4, 6)):
            lv = START_SLICES_LEVELS
        Xp = self.power(X, st, levels=lv) if (first or not reuse) else X
        self._entry_iter = lv is not None
        h = self.basis(Xp, st)
        U = h.Q.narrow(Xp.k)
        Xnext = None
        self._lead = lead
        try:
            if reuse:
                eig, _, Xn, est, Xnext = self.project(U, st, want64=False, top_check=(top if check else None),
                                                      reuse=True)
            else:
                eig, _, Xn, est = self.project(U, st, want64=False, top_check=(top if check else None))
        finally:
            self._lead = False
            self._entry_iter = False
        out = dict(st=st, h=h, U=U, eig=eig, Xn=Xn, est=est, pack=None, Xnext=Xnext, W2=self._last_w2,
                   w2_levels=self._last_w2_levels)
        if self.comm.distributed:
            self.comm.all_reduce_max_(st)        # every rank sees (and raises) the same status
        parts = [st.to(torch.float64), eig.values.reshape(-1).to(torch.float64)]
        if est is not None:
            parts.append(est.reshape(-1).to(torch.float64))
        out["pack"] = torch.cat(parts)
        return out

    def _unpack(self, out, st, eig, est):
        """The iteration's single device->host read (status word, values, estimates)."""
        if out["pack"] is None:
            return self._fetch(st, eig.values, est)
        host = out["pack"].cpu().numpy()
        _prof_collect(out)
        k = eig.values.numel()
        return host[:8].astype(np.int64), host[8:8 + k], (host[8 + k:] if est is not None else None)

    def _graph_capable(self) -> bool:
        """CUDA graphs (and the device-side loop) need capturable collectives when the rows are
        partitioned: NCCL; gloo (CPU tests, host-staged) runs eagerly."""
        import os
        return (self.ops is _ops and self.device.type == "cuda"
                and (not self.comm.distributed or self.comm.graphable)
                and os.environ.get("OFRR_CUDA_GRAPHS", "1") != "0")

    def _graph_key(self, check: bool, top: int, first: bool = True, lead: bool = False):
        A, B = self.A_mv, self.A_pol
        pol = lambda p: (int(p.storage), int(p.compute), int(p.accumulate), float(p.drop_tol),  # noqa: E731
                         int(p.product_levels))
        from . import _lib
        return (A.t.data_ptr(), A.rows, A.cols, A.lda, int(A.fmt), B.t.data_ptr(), B.rows, B.cols, B.lda, int(B.fmt),
                self.n, self.cfg.k, self.cfg.iter, pol(self.pol), pol(self.mv), check, top, self.device.index,
                bool(_lib.load().ofrr_prof_gemm_active()), self._refresh_now and self._res_oz is not None,
                self.cfg.reuse_av, first or not self.cfg.reuse_av, bool(lead) and self._proj_levels_for(lead) != 6,
                bool(first and getattr(self, "_entered_from_block", False)),
                # what else shapes the captured body: basis builder, projection, row partition
                str(self.cfg.basis_method.value), str(self.cfg.projection), bool(self.comm.distributed),
                int(getattr(self, "r0", 0)), int(getattr(self, "r1", 0)), id(self.ops),
                # Ozaki workspaces the captured kernels read (made outside the capture)
                tuple(sorted(oz.ws.data_ptr() for oz in self._oz.values())))

    def _graph_step(self, X, check: bool, top: int, first: bool = True, lead: bool = False):
        """Replay the captured iteration (capturing it first once the shapes have run
        eagerly in this process); None -> run it eagerly."""
        key = self._graph_key(check, top, first, lead)
        g = _GRAPHS.get(key)
        if g is None:
            if key not in _WARM or key in _NO_GRAPH:
                return None
            g = self._capture(X, check, top, key, first, lead)
            if g is None:
                return None
        else:
            _GRAPHS.move_to_end(key)
        if X.t.data_ptr() != g.Xs.t.data_ptr():
            g.Xs.t.copy_(X.t)
        g.graph.replay()
        g.rec.replayed()
        self.stats.a_passes += g.a_passes
        out = dict(g.outs)
        out["prof_group"] = g.prof_group
        out["graph"] = g
        return out

    def _capture(self, X, check: bool, top: int, key, first: bool = True, lead: bool = False):
        import torch
        from . import _lib
        L = _lib.load()
        Xs = self.ops.new_block(self.n, self.cfg.k, self.mv.storage, self.device)
        Xs.t.copy_(X.t)
        rec = self.ops.Recorder()
        graph = torch.cuda.CUDAGraph(keep_graph=True)     # the raw graph also feeds the device loop
        torch.cuda.synchronize(self.device)
        passes0 = self.stats.a_passes
        try:
            with rec:
                with torch.cuda.graph(graph):
                    outs = self._body(Xs, check, top, first, lead)
                    nxt = outs["Xnext"] if self.cfg.reuse_av else outs["Xn"]
                    if first and self.cfg.reuse_av:
                        pass                                       # input: the start block
                    else:
                        Xs.t.copy_(nxt.t)                          # the next iteration's input
        except Exception:                                             # capture unsupported: stay eager
            _NO_GRAPH.add(key)
            L.ofrr_prof_gemm_collect()
            return None
        prof_group = L.ofrr_prof_gemm_claim() if L.ofrr_prof_gemm_active() else -1
        if not (first and self.cfg.reuse_av):
            outs["Xnext" if self.cfg.reuse_av else "Xn"] = Xs
        g = _IterGraph(graph, Xs, outs, rec, prof_group)
        g.keep = [oz.ws for oz in self._oz.values()]     # buffers captured by reference
        g.a_passes = self.stats.a_passes - passes0       # passes the captured body makes
        self.stats.a_passes = passes0                    # counted again by the replay
        _GRAPHS[key] = g
        while len(_GRAPHS) > _GRAPH_MAX:
            _GRAPHS.popitem(last=False)
        return g

    def _fetch(self, st, *vecs):
        """One device->host read: the status word (max over ranks) and fp64 vectors."""
        import torch
        if self.comm.distributed:
            self.comm.all_reduce_max_(st)
        parts = [st.to(torch.float64)] + [v.reshape(-1).to(torch.float64) for v in vecs if v is not None]
        host = torch.cat(parts).cpu().numpy()
        out = [host[:8].astype(np.int64)]
        off = 8
        for v in vecs:
            if v is None:
                out.append(None)
                continue
            out.append(host[off:off + v.numel()])
            off += v.numel()
        return out

    def _finish(self, r, vals_np):
        """Residual estimates read back (already relative: the row-partitioned path finishes
        its all-reduced sums of squares on the device, _relative)."""
        return r

    def report(self, U64, eig, r: int, vals=None) -> RitzSet:
        if vals is None:
            vals = eig.values[:r].cpu().numpy()
        rs = RitzSet(np.array(vals[:r]), DenseMatrix.from_block(U64.narrow(r)), "eig")
        return self.residual_report(rs, U64, eig, r)

    def residual_report(self, rs: RitzSet, U64, eig, r: int) -> RitzSet:
        """ofrr/driver.py:111 -> ofrr/projection.py:136-147 (FP64, every returned pair)."""
        from dataclasses import replace
        res = self.residuals(U64, eig.values, eig.n_out, r)
        return replace(rs, residuals=self.finish_residuals(res, rs.values)[:r])


def _relative(ss, vals, r: int):
    """||.||^2 all-reduced over the row blocks -> sqrt(ss) / |lambda| (inf for lambda = 0), on
    the device (capturable: the device-side loop compares it with tol)."""
    import torch
    lam = vals.reshape(-1)[:r].abs()
    out = ss.clone()
    head = torch.where(lam == 0, torch.full_like(lam, float("inf")), torch.sqrt(ss[:r]) / lam)
    out[:r].copy_(head)
    return out


def _row_slice(B, r0: int, r1: int):
    """Rows [r0, r1) of a column-major block as a block view (same ld)."""
    import torch
    from .ops import DevBlock
    t = B.t
    # strided view: row j = column j starting at element r0, same leading dimension
    view = torch.as_strided(t, (t.shape[0], B.ld - r0), (B.ld, 1), t.storage_offset() + r0)
    return DevBlock(view, r1 - r0, B.k, B.fmt)


def subspace_iter_eig(a: DenseMatrix, cfg: IterConfig, stats: Optional[RunStats] = None,
                      comm: Optional[Comm] = None, n_global: Optional[int] = None) -> RitzSet:
    """Multi-step subspace iteration with the Hessenberg basis and OFRR projection
    (ofrr/driver.py:84-111), on the device.

    ``a``: the operator (host DenseMatrix uploaded once; or device resident).  In a
    row-partitioned run ``a`` holds this rank's rows and ``n_global`` the full n.
    Thread-safe: concurrent calls are serialised on the device (_SOLVE_LOCK)."""
    with _SOLVE_LOCK:
        return _subspace_iter_eig(a, cfg, stats, comm, n_global)


def _subspace_iter_eig(a, cfg, stats, comm, n_global) -> RitzSet:
    _require_ofrr_path(cfg, "subspace iteration")
    n = int(n_global if n_global is not None else a.rows)
    if cfg.k > n:
        raise ValueError("k exceeds the operator dimension")
    X0 = None
    stepped = False
    prepared = None
    hist, iters, passes = [], 0, 0
    if cfg.ladder is not None:
        prepared = _prepare_ahead(a, cfg, comm)
        # precision ladder: run the cheaper policies while they make
        # progress, each continuing from the previous rung's restart block, then cfg.policy
        from dataclasses import replace as _replace
        rungs = list(cfg.ladder) if isinstance(cfg.ladder, (tuple, list)) else [cfg.ladder]
        switches = list(cfg.ladder_switch) if isinstance(cfg.ladder_switch, (tuple, list)) else [cfg.ladder_switch]
        rung_stats = []
        for pol_r, sw in zip(rungs, switches):
            low = _replace(cfg, policy=pol_r, matvec_policy=None, ladder=None, ladder_switch=1e-3,
                           m=max(1, cfg.m - iters))
            with _ph("rung_low"):
                eng0 = EigEngine(a, low, comm=comm, n_global=n, report_scales=False,
                                 prepared=prepared if FpFormat.F64 == pol_r.storage else None)
                out = eng0.run(X0=X0, stop_estimate=sw, stepped=X0 is not None and stepped)
            if isinstance(out, RitzSet):                               # m exhausted in a low rung
                if stats is not None:
                    stats.__dict__.update(eng0.stats.__dict__)
                    stats.rungs = rung_stats + [(cfg_rung_label(low), eng0.stats.iterations, eng0.stats.a_passes)]
                    stats.iterations += iters
                    stats.a_passes += passes
                    stats.history = hist + [(it + iters, w) for it, w in eng0.stats.history]
                return out
            X0 = out
            # the next rung starts from this rung's next iterate (W Y, power step made) when this
            # rung's products are far below its switch threshold (full-f32-lite at 1e-2,
            # full-f64-lite at 1e-6): otherwise from its Ritz vectors (e.g. the full-f32 rung
            # switches at its own product-accuracy floor, so its W Y would carry that noise)
            stepped = sw >= 100 * _rung_floor(pol_r) and getattr(eng0, "handover", None) is not None
            if stepped or (HANDOVER_STEPPED and getattr(eng0, "handover", None) is not None):
                X0 = eng0.handover
                stepped = True
            hist += [(it + iters, w) for it, w in eng0.stats.history]
            iters += eng0.stats.iterations
            passes += eng0.stats.a_passes
            rung_stats.append((cfg_rung_label(low), eng0.stats.iterations, eng0.stats.a_passes))
        cfg = _replace(cfg, ladder=None, ladder_switch=1e-3, m=max(1, cfg.m - iters))
    with _ph("rung_main"):
        eng = EigEngine(a, cfg, comm=comm, n_global=n, prepared=prepared)
        rs = eng.run(X0=X0, stepped=X0 is not None and stepped)
    if stats is not None:
        stats.__dict__.update(eng.stats.__dict__)
        stats.rungs = (rung_stats if X0 is not None else []) + \
            [(cfg_rung_label(cfg), eng.stats.iterations, eng.stats.a_passes)]
        stats.iterations += iters
        stats.a_passes += passes
        stats.history = hist + [(it + iters, w) for it, w in eng.stats.history]
    return rs


_SIDE_STREAMS = {}


def _rung_floor(pol: PrecisionPolicy) -> float:
    """The residual level a rung's block products can carry (measured at C3): fp32-accumulated
    tensor-core products ~1e-4; the lite fp64 (~30-bit) products ~1e-8; FP64-accurate ~1e-13."""
    if pol.storage == FpFormat.F64:
        return 1e-13 if pol.product_levels == 6 else 1e-8
    return 1e-4


def _prepare_ahead(a, cfg: IterConfig, comm):
    """Ladder to an fp64 policy on a 16/8-bit operator: the FP64-accurate products need A's
    row scales and head/tail split (K7z prepare, one read of A).  A does not change during
    the solve, so the prepare runs on a side stream while the low rung computes; the main
    rung's engine waits for its event.  None when the main rung needs no Ozaki operator."""
    import torch
    if FpFormat.F64 not in (cfg.policy.storage, cfg.mv_policy.storage) or not hasattr(a, "device_operator"):
        return None
    A = operator_for(a, FpFormat.F64)
    if A.fmt not in _ops.OZAKI_FMTS:
        return None
    dev = A.device
    side = _SIDE_STREAMS.get(dev.index)
    if side is None:
        side = _SIDE_STREAMS[dev.index] = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        oz = _ops.OzakiOperator(A)
        ev = torch.cuda.Event()
        ev.record(side)
    return oz, ev


def cfg_rung_label(cfg: IterConfig) -> str:
    """Basis storage format of a rung (RunStats.rungs); F64L: the lite fp64 rung."""
    name = FpFormat(cfg.policy.storage).name
    return name + "L" if cfg.policy.product_levels != 6 else name


# -------------------------------------------------------------------------------------
# SVD (single GPU)
# -------------------------------------------------------------------------------------
class SvdEngine:
    """Device state of subspace_iter_svd / ofrr_svd (ofrr/driver.py:141-173,
    ofrr/projection.py:99-133).  A V and A^T U both run K-major on the tensor cores:
    A^T is kept resident as a second row-major operator."""

    def __init__(self, a: DenseMatrix, pol: PrecisionPolicy, mv: PrecisionPolicy, ops=None,
                 comm: Optional[Comm] = None, n1_global: Optional[int] = None):
        """Row-partitioned: ``a`` holds this rank's rows of the tall A
        (n1_global rows in all); V (n2 x k) is replicated.  Per power step A_p V is local,
        A^T U = sum_p A_p^T U_p is an all-reduce(sum) of fp32 partial products (rounded to
        storage after the sum); the U basis is built redundantly from the all-gathered U, its
        Gram and the cross Gram U^T A V are all-reduced partials; the Ritz vectors U Y stay
        row-partitioned (each rank returns its rows)."""
        self.ops = ops or _ops
        self.comm = comm or Comm()
        self.a, self.pol, self.mv = a, pol, mv
        self.A_mv = a.device_operator(mv.storage)
        self.At_mv = a.device_operator_t(mv.storage)
        self.A_pol = self.A_mv if pol.storage == mv.storage else a.device_operator(pol.storage)
        self.device = self.A_mv.device
        _, self.proj_out = projection_policy(pol)
        self.a_passes = 0
        self.n1 = int(n1_global if n1_global is not None else a.rows)
        self.r0, self.r1 = self.comm.row_range(self.n1)
        if self.comm.distributed and a.rows != self.r1 - self.r0:
            raise ValueError(f"rank {self.comm.rank}: local A has {a.rows} rows, expected {self.r1 - self.r0}")

    @classmethod
    def single(cls, a, pol, mv):
        return cls(a, pol, mv)

    def basis(self, X, cfg):
        """Hessenberg basis (K3), or a Gram-Schmidt comparator (csrc/gs.cu)."""
        pol = self.pol
        if cfg.basis_method in GRAM_SCHMIDT_METHODS:
            return self.ops.orthonormalize(X, cfg.basis_method.value, pol.storage, pol.compute, pol.accumulate,
                                           pol.drop_tol)
        return self.ops.hessenberg(X, pol.storage, pol.compute, pol.drop_tol)

    def matvec(self, op, X, st):
        """A X (local rows when partitioned) with inf-norm column scaling over all ranks."""
        import torch
        colmax = torch.zeros(X.k, dtype=torch.float64, device=self.device)
        W = self.ops.new_block(op.rows, X.k, self.mv.storage, self.device)
        self.ops.gemm_av(op, X, W, colmax=colmax, flags=st[S_MV_FLAGS:S_MV_FLAGS + 1])
        self.a_passes += 1
        self.comm.all_reduce_max_(colmax)
        self.ops.scale_columns(W, colmax, self.mv.compute)
        return W

    def matvec_t(self, U, st):
        """A^T U with inf-norm column scaling.  Partitioned: the ranks' fp32 partial products
        A_p^T U_p are all-reduced (sum), then rounded to storage and scaled."""
        import torch
        if not self.comm.distributed:
            return self.matvec(self.At_mv, U, st)
        ops, k, n2 = self.ops, U.k, self.At_mv.rows
        acc = FpFormat.F64 if FpFormat.F64 in (self.At_mv.fmt, U.fmt) else FpFormat.F32
        P = ops.new_block(n2, k, acc, self.device)
        ops.gemm_av(self.At_mv, U, P, flags=st[S_MV_FLAGS:S_MV_FLAGS + 1])
        self.a_passes += 1
        self.comm.all_reduce_sum_(P.t)
        W = ops.new_block(n2, k, self.mv.storage, self.device)
        ops.convert(P, W, flags=st[S_MV_FLAGS:S_MV_FLAGS + 1])
        colmax = W.t[:k, :n2].to(torch.float64).abs().amax(dim=1)
        ops.scale_columns(W, colmax, self.mv.compute)
        return W

    def gather_rows(self, Xp):
        """The full n1 x k block from every rank's rows (all-gather)."""
        if not self.comm.distributed:
            return Xp
        X = self.ops.new_block(self.n1, Xp.k, Xp.fmt, self.device)
        self.comm.all_gather_rows(Xp.t, X.t, self.n1, Xp.k)
        return X

    def project(self, U, V, want64: bool = True, x_fmt=None, classical: bool = False):
        """ofrr_svd on device blocks U (n1 x k1), V (n2 x k2) in policy storage; with
        ``classical`` rr_svd (ofrr/projection.py:90-96): identity mass matrices."""
        import torch
        ops = self.ops
        k1, k2 = U.k, V.k
        kk = k1 + k2
        st = torch.zeros(8, dtype=torch.int32, device=self.device)
        W = ops.new_block(self.A_pol.rows, k2, self.pol.storage, self.device)
        ops.gemm_av(self.A_pol, V, W, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1])
        self.a_passes += 1
        dist = self.comm.distributed
        Ul = _row_slice(U, self.r0, self.r1) if dist else U        # this rank's rows of the U basis
        G, Mu = ops.gram(Ul, W, self.proj_out, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1])
        if dist:
            self.comm.all_reduce_sum_(G)
            self.comm.all_reduce_sum_(Mu)
        _, Mv = ops.gram(V, None, self.proj_out, flags=st[S_GRAM_FLAGS:S_GRAM_FLAGS + 1])
        # block pencil (tensors are column-major: row j = column j)
        Bm = torch.zeros((kk, kk), dtype=torch.float64, device=self.device)
        Mm = torch.zeros((kk, kk), dtype=torch.float64, device=self.device)
        Gk = G[:k2, :k1]                 # column j (< k2) of G = U^T W -> row j
        Bm[k1:, :k1].copy_(Gk)           # columns k1.. of B hold G (rows 0..k1)
        Bm[:k1, k1:].copy_(Gk.t())       # columns 0..k1 of B hold G^T (rows k1..)
        if classical:
            Mm.fill_diagonal_(1.0)
        else:
            Mm[:k1, :k1].copy_((Mu + Mu.t()) / 2.0)
            Mm[k1:, k1:].copy_((Mv + Mv.t()) / 2.0)
        eig = ops.sym_def_gen_eig(Bm, Mm, kk)
        st[S_EIG_STATUS:S_EIG_STATUS + 1].copy_(eig.status)
        st[S_NOUT:S_NOUT + 1].copy_(eig.n_out)
        if dist:
            self.comm.all_reduce_max_(st)
        s = st.cpu().numpy()
        if s[S_MV_FLAGS] & 1:
            raise OverflowDiagnostic("non-finite entries after MatVec")
        if s[S_GRAM_FLAGS] & 1:
            raise OverflowDiagnostic("non-finite entries in projected matrix")
        if s[S_EIG_STATUS] == 6:
            raise ConvergenceError("Jacobi eigendecomposition did not converge", float("nan"))
        nout = int(s[S_NOUT])
        if nout == 0:
            raise EmptyPencilError("mass matrix retained no eigenvalues")
        vals = eig.values[:nout].cpu().numpy()
        smax = float(np.max(vals))
        pos = vals > POSITIVE_EIG_TOL * smax if smax > 0 else vals > 0
        npos = int(np.count_nonzero(pos))   # a prefix: values are sorted descending
        sig = vals[:npos]
        diag = ""
        if npos < min(k1, k2):
            diag = f"{npos} positive eigenvalues (pencil admits {min(k1, k2)})"
        if npos == 0:
            return RitzSet(sig, DenseMatrix(np.zeros((Ul.n, 0)), FpFormat.F64), "svd",
                           right_vectors=DenseMatrix(np.zeros((V.n, 0)), FpFormat.F64), diagnostics=diag), None, None
        U64, _ = ops.ritz(Ul, eig.vectors, kk, None, npos, math.sqrt(2.0), want64=True)
        V64, Vx = ops.ritz(V, eig.vectors, kk, None, npos, math.sqrt(2.0), want64=True,
                           x_fmt=x_fmt, row_offset=k1, flags=st[S_RESTART_FLAGS:S_RESTART_FLAGS + 1])
        rs = RitzSet(sig, DenseMatrix.from_block(U64), "svd", right_vectors=DenseMatrix.from_block(V64),
                     diagnostics=diag)
        return rs, Vx, st


    def residuals(self, rs: RitzSet, t: int) -> np.ndarray:
        """FP64 max(||A v - s u||, ||A^T u - s v||) / s of the first t triplets
        (ofrr/projection.py:136-158).  Partitioned: ||A_p v - s u_p||^2 summed over ranks;
        A^T u = sum_p A_p^T u_p (FP64-accurate partial products, all-reduced)."""
        import torch
        from .projection import residual_report
        if not self.comm.distributed and self.ops is _ops:
            from dataclasses import replace as _rep
            head = _rep(rs, values=rs.values[:t], vectors=_narrow_dm(rs.vectors, t),
                        right_vectors=_narrow_dm(rs.right_vectors, t))
            return residual_report(self.a, head).residuals
        ops, dev = self.ops, self.device
        A = self.a.residual_operator(self.A_mv.fmt)
        At = self.a.residual_operator_t(self.A_mv.fmt)
        if At.fmt not in _ops.OZAKI_FMTS and At.fmt != FpFormat.F64 and self.ops is _ops:
            At = self.a.device_operator_t(FpFormat.F64)      # FP64 product of an f32 operator
        Ub = rs.vectors.device_block(FpFormat.F64).narrow(t)
        Vb = rs.right_vectors.device_block(FpFormat.F64).narrow(t)
        sig = torch.as_tensor(np.asarray(rs.values[:t], dtype=np.float64), device=dev)
        ss1 = torch.zeros(t, dtype=torch.float64, device=dev)
        ops.residual_pair(A, False, Vb, Ub, sig, None, t, ss1, accumulate_max=2)
        n2 = At.rows
        P = ops.new_block(n2, t, FpFormat.F64, dev)
        ops.gemm_av(At, Ub, P)
        self.comm.all_reduce_sum_(ss1)
        self.comm.all_reduce_sum_(P.t)
        d = P.t[:t, :n2] - sig[:, None] * Vb.t[:t, :n2]
        ss2 = (d * d).sum(dim=1)
        r = torch.sqrt(torch.maximum(ss1, ss2)) / sig.abs()
        return r.cpu().numpy()


def subspace_iter_svd(a: DenseMatrix, cfg: IterConfig, stats: Optional[RunStats] = None,
                      comm: Optional[Comm] = None, n_global: Optional[int] = None) -> RitzSet:
    """Alternating subspace iteration for the SVD (ofrr/driver.py:141-173), on device
    (thread-safe like subspace_iter_eig).  Row-partitioned when ``comm`` spans several ranks:
    ``a`` holds this rank's rows of A (``n_global`` rows in all) and the returned left
    singular vectors hold this rank's rows."""
    with _SOLVE_LOCK:
        return _subspace_iter_svd(a, cfg, stats, comm, n_global)


def _subspace_iter_svd(a, cfg, stats, comm=None, n_global=None, ops=None) -> RitzSet:
    """The SVD outer loop.  With cfg.tol the loop stops at the first outer iteration whose
    leading ``top`` triplets have FP64 residuals max(||A v - s u||, ||A^T u - s v||) / s below
    tol (``m`` is the cap); otherwise exactly m iterations (the reference).  ladder / reuse_av
    are eigenvalue-path extensions and are rejected here."""
    from .projection import residual_report
    _require_ofrr_path(cfg, "SVD iteration")
    if cfg.ladder is not None or cfg.reuse_av:
        raise ValueError("subspace_iter_svd: ladder / reuse_av apply to subspace_iter_eig only")
    comm = comm or Comm.world()
    n1, n2 = int(n_global if n_global is not None else a.rows), a.cols
    if cfg.k > min(n1, n2):
        raise ValueError("k exceeds min(n1, n2)")
    pol, mv = cfg.policy, cfg.mv_policy
    eng = SvdEngine(a, pol, mv, ops=ops, comm=comm, n1_global=n1)
    ops = eng.ops
    V = ops.start_block(cfg.seed, n2, cfg.k, mv.storage, eng.device)
    rs = None
    tol, top = cfg.tol, (cfg.top or cfg.k)
    hist = []
    converged = False
    import torch
    its = 0
    checked = None
    for it in range(cfg.m):
        st = torch.zeros(8, dtype=torch.int32, device=eng.device)
        U = V
        for _ in range(cfg.iter):
            U = eng.matvec(eng.A_mv, V, st)
            V = eng.matvec_t(U, st)
        hu, hv = eng.basis(eng.gather_rows(U), cfg), eng.basis(V, cfg)
        st[S_NKEPT:S_NKEPT + 1].copy_(hu.n_kept)
        st[S_NKEPT2:S_NKEPT2 + 1].copy_(hv.n_kept)
        if comm.distributed:
            comm.all_reduce_max_(st)
        s = st.cpu().numpy()
        if s[S_MV_FLAGS] & 1:
            raise OverflowDiagnostic("non-finite entries after MatVec")
        k1, k2 = int(s[S_NKEPT]), int(s[S_NKEPT2])
        if k1 == 0 or k2 == 0:
            raise EmptyBasisError("all columns skipped in basis construction")
        rs, Vx, st2 = eng.project(hu.Q.narrow(k1), hv.Q.narrow(k2), x_fmt=mv.storage,
                                  classical=cfg.projection == "rr")
        if Vx is None:
            raise EmptyPencilError("no positive eigenvalues in the SVD pencil")
        if comm.distributed:
            comm.all_reduce_max_(st2)
        if int(st2[S_RESTART_FLAGS].item()) & 1:
            raise OverflowDiagnostic("non-finite entries after projection")
        V = Vx
        its = it + 1
        if tol is not None:
            # FP64 confirmation on the leading triplets (two FP64-accurate products, K7z)
            t = min(top, len(rs.values))
            checked = eng.residuals(rs, t)
            worst = float(np.max(checked)) if t >= top else float("inf")
            hist.append((its, worst))
            if worst < tol:
                converged = True
                break
    if stats is not None:
        stats.iterations = its
        stats.a_passes = eng.a_passes
        stats.history = hist
        stats.converged = converged
        stats.rungs = [(cfg_rung_label(cfg), its, eng.a_passes)]
    if comm.distributed or eng.ops is not _ops:
        from dataclasses import replace as _rep
        return _rep(rs, residuals=eng.residuals(rs, len(rs.values)))
    return residual_report(a, rs)


def _narrow_dm(m: DenseMatrix, t: int) -> DenseMatrix:
    """The first t columns of a device-resident block DenseMatrix."""
    blk = m.device_block(FpFormat.F64)
    return DenseMatrix.from_block(blk.narrow(t))
