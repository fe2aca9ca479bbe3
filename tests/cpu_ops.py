"""TEST-ONLY CPU stand-in for paper_2505_00281_b200.ops, computing every device op with the
oracle (the reference's arithmetic restated in numpy/C).  It exists so the multi-process
(row-partitioned, torch.distributed) orchestration of the driver can be exercised on CPU
with the gloo backend -- the product never imports it (the product has no CPU fallback).

Same function names, argument meaning and data layout as ops.py: blocks are torch tensors
(k, ld) whose row j is column j; operators are (rows, lda) row-major.
"""

from __future__ import annotations

import numpy as np
import torch

import oracle as o
from paper_2505_00281_b200 import ops as dev_ops
from paper_2505_00281_b200.precision import FpFormat

DevBlock, DevOperator, HessOut, EigOut = dev_ops.DevBlock, dev_ops.DevOperator, dev_ops.HessOut, dev_ops.EigOut
new_block, new_operator = dev_ops.new_block, dev_ops.new_operator
CPU = torch.device("cpu")


def _np(b: DevBlock, k=None) -> np.ndarray:
    k = b.k if k is None else k
    return b.t[:k, : b.n].to(torch.float64).numpy().T.copy()      # n x k


def _put(b: DevBlock, x: np.ndarray) -> None:
    b.t[: x.shape[1], : b.n].copy_(torch.from_numpy(np.ascontiguousarray(x.T)).to(b.t.dtype))


def _op_np(A: DevOperator) -> np.ndarray:
    return A.t[:, : A.cols].to(torch.float64).numpy()


def start_block(seed, n, k, fmt, device):
    X = new_block(n, k, fmt, CPU, zero=True)
    _put(X, o.round_to(np.random.default_rng(seed).random((n, k)), int(fmt)))
    return X


def block_from_host(x, fmt, device):
    x = np.asarray(x, dtype=np.float64)
    X = new_block(x.shape[0], x.shape[1], fmt, CPU, zero=True)
    _put(X, o.round_to(x, int(fmt)))
    return X


def gemm_av(A, X, W, out_fmt=None, colmax=None, flags=None, transpose=False, W2=None):
    a = _op_np(A)
    if transpose:
        a = a.T
    x = _np(X)
    of = int(W.fmt if out_fmt is None else out_fmt)
    exact = o.mixed_gemm(a, x, o.F64, o.F64, o.F64)     # row-partition independent
    w = o.round_to(exact, of)
    _put(W, w)
    if W2 is not None:
        _put(W2, o.round_to(exact, int(W2.fmt)))
    if colmax is not None:
        cm = np.max(np.abs(w), axis=0) if w.shape[0] else np.zeros(w.shape[1])
        colmax[: len(cm)] = torch.maximum(colmax[: len(cm)], torch.from_numpy(cm))
    if flags is not None and not np.all(np.isfinite(w)):
        flags |= 1


def convert(src, dst, flags=None):
    _put(dst, o.round_to(_np(src), int(dst.fmt)))


def scale_columns(X, colmax, compute):
    x = _np(X)
    m = colmax.numpy()
    out = x.copy()
    for j in range(x.shape[1]):
        if m[j] != 0.0:
            out[:, j] = o.round_to(o.round_to(x[:, j] / m[j], int(compute)), int(X.fmt))
    _put(X, out)


def hessenberg(X, storage, compute, tol):
    x = o.round_to(_np(X), int(storage))
    pol = o.Pol(int(storage), int(compute), int(compute))
    k = X.k
    Q = new_block(X.n, k, storage, CPU, zero=True)
    piv = torch.zeros(k, dtype=torch.int64)
    kept = torch.zeros(k, dtype=torch.int32)
    try:
        q, p, kp = o.hessenberg_basis(x, pol)
        _put(Q, q)
        piv[: len(p)] = torch.from_numpy(p)
        kept[:] = torch.from_numpy(kp.astype(np.int32))
        nk = q.shape[1]
    except o.EmptyBasisError:
        nk = 0
    return HessOut(Q, piv, kept, torch.tensor([nk], dtype=torch.int32))


def gram(U, W, out_fmt, flags=None, want_m=True):
    u = _np(U)
    G1 = G2 = None
    if W is not None:
        g1 = o.mixed_gemm(u.T, _np(W), o.F64, o.F64, int(out_fmt))
        G1 = torch.from_numpy(np.ascontiguousarray(g1.T))
    if want_m:
        g2 = o.mixed_gemm(u.T, u, o.F64, o.F64, int(out_fmt))
        G2 = torch.from_numpy(np.ascontiguousarray(g2.T))
    return G1, G2


def sym_def_gen_eig(B, M, k):
    b = B.numpy().T
    m = M.numpy().T
    vals = torch.zeros(k, dtype=torch.float64)
    vecs = torch.zeros((k, k), dtype=torch.float64)
    try:
        v, y = o.sym_def_gen_eig((b + b.T) / 2.0, (m + m.T) / 2.0)
        r = len(v)
        vals[:r] = torch.from_numpy(v)
        vecs[:r, :] = torch.from_numpy(np.ascontiguousarray(y.T))
        status = 0 if r else 5
    except o.ConvergenceError:
        r, status = 0, 6
    return EigOut(vals, vecs, torch.tensor([r], dtype=torch.int32), torch.tensor([status], dtype=torch.int32))


def ritz(U, Y, ldy, r_dev, r_max, scale=1.0, want64=True, x_fmt=None, flags=None, row_offset=0):
    r = int(r_dev.item()) if r_dev is not None else r_max
    y = Y.numpy().T[row_offset: row_offset + U.k, :r]       # kp x r
    ut = scale * (_np(U) @ y)
    full = np.zeros((U.n, r_max))
    full[:, :r] = ut
    U64 = X = None
    if want64:
        U64 = new_block(U.n, r_max, FpFormat.F64, CPU, zero=True)
        _put(U64, full)
    if x_fmt is not None:
        X = new_block(U.n, r_max, x_fmt, CPU, zero=True)
        _put(X, o.round_to(full, int(x_fmt)))
    return U64, X


def reuse_power(W, Y, ldy, r_dev, r_max, x_fmt, colmax, flags=None):
    _, X = ritz(W, Y, ldy, r_dev, r_max, want64=False, x_fmt=x_fmt)
    colmax.copy_(torch.maximum(colmax, torch.from_numpy(np.max(np.abs(_np(X)), axis=0))))
    return X


def residual_estimate(U, W, Y, ldy, vals, r_dev, r_max, mode=0):
    r = min(r_max, int(r_dev.item()) if r_dev is not None else r_max)
    y = Y.numpy().T[: U.k, :r]
    lam = vals.numpy()[:r]
    d = _np(W) @ y - (_np(U) @ y) * lam[None, :]
    ss = np.sum(d * d, axis=0)
    out = torch.zeros(max(r_max, 1), dtype=torch.float64)
    out[:r] = torch.from_numpy(ss if mode == 2 else np.sqrt(ss) / np.abs(lam))
    return out


def residual_eig(A, V, vals, r_dev, r_max):
    a = _op_np(A)
    v = _np(V)[:, :r_max]
    lam = vals.numpy()[:r_max]
    d = a @ v - v * lam[None, :]
    return torch.from_numpy(np.linalg.norm(d, axis=0) / np.abs(lam))


def residual_pair(A, transpose, Xv, Yv, vals, r_dev, r_max, res, accumulate_max):
    a = _op_np(A)
    if transpose:
        a = a.T
    lam = vals.numpy()[:r_max]
    d = a @ _np(Xv)[:, :r_max] - _np(Yv)[:, :r_max] * lam[None, :]
    ss = np.sum(d * d, axis=0)
    if accumulate_max == 2:
        res[:r_max] = torch.from_numpy(ss)
    else:
        rr = np.sqrt(ss) / np.abs(lam)
        res[:r_max] = torch.maximum(res[:r_max], torch.from_numpy(rr)) if accumulate_max else torch.from_numpy(rr)
    return res


class RowBlock:
    """Minimal stand-in for a DenseMatrix holding this rank's rows on the CPU."""

    def __init__(self, a_rows: np.ndarray, fmt: FpFormat):
        self.fmt = FpFormat(fmt)
        rows, cols = a_rows.shape
        self.op = new_operator(rows, cols, self.fmt, CPU)
        self.op.t.zero_()
        self.op.t[:, :cols].copy_(torch.from_numpy(a_rows).to(self.op.t.dtype))
        self._dev = {self.fmt: self.op}
        self.rows, self.cols = rows, cols

    def device_operator(self, fmt=None, device=None):
        return self.op

    def exact_in(self, fmt):
        return True

    def residual_operator(self, prefer):
        return self.op

    def device_operator_t(self, fmt=None, device=None):
        if not hasattr(self, "op_t"):
            self.op_t = new_operator(self.cols, self.rows, self.fmt, CPU)
            self.op_t.t.zero_()
            self.op_t.t[:, : self.rows].copy_(self.op.t[:, : self.cols].t())
        return self.op_t

    def residual_operator_t(self, prefer):
        return self.device_operator_t()
