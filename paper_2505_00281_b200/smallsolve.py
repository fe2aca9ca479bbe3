"""FP64 small dense eigen-solves on the device (K5).

Same names and contracts as ofrr/smallsolve.py:34-88: ``sym_eig`` (symmetrise, Jacobi,
descending order, largest-|entry|-positive signs) and ``sym_def_gen_eig`` (whitening of
M with the mu > k*eps*mu_max independence safeguard).  Inputs may be host numpy arrays
(copied to the device) or CUDA tensors; results are returned as host numpy arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConvergenceError, EmptyPencilError

MAX_SWEEPS = 30


@dataclass(frozen=True)
class EigResult:
    values: np.ndarray   # FP64, descending
    vectors: np.ndarray  # FP64, one column per value


def _dev(a):
    import torch
    if isinstance(a, torch.Tensor):
        t = a.to(torch.float64)
        if not t.is_cuda:
            t = t.cuda()
        return t.t().contiguous()   # column-major (row j = column j)
    a = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda()


def sym_eig(s) -> EigResult:
    """ofrr/smallsolve.py:34-49."""
    from . import ops
    k = int(np.shape(s)[0])
    if k == 0:
        return EigResult(np.zeros(0), np.zeros((0, 0)))
    out = ops.sym_eig(_dev(s), k)
    st = int(out.status.item())
    if st != 0:
        raise ConvergenceError("Jacobi eigendecomposition did not converge", float("nan"))
    vals = out.values[:k].cpu().numpy()
    vecs = out.vectors[:k, :k].cpu().numpy().T.copy()
    return EigResult(vals, vecs)


def sym_def_gen_eig(b, m) -> EigResult:
    """ofrr/smallsolve.py:64-88 (B is symmetrised on the device as ofrr_eig does)."""
    from . import ops
    k = int(np.shape(m)[0])
    if k == 0:
        return EigResult(np.zeros(0), np.zeros((0, 0)))
    out = ops.sym_def_gen_eig(_dev(b), _dev(m), k)
    st = int(out.status.item())
    if st == 6:  # OFRR_ERR_CONVERGENCE
        raise ConvergenceError("Jacobi eigendecomposition did not converge", float("nan"))
    if st == 5:  # nothing retained: the reference returns an empty result
        return EigResult(np.zeros(0), np.zeros((k, 0)))
    r = int(out.n_out.item())
    vals = out.values[:r].cpu().numpy()
    vecs = out.vectors[:r, :k].cpu().numpy().T.copy()
    return EigResult(vals, vecs)


__all__ = ["EigResult", "sym_eig", "sym_def_gen_eig", "ConvergenceError", "EmptyPencilError", "MAX_SWEEPS"]
