"""Dense operator container and synthetic inputs.

``DenseMatrix`` keeps the reference's contract (ofrr/matrix.py:25-47): a 2-D matrix
with a storage-format tag, ``.data`` as column-major float64, ``rows/cols/shape``,
``from_array``.  It additionally holds the matrix on the device: the first device use
uploads it once (row-major, in the requested storage format, HBM resident) and later
calls reuse that copy.  A ``DenseMatrix`` can also be built directly from a device
tensor (``DenseMatrix.on_device``), in which case ``.data`` is materialised lazily.

Synthetic symmetric matrices with a prescribed spectrum are built as
A = Q B Q^T with B = S C S (C[i, j] = c[i xor j], the Walsh-Hadamard diagonalisation of
diag(lambda); n a power of two) or B = diag(lambda) (otherwise), and Q a product of r
seeded Householder reflectors in compact-WY form.  That gives
A = B + Wf Mf^T + Mf Wf^T with n x r factors, so any row block of A is evaluated on the
device from O(n r) host data (K8) -- no n x n host work.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .precision import FpFormat, round_to


class DenseMatrix:
    """2-D matrix with a storage-format tag (ofrr/matrix.py:25-47) plus a device copy."""

    def __init__(self, data, fmt: FpFormat, uplo: Optional[str] = None):
        """``uplo`` ("U"/"L", extension): A is symmetric and only that triangle of a host
        torch tensor in the storage dtype is read -- it is the only part copied to the device
        (ops.upload_symmetric; the dsyev(uplo) convention).  None: the whole array is read."""
        if uplo not in (None, "U", "L"):
            raise ValueError("uplo must be None, 'U' or 'L'")
        self.uplo = uplo
        self.fmt = FpFormat(fmt)
        self._host = None
        self._dev = {}          # FpFormat -> ops.DevOperator (row-major operator copies)
        self._blocks = {}       # FpFormat -> ops.DevBlock (column-major block copies)
        self._exact = {}        # FpFormat -> operator copy holds the data exactly
        self._dev_t = {}        # FpFormat -> ops.DevOperator of A^T (SVD)
        self._exact_t = {}
        self._src_tensor = None  # host/device torch tensor given by the caller
        try:
            import torch
            is_t = isinstance(data, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_t = False
        if is_t:
            if data.dim() != 2:
                raise ValueError("DenseMatrix expects a 2-D array")
            self._src_tensor = data
            self._shape = tuple(int(s) for s in data.shape)
        else:
            self._host = np.asfortranarray(data, dtype=np.float64)
            if self._host.ndim != 2:
                raise ValueError("DenseMatrix expects a 2-D array")
            self._shape = self._host.shape

    # -- reference API ------------------------------------------------------------
    @classmethod
    def from_array(cls, arr, fmt: FpFormat) -> "DenseMatrix":
        return cls(round_to(np.asarray(arr, dtype=np.float64), fmt), fmt)

    @property
    def data(self) -> np.ndarray:
        """Column-major float64 host array (materialised from the device if needed)."""
        if self._host is None:
            import torch
            if self.uplo is not None and self._src_tensor is not None and not self._dev:
                self.device_operator()          # the declared triangle, mirrored on the device
            if self._src_tensor is not None and self.uplo is None:
                self._host = np.asfortranarray(self._src_tensor.to(torch.float64).cpu().numpy())
            elif self._blocks:
                blk = max(self._blocks.values(), key=lambda b: b.fmt.itemsize)
                self._host = blk.to_numpy_f64()
            else:
                op = max(self._dev.values(), key=lambda o: o.fmt.itemsize)
                t = op.t[:, : op.cols]
                self._host = np.asfortranarray(t.to(torch.float64).cpu().numpy())
        return self._host

    @property
    def rows(self) -> int:
        return self._shape[0]

    @property
    def cols(self) -> int:
        return self._shape[1]

    @property
    def shape(self):
        return self._shape

    def __repr__(self):
        where = "device" if (self._dev or self._blocks) else "host"
        return f"DenseMatrix({self.rows}x{self.cols}, fmt={self.fmt.name}, {where})"

    # -- device side ----------------------------------------------------------------
    @classmethod
    def on_device(cls, op) -> "DenseMatrix":
        """Wrap an existing ops.DevOperator (row-major, HBM resident)."""
        m = cls.__new__(cls)
        m.uplo = None
        m.fmt = FpFormat(op.fmt)
        m._host = None
        m._src_tensor = None
        m._dev = {m.fmt: op}
        m._blocks = {}
        m._exact = {m.fmt: True}
        m._dev_t = {}
        m._exact_t = {}
        m._shape = (op.rows, op.cols)
        return m

    def device_operator(self, fmt: Optional[FpFormat] = None, device=None):
        """The matrix as a row-major device operator in ``fmt`` (uploaded once).

        The reference keeps A in float64 and rounds every product instead
        (ofrr/matrix.py:253-254); the tensor cores need A in the
        storage format, so A is rounded once on upload (identical whenever A's values are
        representable in that format, which is how the parity tests set A up).  Whether
        the rounding was exact is recorded (``exact_in``) so that FP64 residuals are taken
        against A as the caller stored it (ofrr/projection.py:136-147)."""
        import torch
        from . import ops, _lib
        fmt = self.fmt if fmt is None else FpFormat(fmt)
        if fmt in self._dev:
            return self._dev[fmt]
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        op = ops.new_operator(self.rows, self.cols, fmt, device)
        L = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        flags = torch.zeros(1, dtype=torch.int32, device=device)
        if self._dev:
            # convert from an existing device copy (the widest one)
            src = max(self._dev.values(), key=lambda o: o.fmt.itemsize)
            _lib.check(L.ofrr_convert(src.ptr, int(src.fmt), src.lda, op.ptr, int(fmt), op.lda, self.cols,
                                      self.rows, flags.data_ptr(), st), "convert operator")
            exact = self._exact.get(src.fmt, False) and fmt >= src.fmt
        elif self.uplo is not None and self._src_tensor is not None and self._src_tensor.device.type == "cpu" \
                and self._src_tensor.dtype == fmt.torch_dtype and self._src_tensor.stride(1) == 1 \
                and self.rows == self.cols:
            ops.upload_symmetric(op, self._src_tensor, self.uplo)   # one triangle over PCIe
            exact = True
        elif self._src_tensor is not None and self._src_tensor.dtype == fmt.torch_dtype \
                and self._src_tensor.stride(1) == 1:
            op.t[:, : self.cols].copy_(self._src_tensor, non_blocking=True)   # plain H2D / D2D copy
            exact = True
        else:
            if self._src_tensor is not None:
                d64 = self._src_tensor.to(device=device, dtype=torch.float64).t().contiguous()
            else:
                # host F-order float64: upload as is, transpose + round on the device
                d64 = torch.from_numpy(self._host.T).to(device)
            _lib.check(L.ofrr_transpose_convert(d64.data_ptr(), int(FpFormat.F64), self.rows, op.ptr, int(fmt),
                                                op.lda, self.rows, self.cols, flags.data_ptr(), st),
                       "upload operator")
            exact = None
        fl = int(flags.item())
        if exact is None:
            exact = not (fl & _lib.FLAG_INEXACT)
        self._exact[fmt] = bool(exact)
        self._dev[fmt] = op
        return op

    def device_operator_t(self, fmt: Optional[FpFormat] = None, device=None):
        """A^T as a row-major device operator (cols x rows) in ``fmt`` -- the second
        operand layout of the SVD's A^T U products (ofrr/matrix.py:253), kept resident
        so both A V and A^T U stream K-major tiles through the tensor-core kernel."""
        import torch
        from . import ops, _lib
        fmt = self.fmt if fmt is None else FpFormat(fmt)
        if fmt in self._dev_t:
            return self._dev_t[fmt]
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        op = ops.new_operator(self.cols, self.rows, fmt, device)
        L = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        flags = torch.zeros(1, dtype=torch.int32, device=device)
        if self._host is not None and not self._dev:
            d64 = torch.from_numpy(self._host.T).to(device)          # row-major A^T, fp64
            _lib.check(L.ofrr_convert(d64.data_ptr(), int(FpFormat.F64), self.rows, op.ptr, int(fmt), op.lda,
                                      self.rows, self.cols, flags.data_ptr(), st), "upload operator^T")
            exact = None
        else:
            src = self.device_operator(max(self._dev, key=lambda f: f.itemsize) if self._dev else fmt)
            # row-major A (rows x lda) is column-major A^T (cols x rows, ld = lda)
            _lib.check(L.ofrr_transpose_convert(src.ptr, int(src.fmt), src.lda, op.ptr, int(fmt), op.lda,
                                                self.cols, self.rows, flags.data_ptr(), st), "transpose operator")
            exact = None if src.fmt == FpFormat.F64 else (self._exact.get(src.fmt, False) and fmt >= src.fmt)
        fl = int(flags.item())
        if exact is None:
            exact = not (fl & (_lib.FLAG_INEXACT | 0))
        self._exact_t[fmt] = bool(exact)
        self._dev_t[fmt] = op
        return op

    def residual_operator_t(self, prefer: FpFormat):
        op = self.device_operator_t(prefer)
        if self._exact_t.get(FpFormat(prefer), False):
            return op
        return self.device_operator_t(FpFormat.F64)

    def exact_in(self, fmt: FpFormat) -> bool:
        """True if the device copy in ``fmt`` holds A exactly (no rounding on upload)."""
        return self._exact.get(FpFormat(fmt), False)

    def residual_operator(self, prefer: FpFormat):
        """Device operator for FP64 residuals: ``prefer`` if it holds A exactly, else F64."""
        op = self.device_operator(prefer)
        if self.exact_in(prefer):
            return op
        return self.device_operator(FpFormat.F64)

    # -- column-major blocks (X, U, Q, Ritz vectors) ---------------------------------
    @classmethod
    def from_block(cls, blk) -> "DenseMatrix":
        """Wrap an ops.DevBlock (column-major n x k on the device)."""
        m = cls.__new__(cls)
        m.uplo = None
        m.fmt = FpFormat(blk.fmt)
        m._host = None
        m._src_tensor = None
        m._dev = {}
        m._exact = {}
        m._dev_t = {}
        m._exact_t = {}
        m._blocks = {m.fmt: blk}
        m._shape = (blk.n, blk.k)
        return m

    def device_block(self, fmt: Optional[FpFormat] = None, device=None):
        """The matrix as a column-major device block in ``fmt``."""
        import torch
        from . import ops
        fmt = self.fmt if fmt is None else FpFormat(fmt)
        if fmt in self._blocks:
            return self._blocks[fmt]
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        if self._blocks:
            src = max(self._blocks.values(), key=lambda b: b.fmt.itemsize)
            out = ops.new_block(src.n, src.k, fmt, device, zero=True)
            ops.convert(src, out)
        else:
            out = ops.block_from_host(self.data, fmt, device)
        self._blocks[fmt] = out
        return out

    def release_device(self) -> None:
        self._dev.clear()
        self._blocks.clear()
        self._dev_t.clear()


def to_dense_f64(a) -> np.ndarray:
    """FP64 dense promotion (ofrr/matrix.py:257-261)."""
    return np.array(a.data, dtype=np.float64)


# ------------------------------------------------------------------------------------
# synthetic inputs
# ------------------------------------------------------------------------------------
def _fwht(x: np.ndarray) -> np.ndarray:
    """Unnormalised fast Walsh-Hadamard transform along axis 0 (Sylvester order)."""
    x = np.array(x, dtype=np.float64, copy=True)
    n = x.shape[0]
    h = 1
    while h < n:
        x = x.reshape((n // (2 * h), 2, h) + x.shape[1:])
        a = x[:, 0].copy()
        b = x[:, 1].copy()
        x[:, 0] = a + b
        x[:, 1] = a - b
        x = x.reshape((n,) + x.shape[3:])
        h *= 2
    return x


@dataclass
class SymFactors:
    """Host factors of A = base + Wf Mf^T + Mf Wf^T (see module docstring)."""
    n: int
    hadamard: bool
    c: np.ndarray        # n: c[i ^ j] (hadamard) or diag (otherwise)
    s: np.ndarray        # n: +-1 signs (hadamard), ones otherwise
    Wf: np.ndarray       # n x r
    Mf: np.ndarray       # n x r
    eigenvalues: np.ndarray  # exact spectrum (descending)


def geometric_spectrum(n: int, top: int, k: int, rho: Optional[float] = None) -> np.ndarray:
    """lambda_i = rho^i with rho = 0.1^(1/(k-top+1))."""
    if rho is None:
        rho = 0.1 ** (1.0 / (k - top + 1))
    return rho ** np.arange(n, dtype=np.float64)


def clustered_spectrum(n: int, clusters: int = 6, per: int = 8, spread: float = 1e-3,
                       tail_rho: float = 0.9, seed: int = 20240901) -> np.ndarray:
    """C5: `clusters` groups of `per` eigenvalues with relative intra-spread `spread`,
    then a geometric tail."""
    rng = np.random.default_rng(seed)
    vals = []
    for c in range(clusters):
        centre = 0.75 ** c
        vals.extend(centre * (1.0 + spread * rng.uniform(-1, 1, per)))
    rest = n - len(vals)
    tail_start = 0.75 ** clusters * 0.8
    vals.extend(tail_start * tail_rho ** np.arange(rest))
    return np.sort(np.asarray(vals[:n], dtype=np.float64))[::-1].copy()


def sym_factors(lam: np.ndarray, seed: int = 20240901, r: int = 16) -> SymFactors:
    """Factors of A = Q B Q^T for the spectrum ``lam`` (length n)."""
    lam = np.asarray(lam, dtype=np.float64)
    n = lam.shape[0]
    rng = np.random.default_rng(seed)
    hadamard = n >= 2 and (n & (n - 1)) == 0
    if hadamard:
        perm = rng.permutation(n)
        lam_p = lam[perm]                      # eigenvalue of Walsh function perm^-1
        c = _fwht(lam_p) / n                   # C = H diag(lam_p) H / n, C[i,j] = c[i^j]
        s = rng.choice([-1.0, 1.0], size=n)
    else:
        perm = rng.permutation(n)
        c = lam[perm].copy()
        s = np.ones(n)

    def apply_b(y: np.ndarray) -> np.ndarray:
        if hadamard:
            return s[:, None] * (_fwht(lam_p[:, None] * _fwht(s[:, None] * y)) / n)
        return c[:, None] * y

    r = int(min(r, n))
    V = rng.standard_normal((n, r))
    W = np.zeros((n, 0))
    Y = np.zeros((n, 0))
    for i in range(r):
        v = V[:, i]
        tau = 2.0 / float(v @ v)
        w = tau * (v - W @ (Y.T @ v))
        W = np.column_stack([W, w])
        Y = np.column_stack([Y, v])
    Z = apply_b(Y)
    G = Y.T @ Z
    G = (G + G.T) / 2.0
    M = -Z + 0.5 * (W @ G)
    return SymFactors(n, hadamard, np.ascontiguousarray(c), np.ascontiguousarray(s),
                      np.asfortranarray(W), np.asfortranarray(M), np.sort(lam)[::-1].copy())


def synthetic_symmetric(lam: np.ndarray, fmt: FpFormat, seed: int = 20240901, r: int = 16,
                        device=None, row0: int = 0, rows: Optional[int] = None):
    """Build (rows of) the synthetic symmetric matrix on the device (K8).

    Returns (DenseMatrix on device, SymFactors).  ``row0``/``rows`` select a row block
    (row-partitioned multi-GPU runs: each rank builds only its own rows)."""
    import torch
    from . import ops
    f = sym_factors(lam, seed=seed, r=r)
    n = f.n
    rows = n - row0 if rows is None else rows
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    op = ops.new_operator(rows, n, fmt, device)
    ops.generate_sym(op, row0, f.hadamard, f.c, f.s, f.Wf, f.Mf)
    return DenseMatrix.on_device(op), f


def synthetic_lowrank(n1: int, n2: int, fmt: FpFormat, r: int = 256, rho: float = 0.9, nu_rel: float = 1e-4,
                      seed: int = 20240901, device=None, row0: int = 0, rows: Optional[int] = None):
    """C4: A = G1 diag(sigma) G2^T + nu N, G1 (n1 x r) and G2 (n2 x r) with
    orthonormal seeded Gaussian columns, sigma_i = rho^i, nu = nu_rel * sigma_1, N i.i.d.
    N(0,1)/sqrt(n2); built on the device in fp32 (torch, input generation only -- outside any
    timed region) and rounded once to ``fmt``.  ``row0``/``rows``: this rank's row block
    (G1 is generated in full from the seed, so row blocks agree across ranks).

    Returns (DenseMatrix on device, sigma)."""
    import torch
    from . import ops
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    rows = n1 - row0 if rows is None else rows
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    g1, _ = torch.linalg.qr(torch.randn(n1, r, generator=g, device=device, dtype=torch.float32))
    g2, _ = torch.linalg.qr(torch.randn(n2, r, generator=g, device=device, dtype=torch.float32))
    sigma = rho ** np.arange(r, dtype=np.float64)
    sig_t = torch.tensor(sigma, dtype=torch.float32, device=device)
    op = ops.new_operator(rows, n2, fmt, device)
    nu = nu_rel * float(sigma[0])
    # rows of A in globally aligned slabs of 4096 rows (bounded fp32 temporaries); the noise
    # of a slab comes from a stream keyed by its global index, so any row partition agrees
    SL = 4096
    for gs in range((row0 // SL) * SL, row0 + rows, SL):
        ge = min(n1, gs + SL)
        lo, hi = max(gs, row0), min(ge, row0 + rows)
        if lo >= hi:
            continue
        gn = torch.Generator(device=device)
        gn.manual_seed(seed * 1_000_003 + gs // SL)
        noise = torch.randn(ge - gs, n2, generator=gn, device=device, dtype=torch.float32)
        blk = (g1[lo:hi] * sig_t) @ g2.T
        blk += (nu / np.sqrt(n2)) * noise[lo - gs: hi - gs]
        op.t[lo - row0: hi - row0, :n2].copy_(blk.to(FpFormat(fmt).torch_dtype))
        del blk, noise
    del g1, g2
    return DenseMatrix.on_device(op), sigma
