"""Typed device operations: thin wrappers that pass torch CUDA tensors to the C ABI.

Layout on the device:
* ``DevOperator``: the operator A, row-major ``rows x cols`` in its storage format,
  leading dimension padded to 64 elements (TMA needs 16-byte strides).
* ``DevBlock``: an ``n x k`` block (X, W, U, Q, Ritz vectors) column-major, i.e. the
  reference's Fortran order (ofrr/matrix.py:25-31), stored as a torch tensor of shape
  ``(k, ld)`` whose row j is column j; ``ld`` = n padded to 64.

Every function enqueues on the current torch stream and returns without
synchronising.  Nothing here computes on the host.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from .precision import FpFormat

PAD = 64

# launch accounting (bench.py "gpu_launches"): number of libofrr_b200 kernels enqueued
LAUNCHES = [0]
# optional log of the tensor-core block products (bench.py roofline): when a list is
# installed here, gemm_av appends (algorithmic bytes, flops) of every k_gemm_av_tc launch;
# the kernel-only durations come from the library (ofrr_prof_gemm_read), in launch order
GEMM_LOG = None


import threading

_TLS = threading.local()          # .recorder: the Recorder of the graph this thread is capturing
_ACCT = threading.Lock()          # LAUNCHES / GEMM_LOG updates from concurrent callers


def _recorder():
    return getattr(_TLS, "recorder", None)


class Recorder:
    """Launch / GEMM-log accounting of a captured CUDA graph, re-applied on every replay."""

    def __init__(self):
        self.launches = 0
        self.gemm = []

    def __enter__(self):
        self._prev = _recorder()
        _TLS.recorder = self
        return self

    def __exit__(self, *exc):
        _TLS.recorder = self._prev
        return False

    def replayed(self) -> None:
        with _ACCT:
            LAUNCHES[0] += self.launches
            if GEMM_LOG is not None:
                GEMM_LOG.extend(self.gemm)


def _count(n: int) -> None:
    with _ACCT:
        LAUNCHES[0] += n
    rec = _recorder()
    if rec is not None:
        rec.launches += n


def _log_gemm(entry) -> None:
    with _ACCT:
        if GEMM_LOG is not None:
            GEMM_LOG.append(entry)
    rec = _recorder()
    if rec is not None:
        rec.gemm.append(entry)


def pad_ld(n: int) -> int:
    return max(PAD, (int(n) + PAD - 1) // PAD * PAD)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


@dataclass
class DevBlock:
    """Column-major n x k block in format ``fmt`` (tensor shape (k_alloc, ld))."""
    t: torch.Tensor
    n: int
    k: int
    fmt: FpFormat

    @property
    def ld(self) -> int:
        return self.t.stride(0)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def device(self):
        return self.t.device

    def col_view(self, k: Optional[int] = None) -> torch.Tensor:
        """(k, n) view: row j = column j."""
        k = self.k if k is None else k
        return self.t[:k, : self.n]

    def to_numpy_f64(self, k: Optional[int] = None):
        """Host copy as an F-order float64 n x k array (the reference's layout).  The copy
        lands in pinned memory from torch's caching host allocator (fast DMA, no page faults
        on fresh pages; the block returns to the cache when the caller drops the array)."""
        import numpy as np
        v = self.col_view(k)
        if v.is_cuda:
            h = torch.empty(v.shape, dtype=torch.float64, pin_memory=True)
            h.copy_(v)                                    # (k, n) C-order == (n, k) F-order
            return h.numpy().T
        return np.asfortranarray(v.to(torch.float64).numpy().T)

    def narrow(self, k: int) -> "DevBlock":
        return DevBlock(self.t, self.n, int(k), self.fmt)


@dataclass
class DevOperator:
    """Row-major rows x cols operator in format ``fmt`` (tensor shape (rows, lda))."""
    t: torch.Tensor
    rows: int
    cols: int
    fmt: FpFormat

    @property
    def lda(self) -> int:
        return self.t.stride(0)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def device(self):
        return self.t.device


def new_block(n: int, k: int, fmt: FpFormat, device, zero: bool = False) -> DevBlock:
    fmt = FpFormat(fmt)
    shape = (max(int(k), 1), pad_ld(n))
    t = (torch.zeros if zero else torch.empty)(shape, dtype=fmt.torch_dtype, device=device)
    return DevBlock(t, int(n), int(k), fmt)


def new_operator(rows: int, cols: int, fmt: FpFormat, device) -> DevOperator:
    fmt = FpFormat(fmt)
    t = torch.empty((int(rows), pad_ld(cols)), dtype=fmt.torch_dtype, device=device)
    return DevOperator(t, int(rows), int(cols), fmt)


def upload_symmetric(op: DevOperator, a_host: torch.Tensor, uplo: str = "U", block_rows: int = 2048) -> int:
    """Fill the square device operator ``op`` from a host row-major tensor already in
    ``op.fmt``'s dtype, reading only the ``uplo`` triangle of ``a_host`` (dsyev convention;
    the eigen path, ofrr/driver.py:84-111, is defined for symmetric A): about half of A
    crosses PCIe, the other triangle is mirrored on the device as the blocks land
    (csrc/upload.cu).  Returns the host bytes copied; queued on the current stream."""
    if uplo not in ("U", "L"):
        raise ValueError("uplo must be 'U' or 'L'")
    if op.rows != op.cols or tuple(a_host.shape) != (op.rows, op.cols):
        raise ValueError("upload_symmetric needs a square host array of the operator's shape")
    if a_host.device.type != "cpu" or a_host.dtype != op.fmt.torch_dtype or a_host.stride(1) != 1:
        raise ValueError("upload_symmetric needs a row-major host tensor in the operator's storage dtype")
    L = _lib.load()
    nbytes = ctypes.c_longlong(0)
    _lib.check(L.ofrr_upload_sym(a_host.data_ptr(), a_host.stride(0), op.ptr, op.lda, op.rows, int(op.fmt),
                                 0 if uplo == "U" else 1, int(block_rows), ctypes.addressof(nbytes),
                                 torch.cuda.current_stream(op.device).cuda_stream), "upload symmetric operator")
    return int(nbytes.value)


def block_from_host(x, fmt: FpFormat, device) -> DevBlock:
    """Upload a host n x k float64 array (values representable in ``fmt``)."""
    import numpy as np
    x = np.asarray(x, dtype=np.float64)
    n, k = x.shape
    b = new_block(n, k, FpFormat.F64, device, zero=True)
    b.t[:k, :n].copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
    if FpFormat(fmt) == FpFormat.F64:
        return b
    out = new_block(n, k, fmt, device, zero=True)
    convert(b, out)
    return out


_PCG_STATE = {}


def _pcg64_state(seed: int):
    """numpy's PCG64 (state, increment) for default_rng(seed) (SeedSequence hashing on the
    host; memoised, it is a pure function of the seed)."""
    st = _PCG_STATE.get(seed)
    if st is None:
        import numpy as np
        raw = np.random.default_rng(seed).bit_generator.state["state"]
        st = (int(raw["state"]), int(raw["inc"]))
        if len(_PCG_STATE) < 64:
            _PCG_STATE[seed] = st
    return st


def _zeros_pack(dev, *specs):
    """Zeroed tensors of the given (shape, dtype) as views of ONE allocation (one fill kernel
    instead of one per tensor -- inside a captured iteration each fill is a graph node)."""
    sizes, off, total = [], [], 0
    for shape, dt in specs:
        nb = math.prod(shape) * torch.empty((), dtype=dt).element_size()
        off.append(total)
        sizes.append(nb)
        total += (nb + 255) // 256 * 256
    buf = torch.zeros(max(total, 256), dtype=torch.uint8, device=dev)
    return [buf[o:o + nb].view(dt).view(shape) for o, nb, (shape, dt) in zip(off, sizes, specs)]


def start_block(seed: int, n: int, k: int, fmt: FpFormat, device, out: Optional[DevBlock] = None) -> DevBlock:
    """X0 = numpy default_rng(seed).random((n, k)) rounded to fmt, generated on the device
    bit for bit (ofrr/driver.py:97-99): numpy derives the PCG64 state from the seed, the
    device walks the stream.  ``out``: an n x k block of format fmt to write (its padding is
    left as it is)."""
    s, inc = _pcg64_state(seed)
    m64 = (1 << 64) - 1
    if out is not None:
        if (out.n, out.k, FpFormat(out.fmt)) != (n, k, FpFormat(fmt)):
            raise ValueError("start_block: output block shape/format mismatch")
        X = out
    else:
        X = new_block(n, k, fmt, device, zero=True)
    L = _lib.load()
    _lib.check(L.ofrr_start_block_pcg64(s >> 64, s & m64, inc >> 64, inc & m64, n, k, X.ptr, X.ld, int(fmt),
                                        _stream()), "start_block")
    _count(1)
    return X


def convert(src: DevBlock, dst: DevBlock, flags: Optional[torch.Tensor] = None) -> None:
    """dst <- round(src) column by column (ofrr/precision.py:90-104)."""
    L = _lib.load()
    _lib.check(L.ofrr_convert(src.ptr, int(src.fmt), src.ld, dst.ptr, int(dst.fmt), dst.ld, src.n, src.k,
                              _p(flags), _stream()), "convert")
    _count(1)


def round_tensor(x: torch.Tensor, fmt: FpFormat) -> torch.Tensor:
    """Device round_to for a 1-D/2-D CUDA tensor: returns float64 with values in fmt."""
    x64 = x.to(torch.float64).contiguous()
    flat = x64.reshape(1, -1) if x64.dim() <= 1 else x64.reshape(-1, x64.shape[-1])
    rows, cols = flat.shape
    out = torch.empty_like(flat)
    tmp = torch.empty((rows, cols), dtype=FpFormat(fmt).torch_dtype, device=x.device)
    L = _lib.load()
    # treat each row of `flat` as a column (n = cols, k = rows)
    _lib.check(L.ofrr_convert(flat.data_ptr(), int(FpFormat.F64), cols, tmp.data_ptr(), int(fmt), cols, cols, rows,
                              None, _stream()), "round_to")
    _lib.check(L.ofrr_convert(tmp.data_ptr(), int(fmt), cols, out.data_ptr(), int(FpFormat.F64), cols, cols, rows,
                              None, _stream()), "round_to")
    return out.reshape(x.shape)


# ---------------------------------------------------------------------------------
# K1 / K2
# ---------------------------------------------------------------------------------
# ---------------------------------------------------------------------------------
# K7z: FP64-accurate products with a 16/8-bit operator (int8 tensor cores, Ozaki digits)
# ---------------------------------------------------------------------------------
OZAKI_FMTS = (FpFormat.BF16, FpFormat.F16, FpFormat.FP8_E4M3)
_OZ_BUFFERS = {}   # operator workspace per (A pointer, shape, format): stable addresses


class OzakiOperator:
    """The digit planes of a 16/8-bit operator (ofrr_ozaki_prepare), reusable for every
    FP64-accurate product with it until A changes; ``refresh`` re-slices A in place."""

    def __init__(self, A: DevOperator, prepare: bool = True):
        if A.fmt not in OZAKI_FMTS:
            raise ValueError(f"Ozaki products need a 16/8-bit operator, got {A.fmt.name}")
        L = _lib.load()
        self.A = A
        key = (A.ptr, A.rows, A.cols, A.lda, int(A.fmt), str(A.device))
        nb = L.ofrr_ozaki_operator_workspace(A.rows, A.cols)
        ws = _OZ_BUFFERS.get(key)
        if ws is None or ws.numel() < nb:
            ws = _ws(nb, A.device)
            if len(_OZ_BUFFERS) >= 2:
                _OZ_BUFFERS.pop(next(iter(_OZ_BUFFERS)))
            _OZ_BUFFERS[key] = ws
        self.ws = ws
        if prepare:
            self.refresh()

    def info(self):
        """(full, tails): whether products use all six digit planes of A (else the 3-digit
        heads plus the exact fp64 tails), and the number of listed tail entries (synchronous;
        diagnostics and tests)."""
        import ctypes
        L = _lib.load()
        full, tails = ctypes.c_int(0), ctypes.c_longlong(0)
        _lib.check(L.ofrr_ozaki_operator_info(self.ws.data_ptr(), self.A.rows, ctypes.byref(full), ctypes.byref(tails)),
                   "ozaki_operator_info")
        return bool(full.value), int(tails.value)

    def refresh(self) -> None:
        L = _lib.load()
        A = self.A
        _lib.check(L.ofrr_ozaki_prepare(A.ptr, A.rows, A.cols, A.lda, int(A.fmt), self.ws.data_ptr(), self.ws.numel(),
                                        _stream()), "ozaki_prepare")
        _count(1)


def ozaki_gemm(oz: OzakiOperator, X: DevBlock, W: DevBlock, colmax=None, flags=None, W2: Optional[DevBlock] = None,
               levels: int = 6):
    """W = A X for an fp64 block X, FP64-accurate (rounded to W.fmt); ``levels`` = 4: the
    ~2^-30 lite product (ofrr_ozaki_gemm_levels)."""
    L = _lib.load()
    A = oz.A
    if X.fmt != FpFormat.F64:
        raise ValueError("ozaki_gemm: the block must be fp64")
    ws = _ws(L.ofrr_ozaki_workspace(A.rows, A.cols, X.k), A.device)
    _lib.check(L.ofrr_ozaki_gemm_levels(A.ptr, A.rows, A.cols, A.lda, int(A.fmt), oz.ws.data_ptr(), X.ptr, X.ld, X.k,
                                        W.ptr, W.ld, int(W.fmt),
                                        _p(colmax), _p(flags), W2.ptr if W2 is not None else None,
                                        W2.ld if W2 is not None else 0, int(W2.fmt) if W2 is not None else int(W.fmt),
                                        int(levels), ws.data_ptr(), ws.numel(), _stream()), "ozaki_gemm")
    bn = 64 if levels >= 5 else 128
    _count(2 + (X.k + bn - 1) // bn * 4)   # digits of X, X row-major; per column pass: 2 product variants, tails, fixup


def ozaki_residual(oz: OzakiOperator, Xv: DevBlock, Yv: DevBlock, vals: torch.Tensor,
                   r_dev: Optional[torch.Tensor], r_max: int, res: torch.Tensor, accumulate_max: int = 0):
    L = _lib.load()
    A = oz.A
    ws = _ws(L.ofrr_ozaki_workspace(A.rows, A.cols, r_max), A.device)
    _lib.check(L.ofrr_ozaki_residual(A.ptr, A.rows, A.cols, A.lda, int(A.fmt), oz.ws.data_ptr(), Xv.ptr, Xv.ld, Yv.ptr,
                                     Yv.ld, vals.data_ptr(),
                                     _p(r_dev), r_max, res.data_ptr(), int(accumulate_max), ws.data_ptr(), ws.numel(),
                                     _stream()), "ozaki_residual")
    _count(3 + (r_max + 63) // 64 * 4)
    return res


def gemm_av(A: DevOperator, X: DevBlock, W: DevBlock, out_fmt: Optional[FpFormat] = None,
            colmax: Optional[torch.Tensor] = None, flags: Optional[torch.Tensor] = None,
            transpose: bool = False, W2: Optional[DevBlock] = None, oz: Optional[OzakiOperator] = None,
            levels: int = 6) -> None:
    """W = op(A) X rounded to out_fmt (default W.fmt); colmax[j] = max|W[:,j]|; optionally
    W2 = the same product in W2.fmt (e.g. the fp32 accumulator).  An fp64 block against a
    16/8-bit operator runs as an FP64-accurate int8 tensor-core product (``oz``: prepared
    digit planes of A, made on the fly when absent)."""
    L = _lib.load()
    k = X.k
    if X.fmt == FpFormat.F64 and A.fmt in OZAKI_FMTS and not transpose:
        if out_fmt is not None and FpFormat(out_fmt) != W.fmt:
            raise ValueError("gemm_av (fp64 block): out_fmt must be W's format")
        ozaki_gemm(oz if oz is not None else OzakiOperator(A), X, W, colmax=colmax, flags=flags, W2=W2, levels=levels)
        return
    ws_b = L.ofrr_gemm_av_workspace(A.rows, A.cols, k, int(A.fmt), int(transpose))
    ws = _ws(ws_b, A.device)
    of = int(W.fmt if out_fmt is None else out_fmt)
    split = A.fmt == FpFormat.BF16 and X.fmt == FpFormat.F32 and not transpose
    slices = {2: 1, 4: 2}.get(int(levels), 3)     # fp32 blocks: "levels" 2 / 4 / 6 = 1 / 2 / 3 bf16 slices
    if split:
        # fp32 block on the bf16 tensor cores (3 bf16 slices -- 2 for the lite policy -- one
        # pass over A)
        ws = _ws(L.ofrr_gemm_av_split_workspace(A.rows, A.cols, k), A.device)
        _lib.check(L.ofrr_gemm_av_split_slices(A.ptr, A.rows, A.cols, A.lda, int(A.fmt), X.ptr, X.ld, k, W.ptr, W.ld,
                                               of, _p(colmax), _p(flags), W2.ptr if W2 is not None else None,
                                               W2.ld if W2 is not None else 0, int(W2.fmt) if W2 is not None else of,
                                               slices, ws.data_ptr(), ws.numel(), _stream()), "gemm_av_split")
    else:
        if X.fmt != A.fmt:
            raise ValueError(f"gemm_av: block format {X.fmt.name} with operator format {A.fmt.name}")
        _lib.check(L.ofrr_gemm_av2(A.ptr, A.rows, A.cols, A.lda, int(A.fmt), int(transpose), X.ptr, X.ld, k,
                                   W.ptr, W.ld, of, _p(colmax), _p(flags), W2.ptr if W2 is not None else None,
                                   W2.ld if W2 is not None else 0, int(W2.fmt) if W2 is not None else of,
                                   ws.data_ptr(), ws.numel(), _stream()), "gemm_av")
    if split or (A.fmt.tensor_core and not transpose):
        # algorithmic bytes of the tensor-core kernel: A once + the B operand
        # once (3 bf16 slices in split mode); W is written by the finalize kernel
        kcs = 256 if slices == 2 else 170
        chunks = [min(kcs, k - j0) for j0 in range(0, k, kcs)] if split else [k]   # one launch per chunk
        for kc in chunks:
            kb = slices * kc if split else kc
            nb = A.rows * A.cols * A.fmt.itemsize + A.cols * kb * (2 if split else X.fmt.itemsize)
            _log_gemm((nb, 2.0 * A.rows * A.cols * kb))
    _count(3 if split else 2 if (A.fmt.tensor_core and not transpose) else 1)


def scale_columns(X: DevBlock, colmax: torch.Tensor, compute: FpFormat) -> None:
    L = _lib.load()
    _lib.check(L.ofrr_scale_columns(X.ptr, X.n, X.k, X.ld, int(X.fmt), int(compute), colmax.data_ptr(), _stream()),
               "scale_columns")
    _count(1)


# ---------------------------------------------------------------------------------
# K3
# ---------------------------------------------------------------------------------
@dataclass
class HessOut:
    Q: DevBlock          # k columns allocated; first n_kept valid
    pivots: torch.Tensor  # int64[k]
    kept: torch.Tensor    # int32[k]
    n_kept: torch.Tensor  # int32[1]


def hessenberg(X: DevBlock, storage: FpFormat, compute: FpFormat, tol: float,
               n_kept_out: Optional[torch.Tensor] = None) -> HessOut:
    """K3.  ``n_kept_out`` (int32[1], e.g. a slot of the driver's status word): the kernel
    writes the kept count there directly (no copy node in a captured iteration)."""
    L = _lib.load()
    dev = X.device
    if FpFormat(storage) != X.fmt:
        Xs = new_block(X.n, X.k, storage, dev)
        convert(X, Xs)
        X = Xs
    Q = new_block(X.n, X.k, storage, dev)
    piv, kept, nk = _zeros_pack(dev, ((max(X.k, 1),), torch.int64), ((max(X.k, 1),), torch.int32),
                                ((1,), torch.int32))
    if n_kept_out is not None:
        nk = n_kept_out
    ws_b = L.ofrr_hessenberg_workspace(X.n, X.k, int(storage))
    ws = _ws(ws_b, dev)
    _lib.check(L.ofrr_hessenberg(X.ptr, X.n, X.k, X.ld, int(storage), int(compute), float(tol), Q.ptr, Q.ld,
                                 piv.data_ptr(), kept.data_ptr(), nk.data_ptr(), ws.data_ptr(), ws.numel(),
                                 _stream()), "hessenberg")
    _count(1)
    return HessOut(Q, piv, kept, nk)


# Gram-Schmidt comparators: ofrr/basis.py:65-148 on the device
GS_METHODS = {"mgs-l": 0, "mgs-r": 1, "cgs": 2, "cgs2": 3}


def orthonormalize(X: DevBlock, method: str, storage: FpFormat, compute: FpFormat, accumulate: FpFormat,
                   drop_tol: float, reorth: bool = True) -> HessOut:
    """Gram-Schmidt basis of X (kept columns first; pivots empty)."""
    L = _lib.load()
    dev = X.device
    if FpFormat(storage) != X.fmt:
        Xs = new_block(X.n, X.k, storage, dev)
        convert(X, Xs)
        X = Xs
    Q = new_block(X.n, X.k, storage, dev)
    piv, kept, nk = _zeros_pack(dev, ((1,), torch.int64), ((max(X.k, 1),), torch.int32), ((1,), torch.int32))
    ws = _ws(L.ofrr_orthonormalize_workspace(X.n, X.k), dev)
    _lib.check(L.ofrr_orthonormalize(X.ptr, X.n, X.k, X.ld, int(storage), int(compute), int(accumulate),
                                     float(drop_tol), GS_METHODS[method], int(bool(reorth)), Q.ptr, Q.ld,
                                     kept.data_ptr(), nk.data_ptr(), ws.data_ptr(), ws.numel(), _stream()),
               "orthonormalize")
    _count(1)
    return HessOut(Q, piv[:0], kept, nk)


# ---------------------------------------------------------------------------------
# K4
# ---------------------------------------------------------------------------------
def gram(U: DevBlock, W: Optional[DevBlock], out_fmt: FpFormat, flags: Optional[torch.Tensor] = None,
         want_m: bool = True):
    """(G1 = U^T W, G2 = U^T U) as fp64 (k x kw) / (k x k) tensors, column-major
    (returned as torch tensors of shape (kw, k) / (k, k): row j = column j)."""
    L = _lib.load()
    dev = U.device
    k = U.k
    kw = W.k if W is not None else 0
    G1 = torch.empty((max(kw, 1), k), dtype=torch.float64, device=dev) if W is not None else None
    G2 = torch.empty((k, k), dtype=torch.float64, device=dev) if want_m else None
    ws = _ws(L.ofrr_gram_workspace(U.n, k, kw), dev)
    if W is not None and W.fmt != U.fmt:
        raise ValueError("gram: U and W must share a storage format")
    _lib.check(L.ofrr_gram(U.ptr, U.ld, _p(W.t) if W is not None else None, W.ld if W is not None else 0, U.n, k, kw,
                           int(U.fmt), int(out_fmt), _p(G1), _p(G2), _p(flags), ws.data_ptr(), ws.numel(),
                           _stream()), "gram")
    _count(2)
    return G1, G2


# ---------------------------------------------------------------------------------
# K5
# ---------------------------------------------------------------------------------
@dataclass
class EigOut:
    values: torch.Tensor   # fp64[k]
    vectors: torch.Tensor  # fp64 (k, k): row j = eigenvector j (column-major k x k)
    n_out: torch.Tensor    # int32[1]
    status: torch.Tensor   # int32[1]


def sym_def_gen_eig(B: torch.Tensor, M: torch.Tensor, k: int, n_out_out: Optional[torch.Tensor] = None,
                    status_out: Optional[torch.Tensor] = None) -> EigOut:
    """B, M: fp64 column-major k x k (torch (k, k) with row j = column j).  ``n_out_out`` /
    ``status_out`` (int32[1], zeroed): written by the kernels directly (status-word slots)."""
    L = _lib.load()
    dev = B.device
    kk = max(k, 1)
    vals, vecs, n_out, status = _zeros_pack(dev, ((kk,), torch.float64), ((kk, kk), torch.float64),
                                            ((1,), torch.int32), ((1,), torch.int32))
    if n_out_out is not None:
        n_out = n_out_out
    if status_out is not None:
        status = status_out
    ws = _ws(L.ofrr_small_eig_workspace(k), dev)
    _lib.check(L.ofrr_sym_def_gen_eig(B.data_ptr(), M.data_ptr(), k, vals.data_ptr(), vecs.data_ptr(),
                                      n_out.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), _stream()),
               "sym_def_gen_eig")
    _count(8 if 1 <= k <= 160 else 1)   # pencil pipeline (7) + the gated general kernel
    return EigOut(vals, vecs, n_out, status)


def sym_eig(S: torch.Tensor, k: int) -> EigOut:
    L = _lib.load()
    dev = S.device
    vals = torch.zeros(max(k, 1), dtype=torch.float64, device=dev)
    vecs = torch.zeros((max(k, 1), max(k, 1)), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = _ws(L.ofrr_small_eig_workspace(k), dev)
    _lib.check(L.ofrr_sym_eig(S.data_ptr(), k, vals.data_ptr(), vecs.data_ptr(), status.data_ptr(), ws.data_ptr(),
                              ws.numel(), _stream()), "sym_eig")
    n_out = torch.full((1,), k, dtype=torch.int32, device=dev)
    _count(1)
    return EigOut(vals, vecs, n_out, status)


# ---------------------------------------------------------------------------------
# K6 / K7
# ---------------------------------------------------------------------------------
def ritz(U: DevBlock, Y: torch.Tensor, ldy: int, r_dev: Optional[torch.Tensor], r_max: int, scale: float = 1.0,
         want64: bool = True, x_fmt: Optional[FpFormat] = None, flags: Optional[torch.Tensor] = None,
         row_offset: int = 0):
    """Ut = scale * U Y[:, :r] (fp64 block) and/or X = round(Ut, x_fmt)."""
    L = _lib.load()
    dev = U.device
    U64 = new_block(U.n, r_max, FpFormat.F64, dev) if want64 else None
    X = new_block(U.n, r_max, x_fmt, dev) if x_fmt is not None else None
    Yp = Y.data_ptr() + row_offset * 8
    _lib.check(L.ofrr_ritz_recover(U.ptr, U.ld, int(U.fmt), U.n, U.k, Yp, ldy, _p(r_dev), r_max, float(scale),
                                   _p(U64.t) if U64 else None, U64.ld if U64 else 0, _p(X.t) if X else None,
                                   X.ld if X else 0, int(x_fmt) if x_fmt is not None else 0, _p(flags), _stream()),
               "ritz_recover")
    _count(1)
    return U64, X


def reuse_power(W: DevBlock, Y: torch.Tensor, ldy: int, r_dev: Optional[torch.Tensor], r_max: int,
                x_fmt: FpFormat, colmax: torch.Tensor, flags: Optional[torch.Tensor] = None) -> DevBlock:
    """The next power step from the projection (A-pass reuse): X = round(W Y, x_fmt) with
    W = A U, so X = A (U Y); colmax gets the column inf-norms of X (zeroed by the caller)."""
    L = _lib.load()
    X = new_block(W.n, r_max, x_fmt, W.device)
    _lib.check(L.ofrr_reuse_power(W.ptr, W.ld, int(W.fmt), W.n, W.k, Y.data_ptr(), ldy, _p(r_dev), r_max, _p(X.t),
                                  X.ld, int(x_fmt), colmax.data_ptr(), _p(flags), _stream()), "reuse_power")
    _count(1)
    return X


def restart(U: DevBlock, W: Optional[DevBlock], Y: torch.Tensor, ldy: int, r_dev: Optional[torch.Tensor], r_max: int,
            want64: bool = False, xu_fmt: Optional[FpFormat] = None, flags_u: Optional[torch.Tensor] = None,
            xw_fmt: Optional[FpFormat] = None, colmax: Optional[torch.Tensor] = None,
            flags_w: Optional[torch.Tensor] = None, vals: Optional[torch.Tensor] = None, t: int = 0, mode: int = 0):
    """K6f: the restart step in one pass over (U, W) -- ritz (U64 = U Y, Xu = round(U Y)),
    reuse_power (Xw = round(W Y) + colmax, zeroed by the caller) and residual_estimate
    (columns < t) fused.  Returns (U64, Xu, Xw, est); absent outputs are None."""
    L = _lib.load()
    dev = U.device
    t = min(int(t), r_max) if (W is not None and vals is not None) else 0
    U64 = new_block(U.n, r_max, FpFormat.F64, dev) if want64 else None
    Xu = new_block(U.n, r_max, xu_fmt, dev) if xu_fmt is not None else None
    Xw = new_block(U.n, r_max, xw_fmt, dev) if (xw_fmt is not None and W is not None) else None
    est = torch.zeros(max(t, 1), dtype=torch.float64, device=dev) if t > 0 else None
    ws = _ws(L.ofrr_restart_workspace(U.n, t), dev) if t > 0 else None
    _lib.check(L.ofrr_restart(U.ptr, U.ld, int(U.fmt), W.ptr if W is not None else None, W.ld if W is not None else 0,
                              int(W.fmt) if W is not None else 0, U.n, U.k, Y.data_ptr(), ldy, _p(r_dev), r_max,
                              _p(Xu.t) if Xu else None, Xu.ld if Xu else 0, int(xu_fmt) if Xu else 0, _p(flags_u),
                              _p(U64.t) if U64 else None, U64.ld if U64 else 0,
                              _p(Xw.t) if Xw else None, Xw.ld if Xw else 0, int(xw_fmt) if Xw else 0, _p(flags_w),
                              _p(colmax) if Xw is not None else None,
                              vals.data_ptr() if t > 0 else None, t, est.data_ptr() if t > 0 else None, int(mode),
                              ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0,
                              _stream()), "restart")
    _count(2 if t > 0 else 1)
    return U64, Xu, Xw, est


def residual_estimate(U: DevBlock, W: DevBlock, Y: torch.Tensor, ldy: int, vals: torch.Tensor,
                      r_dev: Optional[torch.Tensor], r_max: int, mode: int = 0) -> torch.Tensor:
    """K7e: ||(W - lambda_j U) y_j|| / |lambda_j| (mode 0) or raw sums of squares (mode 2)."""
    L = _lib.load()
    res = torch.zeros(max(r_max, 1), dtype=torch.float64, device=U.device)
    ws = _ws(L.ofrr_residual_estimate_workspace(U.n, r_max), U.device)
    _lib.check(L.ofrr_residual_estimate(U.ptr, U.ld, int(U.fmt), W.ptr, W.ld, int(W.fmt), U.n, U.k, Y.data_ptr(),
                                        ldy, vals.data_ptr(), _p(r_dev), r_max, res.data_ptr(), mode, ws.data_ptr(),
                                        ws.numel(), _stream()), "residual_estimate")
    _count(2)
    return res


def residual_eig(A: DevOperator, V: DevBlock, vals: torch.Tensor, r_dev: Optional[torch.Tensor], r_max: int):
    L = _lib.load()
    res = torch.zeros(max(r_max, 1), dtype=torch.float64, device=A.device)
    ws = _ws(L.ofrr_residual_workspace2(A.rows, A.cols, r_max, int(A.fmt), 0), A.device)
    _lib.check(L.ofrr_residual_eig(A.ptr, A.rows, A.lda, int(A.fmt), V.ptr, V.ld, vals.data_ptr(), _p(r_dev), r_max,
                                   res.data_ptr(), ws.data_ptr(), ws.numel(), _stream()), "residual_eig")
    _count(5 if A.fmt in (FpFormat.BF16, FpFormat.F16, FpFormat.FP8_E4M3) else 2)
    return res


def residual_pair(A: DevOperator, transpose: bool, Xv: DevBlock, Yv: DevBlock, vals: torch.Tensor,
                  r_dev: Optional[torch.Tensor], r_max: int, res: torch.Tensor, accumulate_max: bool):
    L = _lib.load()
    m = A.cols if transpose else A.rows
    ws = _ws(L.ofrr_residual_workspace2(A.rows, A.cols, r_max, int(A.fmt), int(transpose)), A.device)
    _lib.check(L.ofrr_residual_pair(A.ptr, A.rows, A.cols, A.lda, int(A.fmt), int(transpose), Xv.ptr, Xv.ld, Yv.ptr,
                                    Yv.ld, vals.data_ptr(), _p(r_dev), r_max, res.data_ptr(), int(accumulate_max),
                                    ws.data_ptr(), ws.numel(), _stream()), "residual_pair")
    _count(2)
    return res


def generate_sym(A: DevOperator, row0: int, hadamard: bool, c, s, Wf, Mf) -> None:
    """Evaluate the synthetic symmetric matrix rows [row0, row0 + A.rows) on device."""
    L = _lib.load()
    dev = A.device
    n = A.cols
    ct = torch.as_tensor(c, dtype=torch.float64).to(dev)
    st = torch.as_tensor(s, dtype=torch.float64).to(dev)
    r = Wf.shape[1]
    Wt = torch.as_tensor(Wf.T.copy(), dtype=torch.float64).to(dev)   # [r][n]
    Mt = torch.as_tensor(Mf.T.copy(), dtype=torch.float64).to(dev)
    _lib.check(L.ofrr_generate_sym(n, row0, A.rows, int(hadamard), ct.data_ptr(), st.data_ptr(), Wt.data_ptr(),
                                   Mt.data_ptr(), r, A.ptr, A.lda, int(A.fmt), _stream()), "generate_sym")
    torch.cuda.current_stream().synchronize()
