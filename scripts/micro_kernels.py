"""Micro-timings (CUDA events, warm) of the non-GEMM kernels at C2/C3 shapes."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops, _lib  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = torch.device("cuda")
rng = np.random.default_rng(0)
for k in (20, 64, 128):
    b = rng.standard_normal((k, k)); b = (b + b.T) / 2
    r = rng.standard_normal((k, k)); m = r.T @ r + 0.5 * np.eye(k)
    B = torch.tensor(b.T.copy(), device=dev); M = torch.tensor(m.T.copy(), device=dev)
    t = timeit(lambda: ops.sym_def_gen_eig(B, M, k))
    # raw Jacobi sweeps via the host plugin entry
    L = _lib.load()
    import ctypes
    vals = np.zeros(k); vecs = np.zeros((k, k)); sw = ctypes.c_int(0); off = ctypes.c_double(0)
    s = np.ascontiguousarray(b)
    L.ofrr_host_jacobi_eig(s.ctypes.data, k, 30, 1e-14 * np.linalg.norm(s), vals.ctypes.data, vecs.ctypes.data,
                           ctypes.addressof(sw), ctypes.addressof(off))
    print(f"K5 sym_def_gen_eig k={k}: {t * 1e3:.1f} us; raw jacobi sweeps={sw.value} off={off.value:.2e}")

for (n, k) in ((16384, 64), (65536, 128)):
    x = rng.random((n, k))
    X = ops.block_from_host(p.round_to(x, p.FpFormat.BF16), p.FpFormat.BF16, dev)
    t = timeit(lambda: ops.hessenberg(X, p.FpFormat.BF16, p.FpFormat.F32, 2.0**-7))
    print(f"K3 hessenberg n={n} k={k}: {t * 1e3:.1f} us")
    G1 = timeit(lambda: ops.gram(X, X, p.FpFormat.F64))
    print(f"K4 gram n={n} k={k}: {G1 * 1e3:.1f} us")
    Y = torch.tensor(rng.standard_normal((k, k)), device=dev)
    tr = timeit(lambda: ops.ritz(X, Y, k, None, k, 1.0, want64=True, x_fmt=p.FpFormat.BF16))
    print(f"K6 ritz n={n} k={k}: {tr * 1e3:.1f} us")
    if n == 16384:
        lam = p.geometric_spectrum(n, 32, 64)
        A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=1)
        Aop = A.device_operator()
        U64, _ = ops.ritz(X, Y, k, None, k, 1.0, want64=True)
        vals = torch.ones(k, dtype=torch.float64, device=dev)
        for r in (32, 64):
            t7 = timeit(lambda: ops.residual_eig(Aop, U64, vals, None, r))
            print(f"K7 residual n={n} r={r}: {t7 * 1e3:.1f} us ({2 * n * n * r / t7 / 1e9:.2f} TFLOP/s fp64)")
