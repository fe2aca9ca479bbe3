"""Hessenberg timing vs rows-per-CTA (OFRR_HESS_MIN_ROWS) and the FP64 residual kernel."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402
from micro_kernels_util import timeit  # noqa: E402

dev = torch.device("cuda")
rng = np.random.default_rng(0)
for (n, k, fmt) in ((16384, 64, p.FpFormat.F32), (16384, 64, p.FpFormat.BF16), (65536, 128, p.FpFormat.BF16)):
    X = ops.block_from_host(p.round_to(rng.random((n, k)), fmt), fmt, dev)
    t = timeit(lambda: ops.hessenberg(X, fmt, p.FpFormat.F32, 2.0**-7))
    print(f"K3 hessenberg n={n} k={k} {fmt.name} min_rows={os.environ.get('OFRR_HESS_MIN_ROWS', '128')}: {t * 1e3:.1f} us")

import ctypes  # noqa: E402
from paper_2505_00281_b200 import _lib  # noqa: E402
L = _lib.load()
for (n, k, fmt) in ((16384, 64, p.FpFormat.F32), (65536, 128, p.FpFormat.F32)):
    X = ops.block_from_host(p.round_to(rng.random((n, k)), fmt), fmt, dev)
    t = timeit(lambda: ops.hessenberg(X, fmt, p.FpFormat.F32, 2.0**-7))
    out = (ctypes.c_ulonglong * 8)()
    L.ofrr_debug_hess_profile.argtypes = [ctypes.c_void_p]
    L.ofrr_debug_hess_profile(ctypes.addressof(out))
    names = ["wait->reduce", "prow", "scale+col j+1", "publish+arrive", "deferred update", "wait"]
    print(f"n={n} k={k} {fmt.name}: {t * 1e3:.1f} us; CTA0 per-step: " +
          ", ".join(f"{nm} {out[i] / 1e3 / k:.2f}" for i, nm in enumerate(names)) + " (us)")
