"""K3 Hessenberg at the C3 shape (65536 x 128): time per launch and CTA 0's per-column phase
breakdown (ofrr_debug_hess_profile), fp32 (rows in shared memory) and fp64 (global panels)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import _lib, ops  # noqa: E402
from micro_kernels_util import timeit  # noqa: E402

dev = torch.device("cuda")
rng = np.random.default_rng(0)
L = _lib.load()
L.ofrr_debug_hess_profile.argtypes = [ctypes.c_void_p]
names = ["wait->reduce", "prow", "scale+col j+1", "publish+arrive", "deferred update", "wait", "panel-end PR", "panel-end blocked update", "panel load", "panel-end scan+barrier", "scale loop (before the pivot-row stores)"]
for (n, k, fmt, comp) in ((65536, 128, p.FpFormat.F32, p.FpFormat.F32), (65536, 128, p.FpFormat.F64, p.FpFormat.F64),
                          (16384, 64, p.FpFormat.F32, p.FpFormat.F32)):
    X = ops.block_from_host(p.round_to(rng.random((n, k)), fmt), fmt, dev)
    t = timeit(lambda: ops.hessenberg(X, fmt, comp, 2.0 ** -20))
    out = (ctypes.c_ulonglong * 11)()
    L.ofrr_debug_hess_profile(ctypes.addressof(out))
    print(f"n={n} k={k} {fmt.name}: {t * 1e3:.1f} us ({t * 1e3 / k:.2f} us/column); CTA0 per column: " +
          ", ".join(f"{nm} {out[i] / 1e3 / k:.2f}" for i, nm in enumerate(names)) + " (us)", flush=True)
