"""K3 at the C4 SVD shapes (U: 1M x 200 fp16 global-memory mode; V: 4096 x 200) with phases."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops, _lib  # noqa: E402
from micro_kernels_util import timeit  # noqa: E402
L = _lib.load()
L.ofrr_debug_hess_profile.argtypes = [ctypes.c_void_p]
L.ofrr_debug_hess_mode.argtypes = [ctypes.c_int, ctypes.c_int]
dev = torch.device("cuda")
for (n, k) in ((1 << 20, 200), (4096, 200)):
    for pb in (-1, 1, 4, 8):
        L.ofrr_debug_hess_mode(0, pb)
        X = ops.start_block(1, n, k, p.FpFormat.F16, dev)
        t = timeit(lambda: ops.hessenberg(X, p.FpFormat.F16, p.FpFormat.F32, 2.0**-7), reps=2)
        out = (ctypes.c_ulonglong * 8)()
        L.ofrr_debug_hess_profile(ctypes.addressof(out))
        names = ["wait->reduce", "prow", "scale+col", "publish+arrive", "deferred", "wait"]
        print(f"K3 n={n} k={k} f16 panel={pb}: {t * 1e3:9.1f} us  CTA0/step: " +
              " ".join(f"{nm} {out[i] / 1e3 / k:.2f}" for i, nm in enumerate(names)))
L.ofrr_debug_hess_mode(0, -1)
