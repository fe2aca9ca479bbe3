"""K3: the global-memory mode with shared-memory panels vs the default mode -- bitwise
agreement and timing (C2 fp32, C3 fp32, C3 fp64, a bf16 case with a dropped column)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops, _lib  # noqa: E402
from micro_kernels_util import timeit  # noqa: E402

L = _lib.load()
L.ofrr_debug_hess_mode.argtypes = [ctypes.c_int, ctypes.c_int]
L.ofrr_debug_hess_profile.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda")
rng = np.random.default_rng(0)
for (n, k, fmt, comp) in ((16384, 64, p.FpFormat.F32, p.FpFormat.F32), (65536, 128, p.FpFormat.F32, p.FpFormat.F32),
                          (65536, 128, p.FpFormat.F64, p.FpFormat.F64), (5000, 40, p.FpFormat.BF16, p.FpFormat.F32)):
    x = p.round_to(rng.random((n, k)) - 0.5, fmt)
    x[:, 7] = x[:, 3] * 2.0                                     # a dropped column
    X = ops.block_from_host(x, fmt, dev)
    ref = None
    for mode in ((0, -1), (1, 1), (1, 8), (1, 16), (1, 32)):
        L.ofrr_debug_hess_mode(*mode)
        h = ops.hessenberg(X, fmt, comp, 2.0**-7)
        q = (h.Q.t.float() if fmt != p.FpFormat.F64 else h.Q.t).cpu().numpy()[:, :n]   # valid rows only
        piv = h.pivots.cpu().numpy()
        if ref is None:
            ref = (q, piv)
        same = np.array_equal(ref[0], q) and np.array_equal(ref[1], piv)
        t = timeit(lambda: ops.hessenberg(X, fmt, comp, 2.0**-7))
        out = (ctypes.c_ulonglong * 8)()
        L.ofrr_debug_hess_profile(ctypes.addressof(out))
        names = ["wait->reduce", "prow", "scale+col", "publish+arrive", "deferred", "wait"]
        print(f"K3 n={n} k={k} {fmt.name}/{comp.name} global={mode[0]} panel={mode[1]}: {t * 1e3:8.1f} us  "
              f"bitwise={same}  CTA0/step: " + " ".join(f"{nm} {out[i] / 1e3 / k:.2f}" for i, nm in enumerate(names)))
    L.ofrr_debug_hess_mode(0, -1)
