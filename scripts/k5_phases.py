"""Phase breakdown (SM clocks) of one K5 pencil solve: python scripts/k5_phases.py [k]"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_00281_b200 import ops, _lib  # noqa: E402
k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rng = np.random.default_rng(0)
b = rng.standard_normal((k, k)); b = (b + b.T) / 2
r = rng.standard_normal((k, k)); m = r.T @ r + 0.5 * np.eye(k)
B = torch.tensor(b.T.copy(), device="cuda"); M = torch.tensor(m.T.copy(), device="cuda")
for _ in range(2):
    ops.sym_def_gen_eig(B, M, k)
torch.cuda.synchronize()
L = _lib.load()
out = (ctypes.c_longlong * 24)()
L.ofrr_debug_k5_profile.argtypes = [ctypes.c_void_p]
L.ofrr_debug_k5_profile(ctypes.addressof(out))
t = list(out)
names = ["cholesky", "tri_inverse", "whiten (2 mm)", "(eig-whitening path)", "jacobi(T)", "back-transform+sort"]
for i, nm in enumerate(names):
    if t[i + 1] and t[i]:
        print(f"{nm:24s} {(t[i + 1] - t[i]) / 1965.0:9.1f} us")
print(f"total {(t[6] - t[0]) / 1965.0:.1f} us")
tn = ["tridiagonalise", "bisection", "inverse iteration", "back-transform"]
for i, nm in enumerate(tn):
    if t[8 + i + 1] and t[8 + i]:
        print(f"  tri {nm:20s} {(t[8 + i + 1] - t[8 + i]) / 1965.0:9.1f} us")
print("  tri ok flag", t[13])
