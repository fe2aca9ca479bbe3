"""Debug: per-step cycle split of K5c k_pc_tri_reg (needs a library built with
-DOFRR_PC_TRI_PROF, selected by OFRR_LIB_OVERRIDE): [0] barrier B -> A (p = tau S u and the
K reduction, slowest warp), [1] A -> B, [2] column j+1's group: A -> its reflector,
[3] the reflector itself."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_00281_b200 import ops, _lib  # noqa: E402
k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rng = np.random.default_rng(0)
b = rng.standard_normal((k, k)); b = (b + b.T) / 2
r = rng.standard_normal((k, k)); m = r.T @ r + 0.5 * np.eye(k)
B = torch.tensor(b.T.copy(), device="cuda"); M = torch.tensor(m.T.copy(), device="cuda")
for _ in range(3):
    ops.sym_def_gen_eig(B, M, k)
torch.cuda.synchronize()
L = _lib.load()
out = (ctypes.c_ulonglong * 24)()
L.ofrr_debug_pencil_profile.argtypes = [ctypes.c_void_p]
L.ofrr_debug_pencil_profile(ctypes.addressof(out))
t = list(out)
steps = k - 2
print(f"k={k}: tri phase {(t[5] - t[4]) / 1e3:.1f} us, {(t[15] - t[14]) / steps:.0f} cycles/step")
for i, name in enumerate(("B->A", "A->B", "grp A->refl", "refl")):
    print(f"  {name:12s} {t[16 + i] / steps:8.0f} cycles/step")
