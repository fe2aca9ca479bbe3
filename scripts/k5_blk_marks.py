"""Debug: raw phase marks (globaltimer ns) of one K5 pencil solve at k (k_pc_chol_blk: 0 load,
4 first diagonal block, 5 first panel, 1 factorisation, 2 inverse, 3 certificate)."""
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
for i in (20, 21, 1, 2, 3):
    print(f"mark {i}: {(t[i] - t[0]) / 1e3:8.1f} us after load")
