"""Phase breakdown (globaltimer) of the K5 fast pipeline's single-CTA kernels for one pencil
solve: python scripts/pc_phases.py [k ...]"""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_00281_b200 import ops, _lib  # noqa: E402

L = _lib.load()
L.ofrr_debug_pencil_profile.argtypes = [ctypes.c_void_p]
names = {1: "chol", 2: "inverse", 3: "certificate", 5: "tri: householder", 6: "eigvec: launch+setup",
         7: "eigvec: multisection", 8: "eigvec: twisted vectors", 9: "eigvec: back-transform"}
for k in [int(a) for a in sys.argv[1:]] or [64, 128]:
    rng = np.random.default_rng(0)
    lam = 0.932 ** np.arange(k)
    q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    b = (q * lam) @ q.T
    r = rng.standard_normal((k, k)) / np.sqrt(k)
    m = np.eye(k) + 0.1 * (r @ r.T)
    B = torch.tensor(b.T.copy(), device="cuda"); M = torch.tensor(m.T.copy(), device="cuda")
    for _ in range(3):
        ops.sym_def_gen_eig(B, M, k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        ops.sym_def_gen_eig(B, M, k)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 20
    out = (ctypes.c_ulonglong * 24)()
    L.ofrr_debug_pencil_profile(ctypes.addressof(out))
    t = list(out)
    print(f"k={k}: pencil solve wall {wall * 1e6:.1f} us")
    for i in range(1, 10):
        if t[i] and t[i - 1] and i != 4 and t[i] >= t[i - 1]:
            print(f"  {names.get(i, str(i)):24s} {(t[i] - t[i - 1]) / 1e3:8.1f} us")
    hc = t[15] - t[14]
    if hc > 0 and t[5] > t[4]:
        print(f"  householder: {hc} SM cycles = {hc / max(k - 2, 1):.0f} per step; effective clock "
              f"{hc / ((t[5] - t[4]) * 1e-3):.0f} MHz")
