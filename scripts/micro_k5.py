"""K5 pencil solve timing (OFRR_K5_LEGACY=1: the single-kernel path)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_00281_b200 import ops  # noqa: E402
from micro_kernels_util import timeit  # noqa: E402

for k in (32, 64, 100, 128, 160):
    rng = np.random.default_rng(k)
    b = rng.standard_normal((k, k))
    b = (b + b.T) / 2
    r = rng.standard_normal((k, k))
    m = r.T @ r + 0.5 * np.eye(k)
    B = torch.tensor(b.T.copy(), device="cuda")
    M = torch.tensor(m.T.copy(), device="cuda")
    t = timeit(lambda: ops.sym_def_gen_eig(B, M, k), reps=10)
    e = ops.sym_def_gen_eig(B, M, k)
    import scipy.linalg as sl
    w = sl.eigh(b, m, eigvals_only=True)[::-1]
    err = np.max(np.abs(e.values.cpu().numpy()[:k] - w)) / np.max(np.abs(w))
    y = e.vectors.cpu().numpy().T[:, :k]
    res = np.max(np.abs(b @ y - m @ y * e.values.cpu().numpy()[None, :k]))
    print(f"K5 k={k:4d} {'legacy' if os.environ.get('OFRR_K5_LEGACY') == '1' else 'pipeline'}: {t * 1e3:8.1f} us"
          f"  max rel err vs scipy {err:.2e}  max |By - My lam| {res:.2e}")

import ctypes  # noqa: E402
from paper_2505_00281_b200 import _lib  # noqa: E402
if os.environ.get("OFRR_K5_LEGACY") != "1":
    L = _lib.load()
    out = (ctypes.c_ulonglong * 24)()
    L.ofrr_debug_pencil_profile.argtypes = [ctypes.c_void_p]
    for k in (64, 128):
        rng = np.random.default_rng(k)
        b = rng.standard_normal((k, k)); b = (b + b.T) / 2
        r = rng.standard_normal((k, k)); m = r.T @ r + 0.5 * np.eye(k)
        B = torch.tensor(b.T.copy(), device="cuda"); M = torch.tensor(m.T.copy(), device="cuda")
        ops.sym_def_gen_eig(B, M, k); torch.cuda.synchronize()
        L.ofrr_debug_pencil_profile(ctypes.addressof(out))
        t = list(out)
        names = ["chol", "inverse", "cert+write", "(gemms)", "tridiag", "bisect", "Q", "eigvec", "mgs+Z"]
        print(f"k={k}: " + ", ".join(f"{nm} {(t[i + 1] - t[i]) / 1e3:.1f}" for i, nm in enumerate(names)) + " us")
