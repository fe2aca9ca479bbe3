"""One C2-sized OFRR solve with per-phase CUDA-event timing (for ncu launch lists and
quick breakdowns).  python scripts/prof_solve.py [n] [k] [top] [m]"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
top = int(sys.argv[3]) if len(sys.argv) > 3 else 32
m = int(sys.argv[4]) if len(sys.argv) > 4 else 3
pol = os.environ.get("POLICY", "tc-bf16")
mvp = os.environ.get("MV_POLICY", pol)
lam = p.geometric_spectrum(n, top, k)
A, _ = p.synthetic_symmetric(lam, p.FpFormat[os.environ.get("A_FMT", "BF16")], seed=20240901)
cfg = p.IterConfig(k=k, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                   policy=p.POLICY_PRESETS[pol], matvec_policy=p.POLICY_PRESETS[mvp], seed=20240901,
                   tol=1e-30, top=top)
p.subspace_iter_eig(A, cfg)  # warm-up
torch.cuda.synchronize()
st = p.RunStats()
t0 = time.perf_counter()
rs = p.subspace_iter_eig(A, cfg, stats=st)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"n={n} k={k} m={m}: {dt * 1e3:.2f} ms, {dt * 1e3 / m:.2f} ms/iter, history={st.history}")
