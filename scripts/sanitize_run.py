"""Small end-to-end solves that launch every hot kernel once or more (K1 incl. the fp32 split,
K2, K3, K4, K5 pipeline, K6, K7e, K7z heads + tails, the device loop), for compute-sanitizer
(memcheck / racecheck / synccheck): python scripts/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402

os.environ.setdefault("OFRR_CUDA_GRAPHS", "0")       # eager: the tools see every launch
dev = torch.device("cuda")
n, top, k = 2048, 16, 32
lam = p.geometric_spectrum(n, top, k)
A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=1, device=dev)
cfg = p.IterConfig(k=k, m=20, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr", policy=p.FULL_F64,
                   ladder=p.FULL_F32, seed=1, tol=1e-8, top=top, reuse_av=True)
st = p.RunStats()
rs = p.subspace_iter_eig(A, cfg, stats=st)
print("eig ladder:", st.iterations, "its, max residual", float(np.max(rs.residuals[:top])), flush=True)
cfg2 = p.IterConfig(k=k, m=3, iter=1, basis_method=p.BasisMethod.CGS2, projection="rr", policy=p.FULL_F32, seed=1)
rs2 = p.subspace_iter_eig(A, cfg2)
print("cgs2 + rr:", float(np.max(rs2.residuals[:top])), flush=True)
rng = np.random.default_rng(0)
a = rng.standard_normal((1500, 300)) * (0.9 ** np.arange(300))[None, :]
cfg3 = p.IterConfig(k=24, m=3, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr", policy=p.TC_F16,
                    seed=1)
rs3 = p.subspace_iter_svd(p.DenseMatrix(p.round_to(a, p.FpFormat.F16), p.FpFormat.F64), cfg3)
print("svd:", float(np.max(rs3.residuals[:8])), flush=True)
