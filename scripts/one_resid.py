"""One FP64 residual launch (K7) at C2 shape, for ncu."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402
n, r = 16384, 64
dev = torch.device("cuda")
A, _ = p.synthetic_symmetric(p.geometric_spectrum(n, 32, 64), p.FpFormat.BF16, seed=1)
Aop = A.device_operator()
rng = np.random.default_rng(0)
U = ops.block_from_host(rng.standard_normal((n, r)), p.FpFormat.F64, dev)
vals = torch.ones(r, dtype=torch.float64, device=dev)
res = ops.residual_eig(Aop, U, vals, None, r)
torch.cuda.synchronize()
print("ok", float(res[0]))
