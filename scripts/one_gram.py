"""Three K4 Gram launches at C2 shape (n=16384, k=kw=64, fp32 basis), for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402

dev = torch.device("cuda")
rng = np.random.default_rng(0)
n, k = 16384, 64
X = ops.block_from_host(rng.random((n, k)).astype(np.float32).astype(np.float64), p.FpFormat.F32, dev)
for _ in range(3):
    ops.gram(X, X, p.FpFormat.F64)
torch.cuda.synchronize()
