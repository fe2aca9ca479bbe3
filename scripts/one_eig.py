"""A single K5 pencil solve (for ncu): python scripts/one_eig.py [k]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_00281_b200 import ops  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rng = np.random.default_rng(0)
b = rng.standard_normal((k, k)); b = (b + b.T) / 2
r = rng.standard_normal((k, k)); m = r.T @ r + 0.5 * np.eye(k)
B = torch.tensor(b.T.copy(), device="cuda"); M = torch.tensor(m.T.copy(), device="cuda")
out = ops.sym_def_gen_eig(B, M, k)
torch.cuda.synchronize()
print("status", int(out.status.item()), "n_out", int(out.n_out.item()))
