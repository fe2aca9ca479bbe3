"""K1 launches at C2 shape for ncu: bf16 block (k=64) and fp32 block via the 3-slice split."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda")
A, _ = p.synthetic_symmetric(p.geometric_spectrum(n, 32, 64), p.FpFormat.BF16, seed=1)
Aop = A.device_operator()
for fmt in (p.FpFormat.BF16, p.FpFormat.F32):
    X = ops.start_block(1, n, k, fmt, dev)
    W = ops.new_block(n, k, fmt, dev)
    cm = torch.zeros(k, dtype=torch.float64, device=dev)
    for _ in range(3):
        ops.gemm_av(Aop, X, W, colmax=cm)
torch.cuda.synchronize()
print("ok")
