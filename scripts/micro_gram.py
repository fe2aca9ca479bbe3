"""K4 Gram micro-timing (CUDA events) over chunk counts: python scripts/micro_gram.py"""
import os
import sys
import subprocess
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402

dev = torch.device("cuda")
rng = np.random.default_rng(0)
for (n, k) in ((16384, 64), (65536, 128)):
    X = ops.block_from_host(rng.random((n, k)).astype(np.float32).astype(np.float64), p.FpFormat.F32, dev)
    for ch in (None, 16, 32, 48, 74, 148, 296):
        if ch is None:
            os.environ.pop("OFRR_GRAM_CHUNKS", None)
        else:
            os.environ["OFRR_GRAM_CHUNKS"] = str(ch)
        f = lambda: ops.gram(X, X, p.FpFormat.F64)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record(); torch.cuda.synchronize()
        print(f"n={n} k={k} chunks={ch}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
