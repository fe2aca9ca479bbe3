"""One K3 launch per storage format at the C3 shape (65536 x 128), F32 then F64 -- the
command profiled by ncu (profiles/r02_hess_c3_*)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402

rng = np.random.default_rng(0)
for fmt in (p.FpFormat.F32, p.FpFormat.F64):
    X = ops.block_from_host(p.round_to(rng.random((65536, 128)), fmt), fmt, torch.device("cuda"))
    ops.hessenberg(X, fmt, fmt, 2.0 ** -20)
    torch.cuda.synchronize()
