"""K7 FP64 residual timing at the C2 / C3 shapes (OFRR_RESID_DMMA=1: the FP64 DMMA kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402
from micro_kernels_util import timeit  # noqa: E402

dev = torch.device("cuda")
rng = np.random.default_rng(0)
for n, r in ((16384, 64), (65536, 128)):
    A, _ = p.synthetic_symmetric(p.geometric_spectrum(n, r // 2, r), p.FpFormat.BF16, seed=1, device=dev)
    Aop = A.device_operator()
    U = ops.block_from_host(rng.standard_normal((n, r)), p.FpFormat.F64, dev)
    vals = torch.ones(r, dtype=torch.float64, device=dev)
    t = timeit(lambda: ops.residual_eig(Aop, U, vals, None, r), reps=5)
    res = ops.residual_eig(Aop, U, vals, None, r).cpu().numpy()
    kind = "dmma" if os.environ.get("OFRR_RESID_DMMA") == "1" else "ozaki-int8"
    print(f"K7 {kind} n={n} r={r}: {t * 1e3:.1f} us  ({2.0 * n * n * r / (t * 1e-3) / 1e12:.1f} fp64-equivalent TFLOP/s)  "
          f"res[0:3]={res[:3]}")
    del A, Aop, U
    torch.cuda.empty_cache()
