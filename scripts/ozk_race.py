import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
import paper_2505_00281_b200 as p
from paper_2505_00281_b200 import ops
import oracle as o
from test_gpu_kernels import _op, _blk
rng = np.random.default_rng(5)
rows, cols, k = 4000, 16000, 64
a = o.round_to(rng.standard_normal((rows, cols)) * np.exp(rng.uniform(-3, 3, (rows, 1))), 3)
x = rng.standard_normal((cols, k))
A = _op(p, a, 3)
oz = ops.OzakiOperator(A)
X = _blk(p, x, 2)
ref = (torch.as_tensor(a, device="cuda") @ torch.as_tensor(x, device="cuda")).cpu().numpy()
mag = np.abs(a) @ np.abs(x)
for flag in ("1", "0"):
    os.environ["OFRR_OZK_TMEM_A"] = flag
    outs = []
    for _ in range(int(os.environ.get("NREP", "6"))):
        W = ops.new_block(rows, k, p.FpFormat.F64, torch.device("cuda"))
        ops.gemm_av(A, X, W, oz=oz)
        torch.cuda.synchronize()
        outs.append(W.to_numpy_f64())
    for i, w in enumerate(outs):
        bad = np.abs(w - ref) > (2.0 ** -44 + cols * 2.0 ** -53) * mag
        r_, c_ = np.nonzero(bad)
        if bad.sum() or not np.array_equal(w, outs[0]) or i == len(outs) - 1: print(flag, i, "bad", bad.sum(), "rows", np.unique(r_)[:20], "cols", np.unique(c_)[:8], "== first", np.array_equal(w, outs[0]))
