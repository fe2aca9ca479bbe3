"""Where the e2e step of bench.py goes: H2D of A, solve, D2H of the results (host clock)."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402
cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda")
n, top, k = cfg["n"], cfg["top"], cfg["k"]
lam = p.geometric_spectrum(n, top, k)
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
icfg = p.IterConfig(k=k, m=bench.MAX_OUTER, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                    policy=p.POLICY_PRESETS[cfg["policy"]], seed=bench.SEED, tol=cfg["tol"], top=top)
fmt = p.FpFormat[cfg["fmt"]]
a_host = A.device_operator(fmt).t[:, :n].to("cpu").pin_memory()
op = ops.new_operator(n, n, fmt, dev)
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op.t[:, :n].copy_(a_host, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    Ah = p.DenseMatrix.on_device(op)
    st = p.RunStats()
    rsh = p.subspace_iter_eig(Ah, icfg, stats=st)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    vals = np.asarray(rsh.values)
    vecs = rsh.vectors.data
    t3 = time.perf_counter()
    print(f"h2d {1e3 * (t1 - t0):.2f} ms  solve {1e3 * (t2 - t1):.2f} ms (device loop {st.device_loop})  "
          f"d2h {1e3 * (t3 - t2):.2f} ms")
