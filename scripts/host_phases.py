"""Host-side phases of one device-loop solve (bench config): EigEngine construction, start
block, the device loop call (launch + the one sync + unpacking), the rest of run().
python scripts/host_phases.py [c2|c3]"""
import os
import sys
import time
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import driver  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dev = torch.device("cuda")
lam = p.geometric_spectrum(cfg["n"], cfg["top"], cfg["k"])
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
icfg = p.IterConfig(k=cfg["k"], m=bench.MAX_OUTER, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                    policy=p.POLICY_PRESETS[cfg["policy"]], seed=bench.SEED, tol=cfg["tol"], top=cfg["top"],
                    reuse_av=bool(cfg.get("reuse", False)))
acc = defaultdict(float)


def wrap(cls, name):
    f = getattr(cls, name)

    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[name] += time.perf_counter() - t
    setattr(cls, name, g)


for nm in ("__init__", "start_block", "_device_loop", "run", "_block_oz", "_graph_capable"):
    wrap(driver.EigEngine, nm)
for _ in range(4):
    p.subspace_iter_eig(A, icfg)
torch.cuda.synchronize()
acc.clear()
R = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(R):
    p.subspace_iter_eig(A, icfg)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / R
print(f"per solve: wall {1e6 * wall:.0f} us, events {1e3 * e0.elapsed_time(e1) / R:.0f} us")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:16s} {1e6 * v / R:8.1f} us")
