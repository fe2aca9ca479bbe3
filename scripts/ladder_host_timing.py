"""Host-side cost of the ladder's rung transitions (EigEngine construction, start-block
conversion, device-rung launch) for the default config: wall-clock phases of one solve
after warm-up, with the device synchronised at each phase boundary (diagnostic only)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import driver  # noqa: E402

cfg = bench.CONFIGS[bench.DEFAULT_CONFIG]
dev = torch.device("cuda")
lam = p.geometric_spectrum(cfg["n"], cfg["top"], cfg["k"])
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
icfg = bench.make_iter_config(p, cfg)
for _ in range(4):
    p.subspace_iter_eig(A, icfg)
torch.cuda.synchronize()

orig_init, orig_run = driver.EigEngine.__init__, driver.EigEngine.run
log = []


def init(self, *a, **k):
    t0 = time.perf_counter()
    orig_init(self, *a, **k)
    log.append(("EigEngine.__init__", time.perf_counter() - t0))


def run(self, *a, **k):
    t0 = time.perf_counter()
    out = orig_run(self, *a, **k)
    log.append((f"run({self.pol.storage.name}, levels {self.pol.product_levels})", time.perf_counter() - t0))
    return out


driver.EigEngine.__init__, driver.EigEngine.run = init, run
for rep in range(3):
    log.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    p.subspace_iter_eig(A, icfg)
    e1.record()
    torch.cuda.synchronize()
    print(f"solve: wall {1e3 * (time.perf_counter() - t0):.2f} ms, device {e0.elapsed_time(e1):.2f} ms; " +
          ", ".join(f"{nm} {1e6 * dt:.0f} us" for nm, dt in log), flush=True)
