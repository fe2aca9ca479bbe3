"""K7z head/tail diagnostics at a bench config: tail counts per row, the operator mode and
the product time with the 3-digit heads vs all six digit planes (OFRR_OZ_FULL semantics).
python scripts/oz_tails.py [config]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402
from paper_2505_00281_b200 import ops  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_CONFIG
cfg = bench.CONFIGS[name]
dev = torch.device("cuda")
n, top, k = cfg["n"], cfg["top"], cfg["k"]
lam = p.geometric_spectrum(n, top, k)
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
op = A.device_operator(p.FpFormat.BF16)
t = op.t[:4096, :n].float().abs()
rm = t.max(dim=1).values
ratio = (rm[:, None] / torch.where(t > 0, t, torch.full_like(t, float("nan"))))
print("row max / entry (first 4096 rows): median", float(ratio.nanmedian()), "rows' max ratio median",
      float(torch.nan_to_num(ratio, nan=0).max(dim=1).values.median()))
print("entries below 2^-15 of the row max per row (mean):", float((t < rm[:, None] * 2.0 ** -15).sum(1).float().mean()))
oz = ops.OzakiOperator(op)
full, tails = oz.info()
print(f"operator: full={full} tails={tails} ({tails / n:.2f} per row)")
X = ops.start_block(1, n, k, p.FpFormat.F64, dev)
W = ops.new_block(n, k, p.FpFormat.F64, dev)
for _ in range(2):
    ops.gemm_av(op, X, W, oz=oz)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    ops.gemm_av(op, X, W, oz=oz)
e1.record()
torch.cuda.synchronize()
print(f"product n={n} k={k}: {e0.elapsed_time(e1) / 5:.3f} ms per A pass (both column passes)")
for _ in range(2):
    ops.gemm_av(op, X, W, oz=oz, levels=4)
e0.record()
for _ in range(5):
    ops.gemm_av(op, X, W, oz=oz, levels=4)
e1.record()
torch.cuda.synchronize()
print(f"lite product (4 levels) n={n} k={k}: {e0.elapsed_time(e1) / 5:.3f} ms per A pass")
e0.record()
for _ in range(3):
    oz.refresh()
e1.record()
torch.cuda.synchronize()
print(f"prepare (row scales + tails): {e0.elapsed_time(e1) / 3:.3f} ms")
if os.environ.get("OZT_NO_PROF"):
    sys.exit(0)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        ops.gemm_av(op, X, W, oz=oz)
    oz.refresh()
    torch.cuda.synchronize()
agg = {}
for ev in prof.events():
    if "cuda" in str(ev.device_type).lower():
        a = agg.setdefault(ev.name[:70], [0, 0.0])
        a[0] += 1
        a[1] += ev.device_time
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {t / c:10.1f} us x{c:3d}  {nm}")
try:
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    print("sm clock now", nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), "reasons", hex(nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
except Exception as e:
    print(e)
