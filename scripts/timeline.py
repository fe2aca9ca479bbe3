"""Device timeline of one bench-configured solve (torch.profiler / CUPTI): per-kernel busy
time, the idle gaps between kernels and the host phases (record_function ranges of the
driver) that overlap each large gap.
python scripts/timeline.py [config] [nsolves]"""
import os
import sys
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_CONFIG
nsol = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = bench.CONFIGS[name]
dev = torch.device("cuda")
n, top, k = cfg["n"], cfg["top"], cfg["k"]
lam = p.geometric_spectrum(n, top, k)
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
icfg = bench.make_iter_config(p, cfg)
for _ in range(4):
    p.subspace_iter_eig(A, icfg)
if os.environ.get("OFRR_TIMELINE_HOST_LOOP", "1") == "1":     # CUPTI misses kernels in conditional nodes
    from paper_2505_00281_b200 import driver
    driver.DEVICE_LOOP = False
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(nsol):
        p.subspace_iter_eig(A, icfg)
    torch.cuda.synchronize()
allev = list(prof.events())
ev = [e for e in allev if e.device_type == torch.autograd.DeviceType.CUDA and not e.name.startswith("ofrr.")]
ranges = [e for e in allev if e.device_type != torch.autograd.DeviceType.CUDA and e.name.startswith("ofrr.")]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy = defaultdict(float)
cnt = defaultdict(int)
gaps = []
prev_end, prev_name = t0, ""
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    busy[e.name[:60]] += d
    cnt[e.name[:60]] += 1
    if s > prev_end:
        gaps.append((s - prev_end, prev_end, s, prev_name[:40], e.name[:40]))
    if e.time_range.end > prev_end:
        prev_end, prev_name = e.time_range.end, e.name
tot = t1 - t0
print(f"{name}: {nsol} solve(s), first kernel -> last kernel {tot / 1e3:.3f} ms, kernels busy "
      f"{sum(busy.values()) / 1e3:.3f} ms, idle {sum(g[0] for g in gaps) / 1e3:.3f} ms in {len(gaps)} gaps")
for nm, b in sorted(busy.items(), key=lambda x: -x[1]):
    print(f"  {b:9.1f} us  x{cnt[nm]:3d}  {nm}")
print("largest gaps (us): after -> before, host phases overlapping")
for g, gs, ge, a, b in sorted(gaps, reverse=True)[:25]:
    ph = sorted({r.name for r in ranges if r.time_range.start < ge and r.time_range.end > gs})
    print(f"  {g:8.1f}  {a} -> {b}  {ph}")
print("host phases (ms total):")
agg = defaultdict(float)
for r in ranges:
    agg[r.name] += (r.time_range.end - r.time_range.start) / 1e3
for nm, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {v:9.3f}  {nm}")
