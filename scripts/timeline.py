"""Device timeline of one bench-configured solve (torch.profiler / CUPTI): per-kernel busy
time, and the idle gaps between launches (host overhead / syncs).
python scripts/timeline.py [c2|c3]"""
import os
import sys
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
dev = torch.device("cuda")
n, top, k = cfg["n"], cfg["top"], cfg["k"]
lam = p.geometric_spectrum(n, top, k)
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
icfg = p.IterConfig(k=k, m=bench.MAX_OUTER, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                    policy=p.POLICY_PRESETS[cfg["policy"]], seed=bench.SEED, tol=cfg["tol"], top=top,
                    ladder=p.POLICY_PRESETS[cfg["ladder"]] if cfg.get("ladder") else None,
                    reuse_av=bool(cfg.get("reuse", False)))
for _ in range(3):
    p.subspace_iter_eig(A, icfg)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    p.subspace_iter_eig(A, icfg)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy = defaultdict(float)
cnt = defaultdict(int)
gaps = []
prev_end = t0
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    busy[e.name[:60]] += d
    cnt[e.name[:60]] += 1
    if s > prev_end:
        gaps.append((s - prev_end, e.name[:40]))
    prev_end = max(prev_end, e.time_range.end)
tot = t1 - t0
print(f"{name}: first kernel -> last kernel {tot / 1e3:.3f} ms, kernels busy {sum(busy.values()) / 1e3:.3f} ms, "
      f"idle {sum(g for g, _ in gaps) / 1e3:.3f} ms in {len(gaps)} gaps")
for nm, b in sorted(busy.items(), key=lambda x: -x[1]):
    print(f"  {b:9.1f} us  x{cnt[nm]:3d}  {nm}")
print("largest gaps (us, next kernel):")
for g, nm in sorted(gaps, reverse=True)[:15]:
    print(f"  {g:8.1f}  {nm}")
