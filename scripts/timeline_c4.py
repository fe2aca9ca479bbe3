"""Device timeline of one C4 SVD solve (per-kernel busy time): python scripts/timeline_c4.py [m]"""
import os, sys
from collections import defaultdict
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00281_b200 as p  # noqa: E402
m = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda")
A, sigma = p.synthetic_lowrank(1 << 20, 4096, p.FpFormat.F16, seed=20240901, device=dev)
cfg = p.IterConfig(k=200, m=m, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr", policy=p.TC_F16,
                   seed=20240901)
p.subspace_iter_svd(A, cfg)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    p.subspace_iter_svd(A, cfg)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy, cnt = defaultdict(float), defaultdict(int)
for e in ev:
    busy[e.name[:70]] += e.time_range.end - e.time_range.start
    cnt[e.name[:70]] += 1
t0, t1 = min(e.time_range.start for e in ev), max(e.time_range.end for e in ev)
print(f"C4 m={m}: first->last kernel {(t1 - t0) / 1e3:.1f} ms, busy {sum(busy.values()) / 1e3:.1f} ms")
for nm, b in sorted(busy.items(), key=lambda x: -x[1])[:20]:
    print(f"  {b / 1e3:9.2f} ms  x{cnt[nm]:3d}  {nm}")
