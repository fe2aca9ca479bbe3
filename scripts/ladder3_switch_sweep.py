"""C3 three-rung ladder (F32L -> F64L -> F64): time-to-1e-8 vs the two switch points,
alternating the candidates over rounds (device events around one solve, after warm-up)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402
cfg = dict(bench.CONFIGS["c3-ladder3l"])
dev = torch.device("cuda")
lam = p.geometric_spectrum(cfg["n"], cfg["top"], cfg["k"])
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
cands = [tuple(float(x) for x in s.split(",")) for s in (sys.argv[1:] or ["1e-4,1e-6", "3e-4,1e-6", "3e-5,1e-6", "1e-4,3e-6"])]
times = {c: [] for c in cands}
info = {}
for rnd in range(4):
    for c in cands:
        icfg = bench.make_iter_config(p, dict(cfg, switch=c))
        for _ in range(2 if rnd == 0 else 1):
            p.subspace_iter_eig(A, icfg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = p.RunStats()
        e0.record()
        rs = p.subspace_iter_eig(A, icfg, stats=st)
        e1.record()
        torch.cuda.synchronize()
        times[c].append(e0.elapsed_time(e1))
        info[c] = (st.iterations, st.a_passes, float(np.max(rs.residuals[:cfg["top"]])), getattr(st, "rungs", None))
for c in cands:
    print(f"switch {c}: median {np.median(times[c]):.2f} ms {[round(t, 2) for t in times[c]]}, its/passes/res/rungs {info[c]}")
