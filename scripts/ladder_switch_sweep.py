"""C3 ladder (fp32 rung -> fp64 rung, A-pass reuse) time-to-1e-8 vs ladder_switch."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3-ladder-reuse"]
dev = torch.device("cuda")
lam = p.geometric_spectrum(cfg["n"], cfg["top"], cfg["k"])
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
for sw in (1e-3, 3e-4, 1e-4, 3e-5):
    icfg = p.IterConfig(k=cfg["k"], m=bench.MAX_OUTER, iter=1, basis_method=p.BasisMethod.HESS_LEFT,
                        projection="ofrr", policy=p.POLICY_PRESETS[cfg["policy"]], seed=bench.SEED, tol=cfg["tol"],
                        top=cfg["top"], ladder=p.POLICY_PRESETS[cfg["ladder"]], ladder_switch=sw,
                        reuse_av=bool(cfg.get("reuse", False)))
    for _ in range(3):
        p.subspace_iter_eig(A, icfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = p.RunStats()
    e0.record()
    rs = p.subspace_iter_eig(A, icfg, stats=st)
    e1.record()
    torch.cuda.synchronize()
    print(f"switch {sw:.0e}: {e0.elapsed_time(e1):.1f} ms, its {st.iterations}, passes {st.a_passes}, "
          f"max res {np.max(rs.residuals[:cfg['top']]):.1e}, history {[f'{w:.0e}' for _, w in st.history]}")
