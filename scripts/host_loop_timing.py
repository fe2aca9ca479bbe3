"""Host-side timing of back-to-back solves of a bench config (device loop diagnostics)."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2505_00281_b200 as p  # noqa: E402
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dev = torch.device("cuda")
lam = p.geometric_spectrum(cfg["n"], cfg["top"], cfg["k"])
A, _ = p.synthetic_symmetric(lam, p.FpFormat[cfg["fmt"]], seed=bench.SEED, device=dev)
icfg = p.IterConfig(k=cfg["k"], m=bench.MAX_OUTER, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                    policy=p.POLICY_PRESETS[cfg["policy"]], seed=bench.SEED, tol=cfg["tol"], top=cfg["top"],
                    reuse_av=bool(cfg.get("reuse", False)))
for _ in range(4):
    p.subspace_iter_eig(A, icfg)
torch.cuda.synchronize()
for _ in range(5):
    t0 = time.perf_counter()
    rs = p.subspace_iter_eig(A, icfg)
    t1 = time.perf_counter()
    print(f"solve wall {1e6 * (t1 - t0):.0f} us")
