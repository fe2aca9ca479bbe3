"""Summaries of the ncu captures of scripts/profile_round.sh -> profiles/ (text, committed).

python scripts/summarize_profiles.py <round tag> [gpurun_out dir]"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
SRC = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (SM cycles)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__cluster_dim_x", "cluster size"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (elapsed)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor memory (smem->TC) active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def summarize_rep(name, note):
    rep = os.path.join(SRC, name + ".ncu-rep")
    if not os.path.exists(rep):
        rep = os.path.join(OUT, f"{TAG}_{name}.ncu-rep")
    if not os.path.exists(rep):
        return
    d = raw(rep)
    if d is None:
        return
    lines = [f"# ncu --set full --clock-control none --import-source on : {name} ({note})",
             f"# kernel: {d.get('Kernel Name', ('?', ''))[0]}", ""]
    for key, label in METRICS:
        if key in d:
            v, u = d[key]
            lines.append(f"{label:32s} {v} {u}")
    txt = os.path.join(OUT, f"{TAG}_{name}_summary.txt")
    with open(txt, "w") as f:
        f.write("\n".join(lines) + "\n")
    dst = os.path.join(OUT, f"{TAG}_{name}.ncu-rep")
    if os.path.abspath(rep) != os.path.abspath(dst):
        os.replace(rep, dst)
    print("wrote", txt)


def launches(name="launches_c2_bench.csv"):
    path = os.path.join(SRC, name)
    if not os.path.exists(path):
        return
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    per = defaultdict(dict)
    for r in rows:
        per[r["ID"]]["name"] = r["Kernel Name"]
        per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for v in per.values():
        nm = v["name"].split("(")[0][:70]
        a = agg[nm]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0)
        a[2] += v.get("dram__bytes_read.sum", 0.0)
        a[3] += v.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = ["# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
             "#   python bench.py --steps 2 --warmup 3 --no-cpu   (all launches: warm-up, timed and e2e solves)",
             "# per kernel: launches, total ns, share, mean ns/launch, DRAM MB read+write per launch",
             "# (cold-cache and serialised under ncu: compare shares, not absolute times)", ""]
    for nm, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:6d}  {t:14.0f} ns  {100 * t / tot:5.1f}%  {t / n:12.0f} ns/launch  "
                     f"{(rd + wr) / n / 1e6:10.1f} MB/launch  {nm}")
    out = os.path.join(OUT, f"{TAG}_launches_c2_bench.txt")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    launches()
    summarize_rep("k1_c2", "K1 bf16 block k=64 at C2 shape, third launch")
    summarize_rep("k1_wide_c3", "K1 wide tile as cluster pairs, fp32 block k=128 split (N=384) at C3 shape 65536^2")
    summarize_rep("ozk_gemm_c2", "K7z int8 Ozaki product with in-kernel digit conversion, C2 residual r=64")
    summarize_rep("oz_rowscale_c2", "K7z row scales of A (one pass over A), C2")
    summarize_rep("gram_c2", "K4 Gram partials (DMMA), n=16384 k=64 fp32 basis")
    summarize_rep("hess_c2", "K3 Hessenberg basis n=16384 k=64")
    summarize_rep("pc_tri_k64", "K5c register-resident Householder tridiagonalisation, k=64")
    summarize_rep("pc_eigvec_k64", "K5d eigenpairs of the tridiagonal + back-transformation (multi-CTA), k=64")
    summarize_rep("pc_chol_k64", "K5a Cholesky + inverse of the Gram M, k=64")
    summarize_rep("resid_est_c2", "K7e residual estimate (DMMA), C2: n=16384, kp=64, r=32")
