"""Benchmark: OFRR top-k eigenpairs, time-to-tolerance on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

Default workload (every N): BASELINE configs[2] / SURVEY.md 8 "C3", the north-star target:
synthetic dense symmetric 65536 x 65536 (bf16 operator, 8 GiB, HBM resident), geometric
spectrum (rho = 0.1^(1/(k-top+1))), top-64 eigenpairs, k = 128, hess-l + ofrr, stopped when
the FP64 relative residuals of the leading 64 pairs are below 1e-8.  The basis runs a
three-rung precision ladder: an fp32 basis whose products take 2 bf16 slices of the block on
the bf16 tensor cores (K1: 16-bit block digits, fp32 sums -- at K = 65536 the fp32 sums'
own noise is of the same order, so the third slice buys no earlier switch) until the
residual estimate reaches 1e-4, then an fp64 basis with
~30-bit int8 Ozaki products (K7z, 4 levels) until 1e-6, then FP64-accurate K7z products (6
levels), whose W = A U also yields the FP64 residual report; A-pass reuse
(IterConfig.reuse_av) makes every outer iteration after the first one A pass.  One step = one complete solve from
X0 until convergence is confirmed in FP64.  A (8 GiB) is larger than L2 (126 MB): no flush.

N > 1: one process per GPU (NCCL).  `python bench.py --gpus N` without WORLD_SIZE re-launches
itself under torch.distributed.run; A is row-partitioned (each rank generates its own rows),
the time is the max over ranks, the problem size is fixed ("strong" scaling).

Other configs (--config): c2 (16384^2, top-32, tol 1e-2), c3 (tol 1e-2), c2-ladder, c3-ladder,
c2-f64, c3-f64, ... (parity/secondary cases).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20240901
DEFAULT_CONFIG = "c3-ladder3l"
CONFIGS = {
    "c2": dict(n=16384, top=32, k=64, fmt="BF16", tol=1e-2, policy="full-f32",
               name="synthetic dense symmetric 16384x16384 (bf16 operator), geometric spectrum, top-32, k=64, "
                    "bf16 tensor-core products with the basis as 3 bf16 slices (fp32-accurate) / fp64 Gram "
                    "(BASELINE configs[1])"),
    "c2-bf16": dict(n=16384, top=32, k=64, fmt="BF16", tol=2e-2, policy="tc-bf16",
                    name="synthetic dense symmetric 16384x16384, geometric spectrum, top-32, k=64, "
                         "pure bf16 basis (floor ~1.7e-2) / fp64 Gram"),
    "c3": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-2, policy="full-f32",
               name="synthetic dense symmetric 65536x65536, geometric spectrum, top-64, k=128, "
                    "bf16 operator, fp32-accurate basis on bf16 tensor cores / fp64 Gram, tol 1e-2"),
    "c2-f64": dict(n=16384, top=32, k=64, fmt="BF16", tol=1e-8, policy="full-f64",
                   name="synthetic dense symmetric 16384x16384 (bf16 operator), geometric spectrum, top-32, k=64, "
                        "to 1e-8: fp64 basis with FP64-accurate products on the int8 tensor cores (Ozaki "
                        "digit planes) / fp64 Gram"),
    "c2-ladder": dict(n=16384, top=32, k=64, fmt="BF16", tol=1e-8, policy="full-f64", ladder="full-f32",
                      name="synthetic dense symmetric 16384x16384 (bf16 operator), geometric spectrum, top-32, "
                           "k=64, to 1e-8 by a precision ladder: fp32 basis on the bf16 tensor cores until the "
                           "estimate reaches 1e-3, then fp64 basis with int8 Ozaki products"),
    "c2-ladder-reuse": dict(n=16384, top=32, k=64, fmt="BF16", tol=1e-8, policy="full-f64", ladder="full-f32",
                            reuse=True, name="as c2-ladder, with A-pass reuse (IterConfig.reuse_av)"),
    "c3-ladder": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-8, policy="full-f64", ladder="full-f32",
                      name="synthetic dense symmetric 65536x65536 (bf16 operator), geometric spectrum, top-64, "
                           "k=128, to 1e-8 (north-star target) by a precision ladder: fp32 basis on the bf16 "
                           "tensor cores, then fp64 basis with int8 Ozaki products"),
    "c2-reuse": dict(n=16384, top=32, k=64, fmt="BF16", tol=1e-2, policy="full-f32", reuse=True,
                     name="as c2, with A-pass reuse (IterConfig.reuse_av): the restart block's MatVec is "
                          "W Y from the projection (one A pass per outer iteration after the first)"),
    "c3-ladder-reuse": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-8, policy="full-f64", ladder="full-f32",
                            reuse=True,
                            name="BASELINE configs[2] (north-star target): synthetic dense symmetric 65536x65536 "
                                 "(bf16 operator), geometric spectrum, top-64, k=128, to FP64 residual 1e-8 by the "
                                 "fp32 -> fp64 basis ladder (bf16 tensor cores -> int8 Ozaki FP64-accurate "
                                 "products), A-pass reuse"),
    "c3-ladder3": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-8, policy="full-f64",
                       ladder=("full-f32", "full-f64-lite"), switch=(1e-4, 1e-6), reuse=True,
                       name="BASELINE configs[2] (north-star target): synthetic dense symmetric 65536x65536 "
                            "(bf16 operator), geometric spectrum, top-64, k=128, to FP64 residual 1e-8 by a "
                            "three-rung basis ladder: fp32 (bf16 tensor cores) -> fp64 with ~30-bit int8 Ozaki "
                            "products -> fp64 with FP64-accurate products, A-pass reuse"),
    "c3-ladder3l": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-8, policy="full-f64",
                        ladder=("full-f32-lite", "full-f64-lite"), switch=(1e-4, 1e-6), reuse=True,
                        name="BASELINE configs[2] (north-star target): synthetic dense symmetric 65536x65536 "
                             "(bf16 operator), geometric spectrum, top-64, k=128, to FP64 residual 1e-8 by a "
                             "three-rung basis ladder: fp32 basis with 2-slice bf16 products (bf16 tensor cores) "
                             "-> fp64 with ~30-bit int8 Ozaki products -> fp64 with FP64-accurate products, "
                             "A-pass reuse"),
    "c3-ladder4": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-8, policy="full-f64",
                       ladder=("full-f32-lite", "full-f32", "full-f64-lite"), switch=(1e-2, 1e-4, 1e-6), reuse=True,
                       name="BASELINE configs[2] (north-star target): synthetic dense symmetric 65536x65536 "
                            "(bf16 operator), geometric spectrum, top-64, k=128, to FP64 residual 1e-8 by a "
                            "four-rung basis ladder: fp32 basis with 2 then 3 bf16 slices on the bf16 tensor cores "
                            "-> fp64 with ~30-bit then FP64-accurate int8 Ozaki products, A-pass reuse"),
    "c2-ladder3": dict(n=16384, top=32, k=64, fmt="BF16", tol=1e-8, policy="full-f64",
                       ladder=("full-f32", "full-f64-lite"), switch=(1e-4, 1e-6), reuse=True,
                       name="as c3-ladder3 at C2's size (16384^2, top-32, k=64)"),
    "c3-f64-reuse": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-8, policy="full-f64", reuse=True,
                         name="as c3-f64 (fp64 basis throughout, to 1e-8), with A-pass reuse (IterConfig.reuse_av)"),
    # sigma_i = 0.9^i puts sigma_100 = 2.7e-5 below the noise level (1e-4 sigma_1), so no basis
    # precision reaches a per-triplet relative tolerance on all top-100: C4 runs the reference's
    # fixed m outer iterations (ofrr/driver.py:141-173), m = 4
    "c4": dict(kind="svd", n1=1048576, n=4096, rank=256, top=100, k=200, fmt="F16", tol=None, m=4, policy="tc-f16",
               name="BASELINE configs[3]: partial SVD of a tall 1048576x4096 synthetic low-rank-plus-noise matrix "
                    "(G1 diag(0.9^i) G2^T + 1e-4 N, rank 256, fp16), top-100 singular triplets, k=200, fp16 basis "
                    "on the tensor cores (fp32 sums) / fp64 Grams, m=4 outer iterations (fixed, as the reference)"),
    "c3-f64": dict(n=65536, top=64, k=128, fmt="BF16", tol=1e-8, policy="full-f64",
                   name="synthetic dense symmetric 65536x65536 (bf16 operator), geometric spectrum, top-64, "
                        "k=128, to 1e-8 (the north-star target): fp64 basis, FP64-accurate int8 tensor-core "
                        "products / fp64 Gram"),
}
MAX_OUTER = 60
METRIC = "OFRR top-k eig time-to-tol"
METRIC_SVD = "OFRR top-k SVD time-to-tol"

# A passes per rung of one solve, as the GPU arm of the same config measured them on a B200
# (bench.py --impl ours prints them as config.rungs; profiles/r02_passes.json holds the run
# they come from).  The reference arm never touches a GPU, so it reads them from that file.
PASSES_FILE = os.path.join(ROOT, "profiles", "r02_passes.json")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def _num(x):
    """JSON-safe float (None for NaN / inf)."""
    return float(x) if x is not None and np.isfinite(x) else None


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML, every 2 ms in
    a background thread)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self._stop = threading.Event()
        self._ok = False

    def _run(self):
        import pynvml as nv
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self._stop.is_set():
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            for nm, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(nm)
            self._stop.wait(0.002)

    def __enter__(self):
        if os.environ.get("OFRR_BENCH_NO_CLOCKS"):       # diagnostics only
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._ok = True
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._ok = False
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


# ------------------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref = the reference's own compiled _kernels.pyx), on
# one host core (the reference's kernels are single-threaded)
# ------------------------------------------------------------------------------------
def _ref_kernels():
    """(gemm_mixed, kind): the reference's compiled kernel when oracle/_ref was built, else
    the oracle's C restatement (bitwise equal, tests/test_oracle_golden.py)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    try:
        import build_ref
        kern = build_ref.load()

        def gemm(a, b, c, acc, out):
            return kern.gemm_mixed(np.asfortranarray(a), np.asfortranarray(b), c, acc, out)
        return gemm, "reference", oracle
    except Exception:
        return oracle.mixed_gemm, "port", oracle


# the reference's gemm_mixed policy per rung label (lite rungs have no reference counterpart:
# the reference computes them at the full format)
_POL_CODES = {"F32": (1, 1, 1), "F32L": (1, 1, 1), "F64": (2, 2, 2), "F64L": (2, 2, 2), "BF16": (1, 1, 3),
              "F16": (1, 1, 0)}


def ref_pass_seconds(gemm, oracle, n: int, k: int, rung: str, rows: int, n_rows: int = None):
    """Seconds for ONE A pass (n x n operator times the n x k block) of the reference's
    gemm_mixed under the rung's policy, from `rows` rows timed (F-order A rows, exactly
    as apply_dense hands them to the kernel, ofrr/matrix.py:242-254), scaled to n rows."""
    c, acc, out = _POL_CODES.get(rung, (1, 1, 1))
    rng = np.random.default_rng(SEED)
    x = oracle.round_to(rng.random((n, k)), oracle.F64 if rung in ("F64", "F64L") else oracle.F32)
    a = np.asfortranarray(oracle.round_to(rng.standard_normal((rows, n)) * 1e-3, oracle.BF16))
    t0 = time.perf_counter()
    gemm(a, x, c, acc, out)
    dt = time.perf_counter() - t0
    return dt * (n if n_rows is None else n_rows) / rows, dt


def ref_c1_full_solve(gemm, oracle):
    """C1 (BASELINE configs[0]) solved in full in the reference's driver order
    (apply_dense -> scale_columns_inf -> hessenberg_basis -> ofrr_eig -> round_to, FP64
    residual report after every outer iteration, ofrr/driver.py:84-111) with the reference's
    own gemm_mixed for every A pass: 2000^2 geometric spectrum, top-10, k=20, full-f32,
    tol 1e-5 (the fp32 tolerance of SURVEY.md 8(d))."""
    import paper_2505_00281_b200 as p
    n, top, k = 2000, 10, 20
    lam = p.geometric_spectrum(n, top, k)
    f = p.sym_factors(lam, seed=SEED)
    a = np.asfortranarray(oracle.sym_from_factors(n, f.hadamard, f.c, f.s, f.Wf, f.Mf, oracle.F32))
    saved = oracle.mixed_gemm
    oracle.mixed_gemm = gemm
    try:
        hist = []
        t0 = time.perf_counter()
        rs = oracle.subspace_iter_eig(a, k=k, m=60, iters=1, pol=oracle.FULL_F32, seed=SEED, top=top, tol=1e-5,
                                      history=hist)
        dt = time.perf_counter() - t0
    finally:
        oracle.mixed_gemm = saved
    return {"seconds": dt, "outer_iterations": len(hist), "max_residual_top": float(np.max(rs.residuals[:top])),
            "workload": "C1: 2000x2000 geometric spectrum, top-10, k=20, full-f32, tol 1e-5, solved in full"}


def _rung_passes(cfg_name: str, cfg):
    """A passes per rung of one solve of this config on the GPU (profiles/r02_passes.json)."""
    try:
        with open(PASSES_FILE) as f:
            rec = json.load(f)[cfg_name]
        return [(r, int(p)) for r, p in rec["rungs"]], rec.get("source", PASSES_FILE)
    except Exception:
        rung = {"full-f64": "F64", "tc-f16": "F16", "native-f16": "F16", "mixed-half": "F16",
                "tc-bf16": "BF16"}.get(cfg["policy"], "F32")
        passes = 3 * cfg["m"] if cfg.get("kind") == "svd" and cfg.get("m") else 4
        return [(rung, passes)], f"no GPU record for this config: {passes} passes assumed"


def reference_estimate(cfg_name: str, cfg, budget_s: float):
    """One bounded sample of the reference's CPU path on the config: its A passes (94% of
    the reference's time) timed on a row sample for every rung of the ladder
    and extrapolated to the solve's pass count.  Returns (value_s, wall_s, detail)."""
    gemm, kind, oracle = _ref_kernels()
    n, k = cfg["n"], cfg["k"]
    rungs, src = _rung_passes(cfg_name, cfg)
    t0 = time.perf_counter()
    total = 0.0
    parts = []
    per_pass_s = {}
    for rung, passes in rungs:
        rows = max(1, int(budget_s / len(rungs) / max(ref_pass_seconds(gemm, oracle, n, k, rung, 1)[1], 1e-6)))
        per_pass, dt = ref_pass_seconds(gemm, oracle, n, k, rung, rows, n_rows=_rows(cfg))
        per_pass_s[rung] = per_pass
        total += per_pass * passes
        parts.append(f"{rung} rung: {rows} rows x {n} cols x k={k} timed in {dt:.2f} s -> {per_pass:.0f} s per "
                     f"A pass ({_rows(cfg)} rows) x {passes} passes")
    wall = time.perf_counter() - t0
    return total, wall, kind, "; ".join(parts) + f" (pass counts: {src})", per_pass_s


def run_reference(args, cfg):
    """--impl reference: the reference's CPU path on one host core of the box."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    gemm, kind, oracle = _ref_kernels()
    c1 = ref_c1_full_solve(gemm, oracle)
    vals, walls = [], []
    detail = ""
    for i in range(args.warmup + args.steps):
        v, wall, kind, detail, _ = reference_estimate(args.config, cfg, args.ref_seconds)
        if i >= args.warmup:
            vals.append(v)
            walls.append(wall)
    v = float(np.median(vals))
    ms_step = float(np.mean(walls)) * 1e3
    sample = (f"per step: {detail}; A passes only (lower bound on the reference's solve); "
              f"1 core of {os.cpu_count()} (the reference's kernels are single-threaded)")
    line = {
        "impl": "reference", "metric": METRIC_SVD if cfg.get("kind") == "svd" else METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "value_kind": "extrapolated: one A pass per rung timed on a row sample, times the GPU run's pass count; "
                      "ms_per_step is the measured wall time of one such bounded sample",
        "extrapolated": True,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": _dtype(cfg),
        "data": "synthetic", "config": _config_block(args.config, cfg, args.gpus),
        "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": kind, "sample": sample,
                         "extrapolated": True, "c1_full_solve": c1},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------
def _rows(cfg) -> int:
    """Rows of A: n1 for the tall SVD configs, n for the square eigen configs."""
    return int(cfg.get("n1", cfg["n"]))


def make_iter_config(p, cfg):
    """The IterConfig of a bench config (also used by tests/ and scripts/)."""
    return p.IterConfig(k=cfg["k"], m=cfg.get("m", MAX_OUTER), iter=cfg.get("iter", 1), basis_method=p.BasisMethod.HESS_LEFT,
                        projection="ofrr", policy=p.POLICY_PRESETS[cfg["policy"]], seed=SEED, tol=cfg["tol"],
                        top=cfg["top"] if cfg["tol"] is not None else None,
                        ladder=_ladder(p, cfg.get("ladder")), ladder_switch=cfg.get("switch", 1e-4),
                        reuse_av=bool(cfg.get("reuse", False)))


def _ladder(p, spec):
    """A ladder preset name, or a tuple of names (one rung each)."""
    if not spec:
        return None
    if isinstance(spec, (tuple, list)):
        return tuple(p.POLICY_PRESETS[s] for s in spec)
    return p.POLICY_PRESETS[spec]


def _dtype(cfg) -> str:
    if cfg.get("ladder"):
        return "bf16 operator; basis f32 (bf16 tensor cores) -> f64 (int8 tensor cores, Ozaki)"
    return {"full-f32": "bf16 operator; f32 basis (bf16 tensor cores)",
            "full-f64": "bf16 operator; f64 basis (int8 tensor cores, Ozaki)",
            "tc-bf16": "bf16", "tc-f16": "f16 operator and basis (f16 tensor cores, fp32 sums)"}.get(cfg["policy"],
                                                                                                   cfg["policy"])


def _config_block(name, cfg, world):
    n, rows = cfg["n"], _rows(cfg)
    out = {"workload": cfg["name"], "name": name, "kind": cfg.get("kind", "eig"), "n": n, "top": cfg["top"],
           "k": cfg["k"], "tol": cfg["tol"], "policy": cfg["policy"], "ladder": cfg.get("ladder"),
           "reuse_av": bool(cfg.get("reuse", False)), "iter": int(cfg.get("iter", 1)),
           "parallelism": f"row-partitioned x{world}" if world > 1 else "single",
           "l2": "inputs larger than L2 (A = %d MiB per GPU)" % (((rows + world - 1) // world) * n * 2 >> 20)}
    if rows != n:
        out["n1"] = rows
    return out


# kernel name -> (label, what its algorithmic work is); bytes / flops per launch are
# computed in _kernel_work from the config (SURVEY.md 8(d) per-unit figures)
_KNOWN = [
    ("k_gemm_av_tc", "K1 A.X block product (bf16 tensor cores)"),
    ("k_ozk_ts", "K7z FP64-accurate A.X (int8 tensor cores, Ozaki digit heads in TMEM)"),
    ("k_ozk_gemm", "K7z FP64-accurate A.X (int8 tensor cores, Ozaki digits)"),
    ("k_oz_gemm", "K7z (digit-plane variant)"),
    ("k_hessenberg", "K3 Hessenberg basis"),
    ("k_finalize", "K1 stream-K fixup + rounding + column norms"),
    ("k_oz_resid", "K7z fixup + scaling + residual sums"),
    ("k_oz_rowscale", "K7z row scales of A"),
    ("k_oz_slices_v", "K7z digits of the block"),
    ("k_gram", "K4 Grams"),
    ("k_restart_dmma", "K6f restart step: Ritz block + next power step + residual estimate (DMMA)"),
    ("k_ritz", "K6 Ritz recovery / reuse power step"),
    ("k_oz_tailmul", "K7z exact fp64 tails of A"),
    ("k_pc_", "K5 pencil pipeline"),
    ("k_small_eig", "K5 general pencil kernel"),
    ("k_resid_est", "K7e residual estimate"),
    ("k_residual_reduce", "K7e/K7 reduction"),
    ("k_split_bf16", "K1s fp32 -> 3 bf16 slices"),
    ("k_scale_columns", "K2 column scaling"),
    ("k_loop_", "device-loop control"),
]


def _label(name: str) -> str:
    for key, lab in _KNOWN:
        if key in name:
            return lab
    return "other (torch fills/copies, memcpy)"


def _ozk_args(name: str):
    """(BN, NP, NL) of a k_ozk_gemm<FMT, BN, NP, NL> / k_ozk_ts<FMT, BN, NL> (heads: NP = 3)
    instance from its kernel name."""
    import re
    m = re.search(r"k_ozk_ts<\s*(\d+),\s*(\d+),\s*(\d+)>", name)
    if m:
        return int(m.group(2)), 3, int(m.group(3))
    m = re.search(r"k_ozk_gemm<\s*(\d+),\s*(\d+),\s*(\d+)(?:,\s*(\d+))?>", name)
    if not m:
        return 64, 3, 6
    return int(m.group(2)), int(m.group(3)), int(m.group(4) or 6)


def _oz_products(name: str) -> int:
    """Digit products per column block of a K7z launch: plane p of A (p < NP) meets the NL - p
    digits of the block that keep its level below NL -- 15 for the FP64 heads (NP=3, NL=6),
    21 with all six planes, 9 for the ~30-bit lite tier (NP=3, NL=4)."""
    _, np_, nl = _ozk_args(name)
    return sum(nl - p for p in range(min(np_, nl)))


def _kernel_work(name: str, cfg, rows: int):
    """(bytes, ops, ops_kind) per launch of a kernel of this config (algorithmic: SURVEY.md
    8(d)); None where the kernel is latency-bound (pencil, control) or bookkeeping."""
    n, k = cfg["n"], cfg["k"]
    s_blk = 8 if "double" in name else 4
    if "k_ozk_gemm" in name or "k_ozk_ts" in name:
        bn, _, nl = _ozk_args(name)
        bn = min(bn, k)
        return rows * n * 2 + nl * n * bn, _oz_products(name) * 2.0 * rows * n * bn, "int8"
    if "k_hessenberg" in name:
        return 2 * n * k * s_blk, None, None
    if "k_gram_partial" in name:
        return n * k * 2 * s_blk, 4.0 * n * k * k, "fp64"
    if "k_restart_dmma" in name:                 # U Y and W Y: read U, W; write both rounded blocks
        return n * k * 4 * s_blk, 4.0 * n * k * k, "fp64"
    if "k_ritz" in name:
        return n * k * (s_blk + 8), 2.0 * n * k * k, "fp64"
    if "k_resid_est" in name:
        return n * k * 2 * 4, None, None
    if "k_oz_rowscale" in name:
        return rows * n * 2, None, None
    if "k_scale_columns" in name:
        return 2 * n * k * s_blk, None, None
    return None, None, None


def kernel_table(solve, cfg, rows, ms_step, nsolves=2):
    """Per-kernel device time of `nsolves` solves replayed right after the timed region (same
    process, same captured graphs), from CUPTI kernel records (torch.profiler).  The step time
    itself is never taken under the profiler; this only attributes it."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2505_00281_b200 import driver
    torch.cuda.synchronize()
    # CUPTI does not report every kernel replayed inside the conditional (WHILE) nodes of the
    # device-side loop, so these solves run the host-driven loop: the same captured iteration
    # graphs, one host sync per iteration
    driver.DEVICE_LOOP = False
    try:
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(nsolves):
                solve()
            torch.cuda.synchronize()
    finally:
        driver.DEVICE_LOOP = True
    agg = {}
    for ev in prof.events():
        if ev.device_type is None or "cuda" not in str(ev.device_type).lower() or ev.name.startswith("ofrr."):
            continue
        dur = getattr(ev, "device_time", None) or getattr(ev, "cuda_time", 0.0) or 0.0
        if dur <= 0:
            continue
        a = agg.setdefault(ev.name, [0, 0.0])
        a[0] += 1
        a[1] += dur / 1e3                     # us -> ms
    hbm, bf16_peak, _ = _peaks()
    int8_peak = 2.0 * bf16_peak                # nominal int8 : bf16 dense ratio (4.5 : 2.25 PFLOP/s)
    fp64_peak = 37.0                            # B200 nominal FP64 tensor TFLOP/s (no measured figure)
    rows_out = []
    busy = sum(v[1] for v in agg.values()) / nsolves
    for name, (cnt, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        per_solve = tot / nsolves
        avg_us = tot / cnt * 1e3
        r = {"kernel": name[:90], "role": _label(name), "launches_per_solve": cnt / nsolves,
             "avg_us": round(avg_us, 2), "ms_per_solve": round(per_solve, 4),
             "share_of_step": round(per_solve / ms_step, 4) if ms_step > 0 else None}
        nb, ops, kind = _kernel_work(name, cfg, rows)
        if nb is not None:
            gbs = nb / (avg_us * 1e-6) / 1e9
            r.update(bytes_per_launch=nb, hbm_gbs=round(gbs, 1), hbm_frac=round(gbs / hbm, 4))
        if ops is not None:
            tf = ops / (avg_us * 1e-6) / 1e12
            peak = int8_peak if kind == "int8" else fp64_peak
            r.update(ops_per_launch=ops, ops_kind=kind, tops=round(tf, 1), tensor_frac=round(tf / peak, 4),
                     tensor_peak=peak)
        if per_solve / ms_step >= 0.005 or len(rows_out) < 12:
            rows_out.append(r)
    return rows_out, busy


def _spawn(args) -> int:
    """`bench.py --gpus N` outside torchrun: run N ranks on this node (one per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_ours(args, cfg):
    import ctypes
    import torch
    import torch.distributed as dist
    import paper_2505_00281_b200 as p
    from paper_2505_00281_b200 import _lib, ops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return _dry_run(args, cfg, p, torch, dist, world, rank)
    # test knob (not for measurements): the multi-rank path on one GPU over gloo
    if os.environ.get("OFRR_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("OFRR_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    try:
        _run_ours(args, cfg, p, _lib, ops, torch, dist, ctypes, world, rank, local, dev)
    finally:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()


def _dry_run(args, cfg, p, torch, dist, world, rank):
    """--dry-run (CPU test of the launcher): rank set-up, row partition and one collective
    over gloo, no GPU work."""
    if world > 1:
        dist.init_process_group("gloo")
    comm = p.Comm.world()
    r0, r1 = comm.row_range(_rows(cfg))
    rows = torch.tensor([r1 - r0], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(rows)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "rows_total": int(rows.item()), "n": _rows(cfg),
                          "config": args.config}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _run_ours(args, cfg, p, _lib, ops, torch, dist, ctypes, world, rank, local, dev):
    comm = p.Comm.world()
    n, top, k, tol = cfg["n"], cfg["top"], cfg["k"], cfg["tol"]
    rows_all = _rows(cfg)
    fmt = p.FpFormat[cfg["fmt"]]
    r0, r1 = comm.row_range(rows_all)
    icfg = make_iter_config(p, cfg)
    svd = cfg.get("kind") == "svd"
    if svd:
        A, _ = p.synthetic_lowrank(rows_all, n, fmt, r=cfg["rank"], seed=SEED, device=dev, row0=r0, rows=r1 - r0)
        driver = p.subspace_iter_svd
    else:
        lam = p.geometric_spectrum(n, top, k)
        A, _ = p.synthetic_symmetric(lam, fmt, seed=SEED, device=dev, row0=r0, rows=r1 - r0)
        driver = p.subspace_iter_eig

    def solve(stats=None, a=None):
        return driver(A if a is None else a, icfg, stats=stats, comm=comm, n_global=rows_all)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    L = _lib.load()
    # in-kernel timers of the two block-product kernels on (their flags are baked into the CUDA
    # graphs captured during the warm-up: the outer iteration, the FP64 report and the
    # device-side loop that replays them, csrc/loop.cu)
    L.ofrr_prof_k1_stamp(1)
    L.ofrr_prof_oz_stamp(1)
    rs = None
    for _ in range(args.warmup):
        rs = solve()
    barrier()
    # ---- timed region: K solves, CUDA events on the launching stream -------------
    ops.GEMM_LOG = []
    ops.LAUNCHES[0] = 0
    stats = p.RunStats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import gc
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clk:
        barrier()
        L.ofrr_prof_k1_stamp(1)                          # zero the accumulators
        L.ofrr_prof_oz_stamp(1)
        e0.record()
        per = [] if os.environ.get("OFRR_BENCH_PER_STEP") else None
        for _ in range(args.steps):
            if per is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                per.append(ev)
            stats = p.RunStats()
            rs = solve(stats)
        e1.record()
        barrier()
    gc.enable()
    launches = ops.LAUNCHES[0]
    ms_total = e0.elapsed_time(e1)
    if per is not None:
        per.append(e1)
        print("per-step ms:", [round(per[i].elapsed_time(per[i + 1]), 3) for i in range(len(per) - 1)],
              file=sys.stderr)
    log = ops.GEMM_LOG
    ops.GEMM_LOG = None
    stamps = {}
    for nm, fn in (("k1", L.ofrr_prof_k1_read), ("oz", L.ofrr_prof_oz_read),
                   ("oz_fp64", lambda a, b: L.ofrr_prof_oz_read_tier(1, a, b)),
                   ("oz_lite", lambda a, b: L.ofrr_prof_oz_read_tier(2, a, b))):
        sm, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
        fn(ctypes.byref(sm), ctypes.byref(cnt))
        stamps[nm] = (float(sm.value), int(cnt.value))
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps

    # ---- e2e: public API with HOST buffers (A from pinned host memory, results back) --
    # Every step copies this rank's rows of A host -> device into the caller's operator buffer
    # (DenseMatrix.on_device; a fixed buffer keeps the captured CUDA graphs valid), solves, and
    # reads the values, FP64 Ritz vectors and residuals back to the host.
    # A symmetric square operator (one rank, eigen path) crosses PCIe as its upper triangle
    # only (ops.upload_symmetric, the dsyev(uplo) convention): the other triangle is mirrored
    # on the device while later row blocks are still in flight.
    a_host = A.device_operator(fmt).t[:, :n].to("cpu").pin_memory()
    op = ops.new_operator(r1 - r0, n, fmt, dev)
    sym_upload = not svd and world == 1 and (r1 - r0) == n
    times = []
    h2d = d2h = 0
    n_warm_e2e = 3          # eager, capture, device-loop build for the new operator address
    for i in range(max(1, min(3, args.steps)) + n_warm_e2e):
        barrier()
        t0 = time.perf_counter()
        if sym_upload:
            h2d = ops.upload_symmetric(op, a_host, "U")
        else:
            op.t[:, :n].copy_(a_host, non_blocking=True)
            h2d = a_host.numel() * a_host.element_size()
        Ah = p.DenseMatrix.on_device(op)
        rsh = solve(a=Ah)
        vals = np.asarray(rsh.values)
        vecs = rsh.vectors.data
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if i >= n_warm_e2e:
            times.append(float(dt.item()))
        d2h = vals.nbytes + vecs.nbytes + rsh.residuals.nbytes
        del Ah, rsh
    del op, a_host
    e2e = {"value": float(np.median(times)), "unit": "s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h)}
    if sym_upload:
        e2e["upload"] = "upper triangle of the symmetric host A (uplo='U', 2048-row 2-D copies; lower mirrored on the device)"
    if world > 1:
        e2e["note"] = "per-rank bytes (each rank copies its row block and reads its results); max over ranks"

    # ---- attribution: per-kernel device time (CUPTI) of two more solves -------------------
    table, busy = kernel_table(solve, cfg, r1 - r0, ms_step) if not args.no_table else ([], None)

    if rank != 0:
        return
    hbm, bf16_peak, peak_kind = _peaks()
    roof = _roofline(table, stamps, log, cfg, r1 - r0, ms_step, hbm, bf16_peak, peak_kind, args)
    cpu = None
    if world == 1 and not args.no_cpu:
        gemm, kind, oracle = _ref_kernels()
        total, wall, kind, detail, per_pass = reference_estimate(args.config, cfg, args.ref_seconds)
        # weighted by this run's own passes per rung (the same solve)
        total_here = sum(per_pass.get(rg, 0.0) * ps for rg, _, ps in stats.rungs) if stats.rungs else total
        c1 = ref_c1_full_solve(gemm, oracle)
        cpu = {"value": total_here, "unit": "s", "cores": 1, "kind": kind, "extrapolated": True,
               "sample": f"{detail}; re-weighted by this run's passes per rung {stats.rungs}; A passes only "
                         f"(lower bound on the reference's solve); 1 core of {os.cpu_count()}",
               "c1_full_solve": c1}
    line = {
        "metric": METRIC_SVD if svd else METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": _dtype(cfg), "data": "synthetic",
        "config": dict(_config_block(args.config, cfg, world),
                       outer_iterations_per_solve=stats.iterations, a_passes_per_solve=stats.a_passes,
                       rungs=[list(r) for r in stats.rungs], converged=bool(stats.converged),
                       max_residual_top=float(np.max(rs.residuals[:top])), device_loop=bool(stats.device_loop)),
        "roofline": roof,
        "kernels": {"source": "CUPTI kernel records (torch.profiler) of 2 solves run after the timed region with the "
                              "host-driven outer loop (same captured iteration graphs; CUPTI misses kernels inside "
                              "the device loop's conditional nodes); share_of_step = ms_per_solve / ms_per_step",
                    "busy_ms_per_solve": _num(busy), "table": table},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def _roofline(table, stamps, log, cfg, rows, ms_step, hbm, bf16_peak, peak_kind, args):
    """The time-dominant kernel (from the per-kernel table), its algorithmic work per launch
    and its average launch duration from its own in-kernel globaltimer stamps over the timed
    region (K1 / K7z), else from the CUPTI table."""
    n, k = cfg["n"], cfg["k"]
    dom = table[0]["kernel"] if table else ("k_ozk_ts<3, 64, 6>" if cfg["policy"] == "full-f64" else "k_gemm_av_tc")
    if "k_ozk_gemm" in dom or "k_ozk_ts" in dom:
        # the in-kernel stamps of this kernel's accuracy tier only (the lite and FP64-accurate
        # products are different instances with different work per launch)
        _, _, nl = _ozk_args(dom)
        sm, cnt = stamps["oz_lite" if nl == 4 else "oz_fp64"]
        avg_ms = sm / cnt if cnt else float("nan")
        nb, ops_, _ = _kernel_work(dom, cfg, rows)
        tops = ops_ / (avg_ms * 1e-3) / 1e12
        peak = 2.0 * bf16_peak
        gbs = nb / (avg_ms * 1e-3) / 1e9
        tier = "~30-bit lite" if nl == 4 else "FP64-accurate"
        out = {"kernel": f"{dom[:40]} (K7z: {tier} A.X on the int8 tensor cores, {_oz_products(dom)} "
                         "digit products)",
               "bound": "tensor", "achieved": _num(tops), "peak": peak, "unit": "TOP/s (int8)",
               "frac": _num(tops / peak), "peak_kind": f"derived: 2 x {peak_kind} bf16 {bf16_peak} "
                                                     "(nominal dense int8:bf16 ratio, 4.5:2.25 P/s)",
               "hbm_gbs": _num(gbs), "hbm_frac": _num(gbs / hbm), "ops_per_launch": ops_, "bytes_per_launch": nb,
               "avg_launch_ms": _num(avg_ms), "launches": cnt, "timing": "in-kernel globaltimer stamps, timed region",
               "fp64_equiv_tflops": _num(2.0 * rows * n * (64 if k > 32 else 32) / (avg_ms * 1e-3) / 1e12)}
    else:
        sm, cnt = stamps["k1"]
        avg_ms = sm / cnt if cnt else float("nan")
        nbytes = float(np.mean([b for b, _ in log])) if log else float("nan")
        flops = float(np.mean([f for _, f in log])) if log else float("nan")
        achieved = nbytes / (avg_ms * 1e-3) / 1e9
        tensor_bound = np.isfinite(flops) and np.isfinite(nbytes) and flops / nbytes > bf16_peak * 1e3 / hbm
        tf = flops / (avg_ms * 1e-3) / 1e12
        out = {"kernel": "k_gemm_av_tc (K1, A.X block product)", "bytes_per_launch": _num(nbytes),
               "avg_launch_ms": _num(avg_ms), "launches": cnt, "timing": "in-kernel globaltimer stamps, timed region",
               "peak_kind": peak_kind,
               "algorithmic_tflops": _num(2.0 * rows * n * k / (avg_ms * 1e-3) / 1e12) if cnt else None}
        if tensor_bound:
            out.update(bound="tensor", achieved=_num(tf), peak=bf16_peak, unit="TFLOP/s", frac=_num(tf / bf16_peak),
                       hbm_gbs=_num(achieved), hbm_frac=_num(achieved / hbm))
        else:
            out.update(bound="hbm", achieved=_num(achieved), peak=hbm, unit="GB/s", frac=_num(achieved / hbm))
    out["share_of_step"] = _num(sm / ms_step / args.steps) if cnt else None
    out["traffic"], out["traffic_source"] = _profiled_traffic(args.config, out["kernel"])
    return out


def _profiled_traffic(cfg_name: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel from the committed
    ncu capture of the same config (profiles/r02_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            rec = json.load(f)
        key = "k_ozk_ts" if "k_ozk_ts" in kernel else "k_ozk_gemm" if "k_ozk_gemm" in kernel else "k_gemm_av_tc"
        e = rec[cfg_name][key]
        return float(e["bytes_per_launch"]), e["source"]
    except Exception:
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--ref-seconds", type=float, default=1.0, help="CPU seconds per reference sample step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-table", action="store_true", help="skip the per-kernel table")
    ap.add_argument("--dry-run", action="store_true", help="launcher / rank set-up only (CPU test)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("bench.py: --warmup must be >= 3 (the first solves of a shape capture its CUDA graphs)")
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
