"""bench.py's launcher and reference arm on the CPU (no GPU work).

* ``--gpus 2`` without WORLD_SIZE re-launches itself under torch.distributed.run (one rank
  per GPU); ``--dry-run`` stops after the rank set-up, the row partition of C3 and one
  gloo collective, so the spawn path is exercised here.
* ``--impl reference`` times the reference's CPU path (oracle/_ref or the C restatement)
  on a bounded sample and labels the extrapolation.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_spawn_two_ranks_gloo():
    env = dict(os.environ, NCCL_DEBUG="WARN")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["rows_total"] == lines[0]["n"] == 65536


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)


def test_reference_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--ref-seconds", "0.2"], capture_output=True, text=True, timeout=900,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _json_lines(r.stdout)
    assert line["impl"] == "reference" and line["extrapolated"] is True
    assert line["cpu_baseline"]["cores"] == 1
    assert line["steps"] * line["ms_per_step"] < 60_000           # bounded samples, not the extrapolation
    assert line["value"] > 100.0                                    # hours of single-core work at C3
    c1 = line["cpu_baseline"]["c1_full_solve"]
    assert c1["max_residual_top"] < 1e-5 and c1["outer_iterations"] >= 2
    assert line["config"]["n"] == 65536 and line["config"]["tol"] == 1e-8
