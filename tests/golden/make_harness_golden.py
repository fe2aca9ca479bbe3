"""Golden CSV results of the REFERENCE experiment harness (ofrr/cli.py, imported read-only
from /root/reference/pkg/src, pure-numpy kernel backend) on two small spec files, for the
B200 harness parity test (tests/test_harness.py).  Only this script touches
/root/reference; the committed spec texts and CSV outputs travel to the GPU box.

    python tests/golden/make_harness_golden.py
"""
import json
import os
import sys

REF = "/root/reference/pkg/src"
os.environ.setdefault("OFRR_PURE_PYTHON", "1")
sys.path.insert(0, REF)
from ofrr import cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SPECS = {
    "harness_eig": """# small kernel-eig grid (OFRR cells + one classical cell)
experiment = kernel-eig
n = 400
f = 0.2
l = 10
s = 0.01
k = 20
m = 6
iter = 2
top = 10
seed = 20240901
cell = full-f64:full-f64:hess-l:ofrr
cell = full-f32:full-f32:hess-l:ofrr
cell = mixed-half:mixed-half:hess-l:ofrr
cell = full-f64:full-f64:hess-r:ofrr
cell = full-f64:full-f64:mgs-l:rr
""",
    "harness_svd": """# small kernel-svd grid
experiment = kernel-svd
n = 400
n2 = 60
f = 0.2
l = 3
k = 16
m = 6
iter = 1
top = 8
seed = 20240901
cell = full-f64:full-f64:hess-l:ofrr
cell = full-f32:full-f32:hess-l:ofrr
cell = mixed-half:mixed-half:hess-l:ofrr
""",
}


def main():
    out = {}
    for name, text in SPECS.items():
        path = os.path.join(HERE, name + ".cfg")
        with open(path, "w") as fh:
            fh.write(text)
        spec = cli.parse_spec_file(path)
        rows = cli.run_experiment(spec)
        buf_path = os.path.join(HERE, name + ".ref.csv")
        cli.write_results(rows, "csv", buf_path)
        # matrix fingerprint: the reference's own generator on the same spec
        a = cli._kernel_matrix(spec) if spec.experiment == "kernel-eig" else cli._cross_kernel_matrix(spec)
        d = a.data
        out[name] = {"sum": float(d.sum()), "diag0": float(d[0, 0]), "a37": float(d[3, 7]),
                     "shape": list(d.shape)}
    with open(os.path.join(HERE, "harness_fingerprints.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
