"""Build the reference's own compiled kernel module into oracle/_ref/ -- CHECKER ONLY.

Cythonizes /root/reference/pkg/src/ofrr/_kernels.pyx (with its halfround.h) in a
temporary directory and compiles it with gcc -O3 -mf16c (the reference's own flags,
pkg/setup.py:12-15) into oracle/_ref/_kernels.<abi>.so.  No reference source is copied
into the repository; only the built module lands in oracle/_ref/ (git-ignored, travels
to the GPU box).  It serves as `--impl reference` / cpu_baseline kind "reference"
(the reference's gemm_mixed, timed on the box's host cores) and to cross-check the C
restatement in ofrr_oracle.c.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
SRC = "/root/reference/pkg/src/ofrr"


def built_module():
    if not os.path.isdir(OUT):
        return None
    for f in os.listdir(OUT):
        if f.startswith("_kernels") and f.endswith(".so"):
            return os.path.join(OUT, f)
    return None


def build(force: bool = False) -> str:
    if built_module() and not force:
        return built_module()
    if not os.path.isdir(SRC):
        raise FileNotFoundError(SRC)
    import numpy
    os.makedirs(OUT, exist_ok=True)
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    with tempfile.TemporaryDirectory() as tmp:
        c_file = os.path.join(tmp, "_kernels.c")
        subprocess.check_call([sys.executable, "-m", "cython", "-3", "-I", SRC, "-o", c_file,
                               os.path.join(SRC, "_kernels.pyx")])
        so = os.path.join(OUT, "_kernels" + ext)
        subprocess.check_call(["gcc", "-O3", "-mf16c", "-shared", "-fPIC", "-o", so, c_file, "-I", SRC,
                               "-I", sysconfig.get_paths()["include"], "-I", numpy.get_include(),
                               "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION"])
    return so


def load():
    """Import the built reference kernels module (no /root/reference needed at run time)."""
    import importlib.util
    path = built_module()
    if path is None:
        raise ImportError("oracle/_ref/_kernels*.so not built (python oracle/build_ref.py)")
    spec = importlib.util.spec_from_file_location("_kernels", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
