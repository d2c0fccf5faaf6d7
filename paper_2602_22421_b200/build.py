"""Build libspfom.so in-tree with nvcc for sm_100a (explicit -gencode)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libspfom.so")
SOURCES = [os.path.join(CSRC, "spfom.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("spfom_kernels.cuh", "spfom_primal.cuh", "spfom_common.cuh")] + [
    os.path.join(ROOT, "include", "spfom.h")]


def nvcc_cmd(out: str = SO, extra=()):
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-shared", "-Xcompiler", "-fPIC,-fopenmp", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"),
            "-o", out, *SOURCES, "-lgomp", "-ldl", *extra]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO) and all(os.path.getmtime(SO) >= os.path.getmtime(d) for d in DEPS):
        return SO
    res = subprocess.run(nvcc_cmd(), capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libspfom.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
        f.write(res.stderr)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
