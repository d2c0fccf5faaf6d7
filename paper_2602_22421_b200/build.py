"""Build libspfom.so in-tree with nvcc for sm_100a (explicit -gencode)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libspfom.so")
SO_CHECKED = os.path.join(HERE, "libspfom_checked.so")   # SPFOM_DEVICE_CHECKS build (tests only)
SOURCES = [os.path.join(CSRC, "spfom.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("spfom_kernels.cuh", "spfom_primal.cuh", "spfom_common.cuh")] + [
    os.path.join(ROOT, "include", "spfom.h")]


def nvcc_cmd(out: str = SO, extra=()):
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-shared", "-Xcompiler", "-fPIC,-fopenmp", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"),
            "-o", out, *SOURCES, "-lgomp", "-ldl", *extra]


def _fresh(so: str) -> bool:
    return os.path.exists(so) and all(os.path.getmtime(so) >= os.path.getmtime(d) for d in DEPS)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """libspfom.so (the product); checked=True also builds libspfom_checked.so,
    the same sources with the device index / size checks on (tests only).
    The two nvcc runs go in parallel."""
    jobs = []
    if force or not _fresh(SO):
        jobs.append((SO, subprocess.Popen(nvcc_cmd(), stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    if checked and (force or not _fresh(SO_CHECKED)):
        cmd = nvcc_cmd(out=SO_CHECKED, extra=["-DSPFOM_DEVICE_CHECKS"])
        jobs.append((SO_CHECKED, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for so, proc in jobs:
        out, err = proc.communicate()
        if proc.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed building {os.path.basename(so)}")
        if so == SO:
            if verbose:
                sys.stderr.write(err)
            with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
                f.write(err)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
