"""Warp-level Newton loop trips per warp round vs segment-level passes (K1
stream kernel, huge): the warp runs FULL / CHECK passes until its slowest
group converges.  Needs a -DSPFOM_DIAG_TIME build (SPFOM_LIB)."""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, load_library

inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
L = load_library()
n = 4 * 148 * 16
for target in [int(x) for x in os.environ.get("ITERS", "5,25,100,1500").split(",")]:
    s.step(target - s.iteration)
    a = np.zeros(n, dtype=np.uint32)
    b = np.zeros(n, dtype=np.uint32)
    L.spfom_diag_loops(a.ctypes.data_as(C.c_void_p), C.c_int(n))
    r0 = s.residuals()
    s.step(1)
    r1 = s.residuals()
    L.spfom_diag_loops(b.ctypes.data_as(C.c_void_p), C.c_int(n))
    trips = int((b.reshape(-1, 4)[:, 3].astype(np.int64) - a.reshape(-1, 4)[:, 3].astype(np.int64)).sum())
    rounds = (inst.m + 7) // 8
    seg = (r1["newton_passes"] - r0["newton_passes"]) / inst.m
    print(f"iteration {target}: segment passes {seg:.3f}, warp trips per round {trips / rounds:.3f}", flush=True)
