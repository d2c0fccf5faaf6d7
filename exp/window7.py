"""Diagnostic build: per-warp K1 duration vs Newton loop trips of that warp in
the same launch, late in the run."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, load_library

inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
L = load_library()
tb = np.zeros(2 * 148 * 8, dtype=np.uint64)
l0 = np.zeros(148 * 16, dtype=np.uint32)
l1 = np.zeros(148 * 16, dtype=np.uint32)
for target in [100, 1000]:
    s.step(target - s.iteration)
    L.spfom_diag_loops(l0.ctypes.data_as(C.c_void_p), C.c_int(l0.size))
    k1, _ = s.step_timed(1)
    L.spfom_diag_time(tb.ctypes.data_as(C.c_void_p), C.c_int(tb.size))
    L.spfom_diag_loops(l1.ctypes.data_as(C.c_void_p), C.c_int(l1.size))
    t = tb.reshape(-1, 2).astype(np.int64)
    dur = (t[:, 1] - t[:, 0]) / 1e3
    loops = (l1 - l0)[:148 * 8].astype(np.int64)
    print(f"iter {s.iteration}: K1 {k1:.4f} ms; warp dur med {np.median(dur):.1f} max {dur.max():.1f}; loops/warp med {np.median(loops)} max {loops.max()} min {loops.min()}; corr {np.corrcoef(dur, loops)[0,1]:.3f}")
    o = np.argsort(dur)
    print("  fastest:", [(round(dur[i], 1), int(loops[i]), int(i)) for i in o[:4]])
    print("  slowest:", [(round(dur[i], 1), int(loops[i]), int(i)) for i in o[-6:]])
    slow = dur > np.median(dur) * 1.15
    print("  slow warps:", int(slow.sum()), "warp-in-block histogram", np.bincount(np.arange(148 * 8)[slow] % 8, minlength=8).tolist(),
          "blocks", sorted(set((np.arange(148 * 8)[slow] // 8).tolist()))[:40])
