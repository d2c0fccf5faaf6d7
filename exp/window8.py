"""Diagnostic build (static split: -DSPFOM_DYN_CH=0): per warp, duration,
mbarrier wait and scatter time, SM id; slow vs fast warps late in the run."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, load_library

inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
L = load_library()
tb = np.zeros(2 * 148 * 8, dtype=np.uint64)
lb = np.zeros(4 * 148 * 16, dtype=np.uint32)
for target in [100, 1000]:
    s.step(target - s.iteration)
    k1, _ = s.step_timed(1)
    L.spfom_diag_time(tb.ctypes.data_as(C.c_void_p), C.c_int(tb.size))
    L.spfom_diag_loops(lb.ctypes.data_as(C.c_void_p), C.c_int(lb.size))
    t = tb.reshape(-1, 2).astype(np.int64)
    dur = (t[:, 1] - t[:, 0]) / 1e3
    x = lb.reshape(-1, 4)[:148 * 8].astype(np.int64)
    wait_us, red_us, smid = x[:, 0] * 1024 / 1965.0, x[:, 1] * 1024 / 1965.0, x[:, 2]
    slow = dur > np.median(dur) * 1.15
    print(f"iter {s.iteration}: K1 {k1:.4f} ms, warp dur med {np.median(dur):.1f} us; slow warps {int(slow.sum())}")
    for name, m in (("slow", slow), ("fast", ~slow)):
        if m.sum():
            print(f"  {name}: dur {dur[m].mean():.1f} us, mbar wait {wait_us[m].mean():.1f} us, scatter {red_us[m].mean():.1f} us, "
                  f"smid range {smid[m].min()}-{smid[m].max()} (mean {smid[m].mean():.1f})")
    sm_slow = np.zeros(148); np.add.at(sm_slow, smid, slow.astype(float))
    print("  slow fraction by smid/8 group:", np.round(np.add.reduceat(sm_slow, np.arange(0, 148, 8)) / np.add.reduceat(np.bincount(smid, minlength=148).astype(float), np.arange(0, 148, 8)), 2).tolist())
