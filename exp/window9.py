"""Diagnostic build (static split): per block, late in the run: mean warp
duration and Newton loop trips per round."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, load_library

inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
L = load_library()
tb = np.zeros(2 * 148 * 8, dtype=np.uint64)
lb0 = np.zeros(4 * 148 * 16, dtype=np.uint32)
lb1 = np.zeros(4 * 148 * 16, dtype=np.uint32)
s.step(1000)
s.step_timed(1)
L.spfom_diag_loops(lb0.ctypes.data_as(C.c_void_p), C.c_int(lb0.size))
k1, _ = s.step_timed(1)
L.spfom_diag_time(tb.ctypes.data_as(C.c_void_p), C.c_int(tb.size))
L.spfom_diag_loops(lb1.ctypes.data_as(C.c_void_p), C.c_int(lb1.size))
t = tb.reshape(-1, 2).astype(np.int64)
dur = (t[:, 1] - t[:, 0]) / 1e3
trips = (lb1.reshape(-1, 4)[:148 * 8, 3].astype(np.int64) - lb0.reshape(-1, 4)[:148 * 8, 3].astype(np.int64))
rounds = (inst.m + 7) // 8
W = 148 * 8
rpw = np.array([rounds * (w + 1) // W - rounds * w // W for w in range(W)])
print(f"K1 {k1:.4f} ms; corr(dur, trips/round) = {np.corrcoef(dur, trips / rpw)[0, 1]:.3f}")
blk = dur.reshape(148, 8).mean(1)
tpr = (trips / rpw).reshape(148, 8).mean(1)
for b0 in range(0, 148, 12):
    print(" ".join(f"{blk[b]:5.0f}/{tpr[b]:.2f}" for b in range(b0, min(b0 + 12, 148))))
