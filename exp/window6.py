"""Per-warp start/end of one K1 launch (diagnostic build, %globaltimer):
straggler warps / SMs early vs late in the run."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, load_library

import os
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
L = load_library()
buf = np.zeros(2 * 148 * 8, dtype=np.uint64)
for target in [50, 150, 300, 500, 800, 1200]:
    s.step(target - s.iteration)
    k1, _ = s.step_timed(1)
    assert L.spfom_diag_time(buf.ctypes.data_as(C.c_void_p), C.c_int(buf.size)) == 0
    t = buf.reshape(-1, 2).astype(np.int64)
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    dur = en - st
    per_sm = en.reshape(148, 8).max(1)
    print(f"iter {s.iteration:5d} K1(event) {k1:.4f} ms | warp end: min {en.min():.1f} med {np.median(en):.1f} p90 {np.percentile(en,90):.1f} max {en.max():.1f} us"
          f" | start spread {st.max():.1f} us | slowest SMs {np.argsort(per_sm)[-4:].tolist()} fastest {np.argsort(per_sm)[:3].tolist()}", flush=True)
y, y0 = s.primal()
tiny = (y != 0) & (np.abs(y) < 2.2250738585072014e-308)
print("y: nnz", y.size, "zeros", int((y == 0).sum()), "subnormal", int(tiny.sum()), "min |y|>0", float(np.abs(y[y != 0]).min()))
print("y0 subnormal", int(((y0 != 0) & (np.abs(y0) < 2.2250738585072014e-308)).sum()))
# slow warps vs their segment ranges (one bin, contiguous, original order; GPW = 8 segments per round)
m = inst.m
rounds = (m + 7) // 8
W = 148 * 8
seg_of_warp = [(rounds * w // W * 8, rounds * (w + 1) // W * 8) for w in range(W)]
row_tiny = np.add.reduceat(tiny.astype(np.int64), inst.seg_ptr[:-1])
per_w = np.array([row_tiny[a:min(b, m)].sum() for a, b in seg_of_warp])
dur = (buf.reshape(-1, 2)[:, 1].astype(np.int64) - buf.reshape(-1, 2)[:, 0].astype(np.int64)) / 1e3
order = np.argsort(dur)
print("fastest warps: dur", np.round(dur[order[:5]], 1).tolist(), "subnormal entries", per_w[order[:5]].tolist())
print("slowest warps: dur", np.round(dur[order[-5:]], 1).tolist(), "subnormal entries", per_w[order[-5:]].tolist())
print("corr(dur, subnormals)", float(np.corrcoef(dur, per_w)[0, 1]) if per_w.std() > 0 else None)
