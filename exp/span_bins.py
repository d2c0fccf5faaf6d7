"""Per-bin timeline of one full-sweep K1 step (-DSPFOM_DIAG_SPAN): blocks are
indexed by SM and tagged with their bin (G * 10000 + Q * 100 + EQ), so the
concurrent bin launches of medium show each share's start, setup, loop end
and exit.  CFG=medium (default), IT = iteration to sample at (default 20)."""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2602_22421_b200 import Params, Solver, load_library
cfg = os.environ.get("CFG", "medium")
inst = bench.load_instance(cfg, "/tmp/spfom_cache")
L = load_library()
buf = np.zeros(4 * 160 + 80, dtype=np.uint64)
s = Solver(inst, Params.converge(), device="cuda:0")
s.step(int(os.environ.get("IT", "20")))
rows = {}
for rep in range(7):
    torch.cuda.synchronize()
    L.spfom_diag_span(buf.ctypes.data_as(C.c_void_p), C.c_int(1))
    k1, _ = s.step_timed(1)
    torch.cuda.synchronize()
    L.spfom_diag_span(buf.ctypes.data_as(C.c_void_p), C.c_int(0))
    sp = buf[:640].reshape(-1, 4)[:148].astype(np.int64)
    key = buf[640:].view(np.uint32)[:148]
    t0 = sp[:, 0][sp[:, 0] > 0].min()
    sp = (sp - t0) / 1e3
    for k in np.unique(key):
        m = key == k
        r = (m.sum(), np.median(sp[m, 0]), np.median(sp[m, 1]), np.median(sp[m, 2]), sp[m, 2].max(), sp[m, 3].max())
        rows.setdefault(int(k), []).append(r)
    rows.setdefault(-1, []).append((k1 * 1e3,) * 6)
for k, v in sorted(rows.items()):
    r = np.median(np.array(v), axis=0)
    if k < 0:
        print(f"K1 event {r[0]:.1f} us")
    else:
        print(f"bin key {k}: {int(r[0])} SMs | start {r[1]:.1f} | setup end {r[2]:.1f} | loop end median {r[3]:.1f} max {r[4]:.1f} | exit max {r[5]:.1f} us", flush=True)
