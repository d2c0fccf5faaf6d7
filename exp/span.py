"""Prologue / loop / epilogue of one K1 launch per block (-DSPFOM_DIAG_SPAN) on
rank 0's shard of a P-way partition of huge (PS env, default 1,8); FRAC > 1:
sampled blocks of m / FRAC rows."""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2602_22421_b200 import Params, Solver, load_library, partition
inst = bench.load_instance("huge", "/tmp/spfom_cache")
L = load_library()
buf = np.zeros(4 * 160 + 80, dtype=np.uint64)   # + the per-SM bin keys (uint32)
for P in [int(x) for x in os.environ.get("PS", "1,8").split(",")]:
    b = partition(inst.seg_ptr, P)
    shard = inst.segment_slice(int(b[0]), int(b[1])) if P > 1 else inst
    frac = int(os.environ.get("FRAC", "1"))      # > 1: sampled blocks B = m / FRAC of the shard
    from spfom_inputs import block_sequence
    blocks = None if frac == 1 else block_sequence(shard.m, shard.m // frac, 16, 11)
    s = Solver(shard, Params.converge(blocks=blocks, exec_mode=1), device="cuda:0")
    s.step(20)
    res = []
    for rep in range(5):
        torch.cuda.synchronize()
        L.spfom_diag_span(buf.ctypes.data_as(C.c_void_p), C.c_int(1))
        k1, _ = s.step_timed(1)
        torch.cuda.synchronize()
        L.spfom_diag_span(buf.ctypes.data_as(C.c_void_p), C.c_int(0))
        sp = buf[:640].reshape(-1, 4)[:148].astype(np.int64)
        t0 = sp[:, 0].min()
        sp = (sp - t0) / 1e3
        res.append((k1 * 1e3, np.median(sp[:, 0]), sp[:, 0].max(), np.median(sp[:, 1] - sp[:, 0]), np.median(sp[:, 2]), sp[:, 2].max(), np.median(sp[:, 3] - sp[:, 2]), sp[:, 3].max()))
    r = np.median(np.array(res), axis=0)
    print(f"P={P}: K1 event {r[0]:.1f} us | block start median {r[1]:.1f} max {r[2]:.1f} | setup {r[3]:.1f} | loop end median {r[4]:.1f} max {r[5]:.1f} | flush {r[6]:.1f} | last exit {r[7]:.1f} us", flush=True)
    s.close()
