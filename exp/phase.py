"""Per-phase cycles of a K1 stream round (diagnostic build -DSPFOM_DIAG_PHASE).
FRAC > 1: sampled blocks B = m / FRAC; PRESET = converge | paper; ITERS = windows."""
import ctypes as C, sys, os
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, load_library
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
frac = int(os.environ.get("FRAC", "1"))
from spfom_inputs import block_sequence
blocks = None if frac == 1 else block_sequence(inst.m, inst.m // frac, 16, 11)
mk = Params.paper if os.environ.get("PRESET", "converge") == "paper" else Params.converge
s = Solver(inst, mk(blocks=blocks, exec_mode=1), device="cuda:0")
L = load_library()
buf = np.zeros(10, dtype=np.uint64)
names = ["mbar wait", "slot read+gather", "projection", "write-back", "head hists", "global REDs", "rounds", "loop/claim", "TMA issue", "-"]
for target in [int(x) for x in os.environ.get("ITERS", "5,1500").split(",")]:
    s.step(target - s.iteration)
    L.spfom_diag_phase(buf.ctypes.data_as(C.c_void_p), C.c_int(1))
    k1, _ = s.step_timed(20)
    L.spfom_diag_phase(buf.ctypes.data_as(C.c_void_p), C.c_int(1))
    rounds = float(buf[6])
    print(f"iter {target}: K1 {k1/20:.4f} ms, rounds {rounds/20:.0f}/launch; cycles per warp-round:")
    tot = sum(float(buf[k]) for k in range(10) if k != 6)
    print(f"   scatter warps busy per handed-over round: {float(buf[9]) / max(rounds, 1):8.0f}")
    for k in range(10):
        if k not in (6, 9):
            print(f"   {names[k]:18s} {float(buf[k]) / rounds:8.0f}  ({100 * float(buf[k]) / tot:4.1f}%)")
