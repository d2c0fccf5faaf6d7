"""Medium, converge preset: a few iterations at B = m / FRAC (ncu launch list
of the per-bin K1 launches; run under ncu --metrics gpu__time_duration.sum)."""
import os, sys
sys.path.insert(0, ".")
import bench
from paper_2602_22421_b200 import Params, Solver
from spfom_inputs import block_sequence

inst = bench.load_instance(os.environ.get("CFG", "medium"), "/tmp/spfom_cache")
frac = int(os.environ.get("FRAC", "2"))
B = inst.m // frac
blocks = None if frac == 1 else block_sequence(inst.m, B, 16, 11)
s = Solver(inst, Params.converge(blocks=blocks, exec_mode=1))
s.step(int(os.environ.get("ITERS", "8")))
import numpy as np
k = np.diff(inst.seg_ptr)
print("bins info", s.info())
s.close()
