"""Fraction of y entries equal to 0 / unchanged between consecutive iterations (huge)."""
import sys, os
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
prev = None
for t in [5, 6, 10, 11, 20, 21, 100, 101, 500, 501, 2000, 2001]:
    s.step(t - s.iteration)
    y, _ = s.primal()
    if prev is not None and prev[0] == t - 1:
        print(f"t={t}: zero {np.mean(y == 0):.3f}  unchanged {np.mean(y == prev[1]):.3f}  zero->zero {np.mean((y == 0) & (prev[1] == 0)):.3f}", flush=True)
    prev = (t, y)
