"""Newton passes per segment for each of the first iterations (huge)."""
import os, sys
sys.path.insert(0, ".")
import bench
from paper_2602_22421_b200 import Params, Solver
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
prev = 0
out = []
for t in range(1, 61):
    s.step(1)
    p = s.residuals()["newton_passes"]
    out.append(round((p - prev) / inst.m, 3))
    prev = p
print(out)
