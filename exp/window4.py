"""Late-state K1: graph replay vs un-graphed launches vs a fresh handle loaded
with the same state (set_state)."""
import sys
sys.path.insert(0, ".")
import bench
import torch
from paper_2602_22421_b200 import Params, Solver

inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
s.step(800)
k1, tot = s.step_timed(20)
print(f"graph, iter {s.iteration}: K1 {k1/20:.4f} ms", flush=True)
a, b = s.time_kernels(20)
print(f"ungraphed: primal {a/20:.4f} ms rest {b/20:.4f}", flush=True)
y, y0 = s.primal()
eta = s.duals()
t = s.usage()
s2 = Solver(inst, Params.converge(), device="cuda:0")
s2.set_state(y=y, y0=y0, eta=eta)
k1, tot = s2.step_timed(20)
print(f"fresh handle + set_state: K1 {k1/20:.4f} ms", flush=True)
k1, tot = s2.step_timed(200)
print(f"fresh handle +200: K1 {k1/200:.4f} ms", flush=True)
