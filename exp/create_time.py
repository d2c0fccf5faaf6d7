import os, sys, time
sys.path.insert(0, '.')
os.environ["SPFOM_TRACE_CREATE"] = "1"
import torch
from bench import load_instance
from paper_2602_22421_b200 import Solver, Params
inst = load_instance("huge", "/tmp/spfom_cache")
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter(); s = Solver(inst, Params.converge()); torch.cuda.synchronize(); t1 = time.perf_counter()
    print("Solver()", round((t1 - t0) * 1e3, 1), "ms", file=sys.stderr)
    t0 = time.perf_counter(); y, y0 = s.primal(); eta = s.duals(); t1 = time.perf_counter()
    print("primal+duals", round((t1 - t0) * 1e3, 1), "ms", file=sys.stderr)
    s.close()
