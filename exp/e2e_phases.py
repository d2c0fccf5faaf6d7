"""Where the e2e time goes (huge): Solver() create, K steps, duals(), primal()."""
import os, sys, time
sys.path.insert(0, ".")
import bench
import torch
from paper_2602_22421_b200 import Params, Solver

inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = Solver(inst, Params.converge(), device="cuda:0")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s.step(200)
    eta = s.duals()
    t2 = time.perf_counter()
    y, y0 = s.primal()
    t3 = time.perf_counter()
    s.close()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, 200 steps + duals {1e3*(t2-t1):.1f} ms, primal {1e3*(t3-t2):.1f} ms", flush=True)
