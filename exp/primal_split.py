"""Where primal() goes (huge): fresh output arrays (page faults on first touch)
vs pre-faulted ones, and a plain 400 MB first-touch memset for scale."""
import ctypes as C, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2602_22421_b200 import Params, Solver, load_library
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
s.step(20)
L = load_library()
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); y, y0 = s.primal(); t1 = time.perf_counter()
    yy, yy0 = np.empty(s.nnz), np.empty(s.m); yy.fill(0.0); yy0.fill(0.0)
    t2 = time.perf_counter(); L.spfom_primal(s._h, yy.ctypes.data, yy0.ctypes.data); t3 = time.perf_counter()
    z = np.empty(s.nnz); t4 = time.perf_counter(); z.fill(1.0); t5 = time.perf_counter()
    print(f"primal fresh {1e3*(t1-t0):.1f} ms | into pre-faulted arrays {1e3*(t3-t2):.1f} ms | first-touch fill of {s.nnz*8/1e6:.0f} MB {1e3*(t5-t4):.1f} ms", flush=True)
