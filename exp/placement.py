"""Workspace placement vs K1 time: one large device buffer, the
solver's workspace carved out of it at a series of offsets; K1 over iterations
5..55 per offset (fresh solver each time, same instance)."""
import os, sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2602_22421_b200 import Params, Solver
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
free, _ = torch.cuda.mem_get_info()
probe = Solver(inst, Params.converge(), device="cuda:0")
need = probe.workspace_bytes + 512
probe.close()
del probe
torch.cuda.empty_cache()
GiB = 1 << 30
span = int(os.environ.get("SPAN_GIB", "96"))
pool = torch.empty(span * GiB + need, dtype=torch.uint8, device="cuda:0")
print(f"pool at {pool.data_ptr():#x}, workspace {need / GiB:.2f} GiB", flush=True)
offs = [float(x) for x in os.environ.get("OFFS", "0,0.5,1,2,3,4,6,8,12,16,24,32,48,64,80,96").split(",")]
for o in offs:
    b = int(o * GiB)
    if b + need > pool.numel():
        continue
    ws = pool[b:b + need]
    s = Solver(inst, Params.converge(), device="cuda:0", workspace=ws)
    s.step(5)
    k1, tot = s.step_timed(50)
    s.close()
    print(f"offset {o:6.2f} GiB (addr {ws.data_ptr():#x}): K1 {k1 / 50:.4f} ms  step {tot / 50:.4f} ms", flush=True)
