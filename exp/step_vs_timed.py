"""spfom_step(K) (events only around the K iterations) vs spfom_step_timed(K)."""
import sys, os
sys.path.insert(0, ".")
import torch
import bench
from paper_2602_22421_b200 import Params, Solver
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
K = 40
s.step(10)
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s.stream)
    s.step(K)
    e1.record(s.stream)
    torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / K
    k1, tot = s.step_timed(K)
    print(f"step: {plain:.4f} ms/it   step_timed: {tot / K:.4f} ms/it (K1 {k1 / K:.4f}, rest {(tot - k1) / K * 1000:.1f} us)")
