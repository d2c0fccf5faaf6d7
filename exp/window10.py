"""Late-state K1 after idle pauses of increasing length (power-management probe)."""
import sys, time
sys.path.insert(0, ".")
import bench
import torch
from paper_2602_22421_b200 import Params, Solver

inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
s.step(1500)
torch.cuda.synchronize()
k1, _ = s.step_timed(50)
print(f"back-to-back: K1 {k1 / 50:.4f} ms", flush=True)
for pause in (0.005, 0.05, 0.5, 2.0):
    ks = []
    for _ in range(5):
        time.sleep(pause)
        k1, _ = s.step_timed(1)
        ks.append(k1)
    print(f"after {pause * 1e3:6.0f} ms idle: K1 {sum(ks) / len(ks):.4f} ms (min {min(ks):.4f})", flush=True)
