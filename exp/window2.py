"""Is the late-iteration K1 slowdown state- or context-dependent?  After N
iterations, time single iterations (a) back to back, (b) after a pause,
(c) after an L2 flush (memset of 512 MB)."""
import sys, time
sys.path.insert(0, ".")
import bench
import torch
from paper_2602_22421_b200 import Params, Solver

inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
for n in [int(a) for a in sys.argv[1:]] or [0, 300, 1000]:
    if n > s.iteration:
        s.step(n - s.iteration)
    torch.cuda.synchronize()
    k1, tot = s.step_timed(20)
    a = k1 / 20
    p = []
    for _ in range(10):
        torch.cuda.synchronize(); time.sleep(0.05)
        k1, _ = s.step_timed(1); p.append(k1)
    f = []
    for _ in range(10):
        junk.fill_(1); torch.cuda.synchronize()
        k1, _ = s.step_timed(1); f.append(k1)
    print(f"iter {s.iteration:5d}: back-to-back {a:.4f} ms | after pause {sum(p)/len(p):.4f} | after L2 flush {sum(f)/len(f):.4f}", flush=True)
