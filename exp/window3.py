"""Per window: K1 time, Newton passes per segment-iteration and the number of
segment-iterations with more than SPFOM_DIAG_LONG passes (diagnostic build:
reported in newton_restarts)."""
import sys
sys.path.insert(0, ".")
import bench
from paper_2602_22421_b200 import Params, Solver

inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
win, total = int(sys.argv[1]), int(sys.argv[2])
prev = s.residuals()
while s.iteration < total:
    k1, tot = s.step_timed(win)
    r = s.residuals()
    dp = r["newton_passes"] - prev["newton_passes"]
    dl = r["newton_restarts"] - prev["newton_restarts"]
    print(f"iter {s.iteration:5d}  K1 {k1 / win:.4f} ms  passes/seg {dp / (win * s.m):.3f}  long/iter {dl / win:9.1f}  gap {r['rel_gap']:.2e}", flush=True)
    prev = r
