"""K1 time per window of iterations over a long run (huge, converge preset),
with the SM clock / power sampled by nvidia-smi in between windows."""
import subprocess, sys, time
sys.path.insert(0, ".")
import bench  # noqa: E402  (instance cache helper)
import torch
from paper_2602_22421_b200 import Params, Solver

lib = None
import os
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
win, total = int(sys.argv[1]) if len(sys.argv) > 1 else 200, int(sys.argv[2]) if len(sys.argv) > 2 else 2000
done = 0
while done < total:
    p0 = s.info().get("newton_passes", 0)
    k1, tot = s.step_timed(win)
    done += win
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active",
                        "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"iters {done:5d}  K1 {k1 / win:.4f} ms  step {tot / win:.4f} ms  | {q}", flush=True)
