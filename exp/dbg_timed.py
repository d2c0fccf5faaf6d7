import sys
sys.path.insert(0, ".")
import bench
from paper_2602_22421_b200 import Params, Solver
inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
for target in [5, 1500]:
    s.step(target - s.iteration)
    s.residuals()
    for n in [20, 100]:
        try:
            k1, tot = s.step_timed(n)
            print(target, n, "ok", k1 / n, tot / n, flush=True)
        except Exception as e:
            print(target, n, "FAIL", e, flush=True)
