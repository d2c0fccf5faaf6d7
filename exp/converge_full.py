"""Convergence of the converge preset at BASELINE full size (medium / huge /
multi): residuals every `every` iterations until the certificate gate
max(alpha, |D - P| / P) and infeas_rel are both below `stop`."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2602_22421_b200 import Params, Solver  # noqa: E402
from spfom_inputs import generate  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["medium", "huge", "multi"]
max_it = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
every = int(sys.argv[3]) if len(sys.argv) > 3 else 500
stop = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-7
for name in names:
    inst = generate(name)
    s = Solver(inst, Params.converge())
    t0 = time.time()
    it = 0
    while it < max_it:
        s.step(every)
        it += every
        r = s.residuals()
        P, D = r["primal_obj"], r["dual_obj"]
        gate = max(r["alpha"], abs(D - P) / abs(P))
        rec = dict(cfg=name, it=it, P=P, D=D, rel_gap=r["rel_gap"], infeas_rel=r["infeas_rel"], alpha=r["alpha"],
                   gate=gate, passes=r["newton_passes"], fail=r["newton_failures"], wall=round(time.time() - t0, 2))
        print(json.dumps(rec), flush=True)
        if gate <= stop and r["infeas_rel"] <= stop:
            break
    s.close()
