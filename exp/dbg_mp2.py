import numpy as np, sys
sys.path.insert(0, '.')
from spfom_inputs import generate
from paper_2602_22421_b200 import Solver, Params
for (m, T) in [(8, 2), (8, 1), (16, 2), (40, 3)]:
    inst = generate("multi", m=m, N=30, k=(3, 12), T=T) if T > 1 else generate("multi", m=m, N=30, k=(3, 12), T=2)
    a = Solver(inst, Params.converge())
    b = Solver(inst, Params.converge(), shared_periods=False)
    a.step(1); b.step(1)
    ya, y0a = a.primal(); yb, y0b = b.primal()
    ra = a.residuals()
    print(m, T, "periods", a.periods, "ydiff", np.abs(ya - yb).max(), "y0diff", np.abs(y0a - y0b).max(),
          "y0a==lam", np.mean(np.isclose(y0a, inst.arrival)), "passes", ra["newton_passes"], "fail", ra["newton_failures"])
    print("  y0a", np.round(y0a[:10], 3)); print("  y0b", np.round(y0b[:10], 3))
