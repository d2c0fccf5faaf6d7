import numpy as np, sys
sys.path.insert(0, '.')
from spfom_inputs import generate
from paper_2602_22421_b200 import Solver, Params
import oracle
inst = generate("multi", m=40, N=30, k=(3, 12), T=2)
print("m", inst.m, "nnz", inst.nnz, inst.meta.get("T"), inst.meta.get("m_per_period"))
a = Solver(inst, Params.converge())
b = Solver(inst, Params.converge(), shared_periods=False)
print("info a", a.info())
for it in range(2):
    a.step(1); b.step(1)
    ya, y0a = a.primal(); yb, y0b = b.primal()
    print("iter", it + 1, "y diff", np.abs(ya - yb).max(), "y0 diff", np.abs(y0a - y0b).max(),
          "s diff", np.abs(a.usage() - b.usage()).max(), "eta diff", np.abs(a.duals() - b.duals()).max())
    print(" ya[:12]", np.round(ya[:12], 4)); print(" yb[:12]", np.round(yb[:12], 4))
    print(" y0a[:6]", np.round(y0a[:6], 4), "y0b", np.round(y0b[:6], 4))
    print(" sa", np.round(a.usage()[:8], 4), "sb", np.round(b.usage()[:8], 4))
