"""Small SPFOM runs that exercise every primal kernel family -- the CUDA-graph
path and the persistent small-regime kernel on tiny / small, the entry-mapped
k = 50 bin, ragged length bins, shared-structure periods, bundles, sampled
blocks -- plus residuals, getters and recovery.  tests/test_gpu_checks.py runs
it under the SPFOM_DEVICE_CHECKS build (index / size checks in the kernels; a
failed check makes the getters raise SPFOM_ENUMERIC)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2602_22421_b200 import Params, Solver  # noqa: E402
from spfom_inputs import block_sequence, generate  # noqa: E402

cases = [("tiny", {}, Params.converge(exec_mode=1)),
         ("tiny", {}, Params.converge(exec_mode=2)),
         ("small", dict(m=300, N=150, k=(5, 40)), Params.converge(exec_mode=1)),
         ("small", dict(m=300, N=150, k=(5, 40)), Params.converge(exec_mode=2)),
         ("huge", dict(m=3000, N=800, k=50), Params.converge(exec_mode=1)),
         ("medium", dict(m=600, N=400, k=(20, 200)), Params.converge(exec_mode=1)),
         ("medium", dict(m=4000, N=2000, k=(5, 1024)), Params.converge(exec_mode=1)),
         ("multi", dict(m=300, N=200, k=(5, 60), T=3), Params.converge(exec_mode=1)),
         ("huge", dict(m=24005, N=30000, k=(33, 52)), Params.paper(mu=0.2, exec_mode=1))]
for name, kw, p in cases:
    inst = generate(name, **kw)
    s = Solver(inst, p)
    s.step(6)
    s.residuals()
    s.duals()
    s.primal()
    if name != "tiny":
        s.recover()
    s.close()
inst = generate("small", m=300, N=150, k=(5, 40))
s = Solver(inst, Params.paper(blocks=block_sequence(inst.m, 60, 8, 1), exec_mode=1))
s.step(5)
s.duals()
s.close()
inst = generate("medium", m=3000, N=1500, k=(20, 200))
s = Solver(inst, Params.converge(blocks=block_sequence(inst.m, 700, 8, 2), refresh_every=3))
s.step(7)
s.duals()
s.close()
from spfom_inputs import with_bundles  # noqa: E402
s = Solver(with_bundles(generate("small", m=300, N=150, k=(5, 40)), L=40, seed=1), Params.converge())
s.step(5)
s.duals()
s.residuals()
s.close()
print("checks_run ok")
