"""Iterations/s of the sampled (block) regime through the public API."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from spfom_inputs import generate, block_sequence
from paper_2602_22421_b200 import Solver, Params
cases = [("small", None, "full"), ("small", 100, "converge"), ("small", 10, "paper"),
         ("huge", 1000, "paper"), ("huge", 100000, "converge")]
insts = {}
for name, B, preset in cases:
    inst = insts.get(name) or generate(name)
    insts[name] = inst
    blocks = None if B is None else block_sequence(inst.m, B, 64, 7)
    p = Params.converge(blocks=blocks) if preset != "paper" else Params.paper(blocks=blocks)
    s = Solver(inst, p)
    s.step(20)
    torch.cuda.synchronize()
    K = 2000 if name == "small" else 500
    pm, tot = s.step_timed(K)
    t0 = time.perf_counter(); s.step(K); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(json.dumps(dict(config=name, B=B, preset=preset, it_s_timed=K / tot * 1e3, primal_us=pm / K * 1e3,
                          rest_us=(tot - pm) / K * 1e3, it_s_graph=K / dt, launches=s.info()["launches_per_iteration"])))
    s.close()
