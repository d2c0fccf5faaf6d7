"""Time-to-gap of the sampled regime vs the full sweep."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from spfom_inputs import generate, block_sequence
from paper_2602_22421_b200 import Solver, Params
name = sys.argv[1] if len(sys.argv) > 1 else "small"
inst = generate(name)
m = inst.m
for frac in [1, 2, 4, 8]:
    B = m // frac
    blocks = None if frac == 1 else block_sequence(m, B, 512, 11)
    for preset in (["converge"] if frac == 1 else ["converge", "converge-refresh"]):
        p = Params.converge(blocks=blocks, refresh_every=(64 if preset.endswith("refresh") else 0))
        s = Solver(inst, p)
        t_dev = 0.0
        hist = []
        it = 0
        chunk = 50 * frac
        for rep in range(200):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            s.step(chunk); torch.cuda.synchronize()
            t_dev += time.perf_counter() - t0
            it += chunk
            r = s.residuals()
            gap = max(abs(r["rel_gap"]), r["infeas_rel"])
            hist.append((it, t_dev, gap))
            if gap <= 1e-6: break
        def first(th):
            for (i, t, g) in hist:
                if g <= th: return dict(iters=i, seconds=round(t, 5))
            return None
        print(json.dumps(dict(config=name, B=B, preset=preset, small_mode=s.info().get("launches_per_iteration"),
                              ttg_1e3=first(1e-3), ttg_1e4=first(1e-4), ttg_1e6=first(1e-6), final_gap=hist[-1][2],
                              iters=hist[-1][0])))
        s.close()
