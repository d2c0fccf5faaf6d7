"""Writes tests/golden/lp_optima.json: SBLP optima P* of seeded instances,
computed ONLY through oracle/ (oracle.lp.sblp_highs, scipy HiGHS) -- never
from the CUDA path.  Re-run: python tests/golden/make_lp_optima.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from oracle import lp  # noqa: E402
from spfom_inputs import generate  # noqa: E402

CASES = {
    "small": dict(name="small"),
    "small-zipf-mini": dict(name="medium", m=3000, N=400, k=(20, 60)),
}

out = {}
for key, kw in CASES.items():
    kw = dict(kw)
    name = kw.pop("name")
    inst = generate(name, **kw)
    t = time.time()
    P, _y, _y0 = lp.sblp_highs(inst)
    out[key] = dict(config=name, overrides=kw, seed=inst.meta["seed"], nnz=inst.nnz, Pstar=P,
                    solver="scipy.optimize.linprog(method='highs'), U-auxiliary SBLP (oracle/lp.py)",
                    seconds=round(time.time() - t, 1))
    print(key, out[key], flush=True)
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "lp_optima.json"), "w"),
          indent=1)
