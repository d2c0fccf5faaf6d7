"""Per-entry K1 cost of sampled blocks (B = m / FRAC) vs the full sweep, full
BASELINE sizes, paper preset (theta = inf) and converge preset; one JSON line
per (config, preset, B).  ps/nnz = K1 time / entries of the iteration's rows
(mean over the block rows used).  SPFOM_LIB selects the library."""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver
from spfom_inputs import block_sequence

n = int(os.environ.get("N", "64"))
for cfg in os.environ.get("CFGS", "huge,medium").split(","):
    inst = bench.load_instance(cfg, "/tmp/spfom_cache")
    k = np.diff(inst.seg_ptr)
    for preset in ("paper", "converge"):
        for frac in [int(x) for x in os.environ.get("FRACS", "1,8").split(",")]:
            B = inst.m // frac
            blocks = None if frac == 1 else block_sequence(inst.m, B, 16, 11)
            ent = float(inst.nnz) if blocks is None else float(np.mean([k[r].sum() for r in blocks]))
            p = Params.paper(blocks=blocks, exec_mode=1) if preset == "paper" else Params.converge(blocks=blocks, exec_mode=1)
            s = Solver(inst, p)
            s.step(16)
            k1, tot = s.step_timed(n)
            s.close()
            print(json.dumps(dict(config=cfg, preset=preset, B=B, entries=ent, k1_us=round(k1 / n * 1e3, 2),
                                  step_us=round(tot / n * 1e3, 2), ps_per_nnz=round(k1 / n * 1e9 / ent, 2),
                                  lib=os.path.basename(os.environ.get("SPFOM_LIB", "libspfom.so")))), flush=True)
