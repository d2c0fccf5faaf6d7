"""Per-entry K1 cost of sampled blocks (B = m / FRAC) vs the full sweep, full
BASELINE sizes, paper preset (theta = inf) and converge preset; one JSON line
per (config, preset, B).  ps/nnz = K1 time / entries of the iteration's rows
(mean over the block rows used); passes = Newton passes per updated segment
(converge preset).  A sampled run that starts at iteration S0 and times n
iterations updates each segment ~S0/FRAC .. (S0+n)/FRAC times, i.e. it sits in
the Newton transient of a full sweep at those iterations: `matched_full` is the
full sweep timed over that window (same warm-start age), the fair comparison.
SPFOM_LIB selects the library."""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver
from spfom_inputs import block_sequence

n = int(os.environ.get("N", "64"))
S0 = int(os.environ.get("S0", "16"))


def run(inst, preset, blocks, start, iters):
    p = Params.paper(blocks=blocks, exec_mode=1) if preset == "paper" else Params.converge(blocks=blocks, exec_mode=1)
    s = Solver(inst, p)
    if start:
        s.step(start)
    r0 = s.residuals()
    k1, tot = s.step_timed(iters)
    r1 = s.residuals()
    s.close()
    return k1, tot, r1.get("newton_passes", 0) - r0.get("newton_passes", 0)


for cfg in os.environ.get("CFGS", "huge,medium").split(","):
    inst = bench.load_instance(cfg, "/tmp/spfom_cache")
    k = np.diff(inst.seg_ptr)
    for preset in ("paper", "converge"):
        for frac in [int(x) for x in os.environ.get("FRACS", "1,8").split(",")]:
            B = inst.m // frac
            blocks = None if frac == 1 else block_sequence(inst.m, B, 16, 11)
            ent = float(inst.nnz) if blocks is None else float(np.mean([k[r].sum() for r in blocks]))
            k1, tot, passes = run(inst, preset, blocks, S0, n)
            line = dict(config=cfg, preset=preset, B=B, entries=ent, k1_us=round(k1 / n * 1e3, 2),
                        step_us=round(tot / n * 1e3, 2), ps_per_nnz=round(k1 / n * 1e9 / ent, 2),
                        passes=round(passes / (n * B), 3) if preset == "converge" else None,
                        window=f"iterations {S0}..{S0 + n}",
                        lib=os.path.basename(os.environ.get("SPFOM_LIB", "libspfom.so")))
            if frac > 1:
                a, m_it = S0 // frac, max(4, n // frac)
                k1f, _, pf = run(inst, preset, None, a, m_it)
                line["matched_full"] = dict(window=f"full sweep, iterations {a}..{a + m_it}",
                                            ps_per_nnz=round(k1f / m_it * 1e9 / inst.nnz, 2),
                                            passes=round(pf / (m_it * inst.m), 3) if preset == "converge" else None)
                line["ratio_vs_matched"] = round(line["ps_per_nnz"] / line["matched_full"]["ps_per_nnz"], 3)
            print(json.dumps(line), flush=True)
