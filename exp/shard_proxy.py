"""8-GPU budget proxy on one GPU: rank 0's shard of the P-way nnz partition of
huge (segments [0, m/P)), all N products, run with world == 1 through the
NCCL code path (k_fold, ReduceScatter / AllGather with one rank) and without
it.  Per-iteration K1 and rest-of-step device times (CUDA event nodes)."""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, nccl_unique_id, partition
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
out = {}
for P in [int(x) for x in os.environ.get("PS", "1,2,4,8").split(",")]:
    b = partition(inst.seg_ptr, P)
    shard = inst.segment_slice(int(b[0]), int(b[1])) if P > 1 else inst
    for mode in ("single", "nccl"):
        kw = dict(rank=0, world=1, nccl_id=nccl_unique_id()) if mode == "nccl" else {}
        s = Solver(shard, Params.converge(), device="cuda:0", **kw)
        s.step(5)
        k1, tot = s.step_timed(40)
        s.close()
        out[f"P={P} {mode}"] = dict(segments=int(shard.m), nnz=int(shard.nnz), k1_us=round(k1 / 40 * 1e3, 2),
                                    step_us=round(tot / 40 * 1e3, 2), rest_us=round((tot - k1) / 40 * 1e3, 2))
        print(f"P={P} {mode}: {out[f'P={P} {mode}']}", flush=True)
print(json.dumps(out))
