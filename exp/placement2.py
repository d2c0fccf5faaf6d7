"""K1 vs the size of the allocation the workspace is carved from (huge)."""
import os, sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2602_22421_b200 import Params, Solver
inst = bench.load_instance(os.environ.get("CFG", "huge"), "/tmp/spfom_cache")
GiB = 1 << 30
def run(ws=None, label=""):
    s = Solver(inst, Params.converge(), device="cuda:0", workspace=ws)
    s.step(5)
    k1, tot = s.step_timed(50)
    need = s.workspace_bytes
    s.close()
    print(f"{label:40s} K1 {k1 / 50:.4f} ms  step {tot / 50:.4f} ms", flush=True)
    return need
need = run(label="default (torch.empty of the workspace)") + 512
for rep in range(2):
    for extra in [0, 1, 2, 4, 8, 16, 32, 64]:
        torch.cuda.empty_cache()
        pool = torch.empty(need + extra * GiB, dtype=torch.uint8, device="cuda:0")
        run(pool[:need], f"pool of workspace + {extra} GiB, offset 0")
        del pool
    torch.cuda.empty_cache()
    run(label="default again")
