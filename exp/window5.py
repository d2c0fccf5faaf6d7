"""Is K1 speed tied to the workspace placement?  Several handles of the same
instance, each warmed to the steady state, timed in turn; workspace base
addresses printed (mod 2 MB / 1 GB)."""
import sys
sys.path.insert(0, ".")
import bench
import torch
from paper_2602_22421_b200 import Params, Solver

inst = bench.load_instance("huge", "/tmp/spfom_cache")
hs = []
for k in range(3):
    if k == 1:
        pad = torch.empty(int(sys.argv[1]) if len(sys.argv) > 1 else (64 << 20), dtype=torch.uint8, device="cuda:0")
    s = Solver(inst, Params.converge(), device="cuda:0")
    hs.append(s)
    b = s.workspace.data_ptr()
    print(f"handle {k}: workspace 0x{b:x}  mod 2MB {b % (2 << 20)}  mod 1GB {b % (1 << 30)}  bytes {s.workspace_bytes}", flush=True)
for rep in range(2):
    for k, s in enumerate(hs):
        s.step(300 if rep == 0 else 0)
        k1, _ = s.step_timed(50)
        print(f"rep {rep} handle {k}: iter {s.iteration} K1 {k1 / 50:.4f} ms", flush=True)
