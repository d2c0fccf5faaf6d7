"""Lazy module loading: does a large allocation before the solver (shifting
the workspace's placement) change K1?  PAD_MB env: MB allocated first."""
import os, sys
sys.path.insert(0, ".")
import bench
import torch
from paper_2602_22421_b200 import Params, Solver

pad = torch.empty(int(os.environ.get("PAD_MB", "0")) << 20, dtype=torch.uint8, device="cuda:0")
inst = bench.load_instance("huge", "/tmp/spfom_cache")
s = Solver(inst, Params.converge(), device="cuda:0")
print("workspace", hex(s.workspace.data_ptr()), flush=True)
s.step(1200)
k1, _ = s.step_timed(200)
print(f"PAD {os.environ.get('PAD_MB', '0')} MB, {os.environ.get('CUDA_MODULE_LOADING')}: K1 {k1 / 200:.4f} ms", flush=True)
