"""Memory-safety evidence on the GPU (-m gpu).  compute-sanitizer is closed on
this GPU pool (runs under it have left GPUs needing a reset), so the sanitizer
tier of SURVEY §4 is replaced by (1) guard regions around a caller-provided
workspace and (2) a build with index / size checks inside the kernels."""
import os
import subprocess
import sys

import numpy as np
import pytest

from spfom_inputs import block_sequence, generate, with_bundles

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _params(**kw):
    from paper_2602_22421_b200 import Params
    return Params.converge(**kw)


CASES = [
    ("tiny", lambda: generate("tiny"), dict(exec_mode=2)),
    ("small-graph", lambda: generate("small", m=300, N=150, k=(5, 40)), dict(exec_mode=1)),
    ("ragged", lambda: generate("medium", m=4000, N=2000, k=(5, 1024)), dict()),
    ("entry-mapped", lambda: generate("huge", m=24005, N=3000, k=50), dict()),
    ("multi", lambda: generate("multi", m=300, N=200, k=(5, 60), T=3), dict()),
    ("bundles", lambda: with_bundles(generate("small", m=300, N=150, k=(5, 40)), L=40, seed=1), dict()),
    ("sampled", lambda: generate("medium", m=3000, N=1500, k=(20, 200)), dict(refresh_every=3)),
]


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_workspace_guard_regions(name, make, kw):
    """Every kernel writes only inside [aligned base, base + workspace_bytes):
    64 KiB guard regions before and after the workspace (and the alignment
    slack) keep their fill pattern through stepping, residuals, getters and
    recovery."""
    import torch
    from paper_2602_22421_b200 import Solver
    inst = make()
    if name == "sampled":
        kw = dict(kw, blocks=block_sequence(inst.m, 700, 8, 2))
    probe = Solver(inst, _params(**kw))
    need = probe.workspace_bytes + 512
    probe.close()
    G = 1 << 16
    buf = torch.full((need + 2 * G,), 0xA5, dtype=torch.uint8, device="cuda")
    s = Solver(inst, _params(**kw), workspace=buf[G:G + need])
    s.step(9)
    s.residuals()
    s.duals()
    s.primal()
    if name not in ("tiny", "bundles"):
        s.recover()
    base = buf[G:].data_ptr()
    aligned = (base + 255) & ~255
    lo = G + (aligned - base)                      # first byte the library owns
    hi = lo + s.workspace_bytes
    s.close()
    torch.cuda.synchronize()
    host = buf.cpu().numpy()
    assert np.all(host[:lo] == 0xA5), "write below the workspace"
    assert np.all(host[hi:] == 0xA5), "write past the workspace"


def test_device_checks_build():
    """libspfom_checked.so (SPFOM_DEVICE_CHECKS, built by __graft_entry__.build):
    every primal kernel family with its index / size checks on; a failed check
    would make a getter raise SPFOM_ENUMERIC and the script exit non-zero."""
    so = os.path.join(ROOT, "paper_2602_22421_b200", "libspfom_checked.so")
    assert os.path.exists(so), "run __graft_entry__.build()"
    env = dict(os.environ, SPFOM_LIB=so)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "progs", "checks_run.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "checks_run ok" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
