"""CPU oracle for SPFOM's per-iteration update (GAM SBLP) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with the CUDA path
(paper_2602_22421_b200/) and never imports it.

* spfom_oracle.c  -- single-threaded fp64 C: projection, exact argmax,
  FAST-INNER, golden section, one SPFOM iteration, residuals, SBLP->CBLP
  policy recovery (see its header).
* lp.py           -- the SBLP / CBLP optimum: textbook dense simplex (Bland)
  and scipy HiGHS (library primitive), plus assortment enumeration.

Parity status per function is listed in DESIGN.md ("Oracle and pins"); every
function here is pinned by tests in tests/test_oracle_*.py.
"""
from .core import (  # noqa: F401
    OracleSolver,
    argmax,
    build_oracle,
    compute_R,
    dual_step,
    fast_inner,
    golden,
    lib,
    policy_probabilities,
    project,
    recover,
    residual_names,
)
