"""Parity helpers: the CUDA path (through the C ABI) vs the CPU oracle."""
from __future__ import annotations

import numpy as np

TOL_ITER = 1e-10      # north_star: per-iterate rel-inf agreement, first 100 iterations


def rel_inf(a, b, scale: float) -> float:
    """||a - b||_inf / ||b||_inf (reading c13); when b == 0 the error is
    measured against `scale` (max lambda for y, max r for eta)."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    nb = float(np.abs(b).max()) if b.size else 0.0
    d = float(np.abs(a - b).max()) if b.size else 0.0
    return d / nb if nb > 0 else d / scale


def oracle_kwargs(p) -> dict:
    return dict(theta=p.theta, tau=p.tau, tau_mode=p.tau_mode, mu=p.mu, extrapolation=p.extrapolation,
                averaging=p.averaging, refresh_every=p.refresh_every)


def lockstep(inst, params, iters: int, blocks=None, check_every: int = 1, tie_margin=None, check_first: int = 0,
             gpu=None):
    """Run GPU and oracle side by side; return the worst per-iteration errors
    (y, y0, eta) over iterations 1..iters.  Checked after every iteration t with
    t <= check_first, t % check_every == 0, and the last one.  `gpu`: an
    already created Solver for `inst` (at iteration 0)."""
    import oracle
    from paper_2602_22421_b200 import Solver

    gpu = gpu if gpu is not None else Solver(inst, params)
    cpu = oracle.OracleSolver(inst, **oracle_kwargs(params))
    ys = 1.0
    lams = float(inst.arrival.max()) if inst.arrival.size else 1.0     # m = 0: nothing to scale
    rs = float(inst.price.max())
    worst = dict(y=0.0, y0=0.0, eta=0.0, s=0.0)
    for t in range(iters):
        gpu.step(1)
        cpu.step(None if blocks is None else blocks[t % blocks.shape[0]])
        if (t + 1) % check_every == 0 or t + 1 == iters or t + 1 <= check_first:
            y, y0 = gpu.primal()
            eta = gpu.duals()
            s = gpu.usage()
            e = dict(y=rel_inf(y, cpu.y, lams), y0=rel_inf(y0, cpu.y0, lams), eta=rel_inf(eta, cpu.eta, rs),
                     s=rel_inf(s, cpu.s, lams))
            for k in e:
                worst[k] = max(worst[k], e[k])
            worst["checks"] = worst.get("checks", 0) + 1
            if max(e.values()) > TOL_ITER:
                worst["first_bad_iter"] = t + 1
                break
    return worst, gpu, cpu
