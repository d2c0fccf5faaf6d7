"""Independent pins for the oracle (test-only; no import of oracle internals).

* project_bruteforce -- the Euclidean projection onto Y_i by enumerating every
  active set of the QP's inequality rows (textbook KKT enumeration), written
  from the polytope definition (GAM reading c3) in the ORIGINAL
  variables (y0, y) -- it never uses the 3-scalar (nu, kappa, U) reduction the
  oracle is built on.
* kkt_certificate -- checks that a candidate point is THE projection by
  recovering the KKT multipliers with NNLS over the active rows and testing
  stationarity, primal feasibility and multiplier signs (sufficient for a
  convex QP); usable at any k.
"""
from __future__ import annotations

import itertools

import numpy as np
from scipy.optimize import nnls


def polytope_rows(v, w, v0):
    """Inequality rows G x >= 0 of Y_i in x = (y0, y_1..y_k):
    y_j >= 0  and  v_j (y0 + sum_k omega_k y_k) / vt0 - y_j >= 0."""
    v, w = np.asarray(v, float), np.asarray(w, float)
    k = v.shape[0]
    om = w / v
    vt0 = v0 + w.sum()
    G = []
    for j in range(k):
        g = np.zeros(k + 1)
        g[1 + j] = 1.0
        G.append(g)
    for j in range(k):
        g = np.zeros(k + 1)
        g[0] = v[j] / vt0
        g[1:] += v[j] * om / vt0
        g[1 + j] -= 1.0
        G.append(g)
    return np.array(G)


def project_bruteforce(z0, z, v, w, v0, lam):
    z = np.asarray(z, float)
    k = z.shape[0]
    G = polytope_rows(v, w, v0)
    zz = np.concatenate([[z0], z])
    best = None
    for pat in itertools.product(range(3), repeat=k):
        act = [j for j in range(k) if pat[j] == 1] + [k + j for j in range(k) if pat[j] == 2]
        E = np.vstack([np.ones(k + 1)] + [G[a] for a in act])
        b = np.zeros(E.shape[0])
        b[0] = lam
        n = k + 1
        M = np.zeros((n + E.shape[0], n + E.shape[0]))
        M[:n, :n] = np.eye(n)
        M[:n, n:] = -E.T
        M[n:, :n] = E
        try:
            sol = np.linalg.solve(M, np.concatenate([zz, b]))
        except np.linalg.LinAlgError:
            continue
        x, mu = sol[:n], sol[n:]
        if (G @ x >= -1e-11 * lam).all() and (mu[1:] >= -1e-11).all():
            d = float(np.sum((x - zz) ** 2))
            if best is None or d < best[0] - 1e-14:
                best = (d, x)
    return best[1][0], best[1][1:]


def kkt_certificate(z0, z, v, w, v0, lam, y0, y, act_tol=1e-10):
    """Return (stationarity residual, max primal violation, min multiplier) for
    the candidate x = (y0, y): x - zz = nu*1 + sum_active mult_a G_a with
    mult >= 0 (NNLS over active rows, nu split into +/- parts)."""
    z = np.asarray(z, float)
    k = z.shape[0]
    G = polytope_rows(v, w, v0)
    x = np.concatenate([[y0], np.asarray(y, float)])
    zz = np.concatenate([[z0], z])
    slack = G @ x
    scale = max(lam, np.abs(zz).max())
    active = np.flatnonzero(slack <= act_tol * scale)
    # x - zz = nu * 1 + G_act^T mult  (projection onto {x: 1^T x = lam, G x >= 0})
    cols = [np.ones(k + 1), -np.ones(k + 1)] + [G[a] for a in active]
    Amat = np.array(cols).T
    coef, res = nnls(Amat, x - zz, maxiter=50 * Amat.shape[1])
    primal = max(abs(x.sum() - lam), float(np.maximum(-slack, 0).max()))
    return res / scale, primal / scale, float(coef.min()) if coef.size else 0.0
