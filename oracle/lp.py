"""LP optima of the GAM SBLP / CBLP -- TEST INFRASTRUCTURE (oracle side).

* sblp_rows(inst)        the SBLP of P:L229-239 with the GAM scale rows
                         (reading c3), direct form:
                           max  sum_ij r_j y_ij
                           s.t. sum_i y_ij <= c_j                       (Eq. 7)
                                y_i0 + sum_j y_ij = lambda_i            (Eq. 8)
                                vt_i0 y_ij - v_ij (y_i0 + sum_k omega_ik y_ik) <= 0
                                  (GAM form of Eq. 9; omega = 0 gives
                                   y_ij / v_ij <= y_i0 / v_i0 exactly)
                                y >= 0                                   (Eq. 10)
* dense_simplex(...)     textbook two-phase tableau simplex with Bland's rule
                         (the north_star's "textbook dense LP solve").
* sblp_highs(inst)       the same LP through scipy's HiGHS (library primitive),
                         sparse form with the auxiliary U_i = (y_i0 + sum omega y)/vt_i0.
* cblp_lp(inst)          the choice-based LP P:L211-224 over all assortments
                         S subset of C_i with GAM probabilities:
                         pi_ij(S) = v_ij / (v_i0 + sum_{k in S} v_ik + sum_{k in C_i \\ S} w_ik).
"""
from __future__ import annotations

import itertools

import numpy as np


# ---------------------------------------------------------------- simplex
def dense_simplex(c, A_ub=None, b_ub=None, A_eq=None, b_eq=None, tol=1e-11, max_iter=100_000):
    """max c^T x  s.t.  A_ub x <= b_ub, A_eq x = b_eq, x >= 0.

    Two-phase dense tableau, Bland's rule (smallest eligible index enters;
    ratio-test ties leave by smallest basic index).  Returns (x, objective)."""
    c = np.asarray(c, dtype=np.float64)
    n = c.shape[0]
    rows, rhs, nslack = [], [], 0
    A_ub = np.zeros((0, n)) if A_ub is None else np.asarray(A_ub, dtype=np.float64)
    A_eq = np.zeros((0, n)) if A_eq is None else np.asarray(A_eq, dtype=np.float64)
    b_ub = np.zeros(0) if b_ub is None else np.asarray(b_ub, dtype=np.float64)
    b_eq = np.zeros(0) if b_eq is None else np.asarray(b_eq, dtype=np.float64)
    mu, me = A_ub.shape[0], A_eq.shape[0]
    M = mu + me
    ncol = n + mu                                # structural + slacks
    A = np.zeros((M, ncol))
    b = np.zeros(M)
    A[:mu, :n] = A_ub
    A[:mu, n:n + mu] = np.eye(mu)
    b[:mu] = b_ub
    A[mu:, :n] = A_eq
    b[mu:] = b_eq
    neg = b < 0
    A[neg] *= -1.0
    b[neg] *= -1.0
    # phase 1: artificial per row
    T = np.zeros((M + 1, ncol + M + 1))
    T[:M, :ncol] = A
    T[:M, ncol:ncol + M] = np.eye(M)
    T[:M, -1] = b
    basis = list(range(ncol, ncol + M))
    # objective row for phase 1: minimise sum of artificials == maximise -sum
    T[M, :ncol] = -A.sum(axis=0)
    T[M, -1] = -b.sum()

    def pivot(r, q):
        T[r] /= T[r, q]
        for i in range(M + 1):
            if i != r and T[i, q] != 0.0:
                T[i] -= T[i, q] * T[r]
        basis[r] = q

    def run(ncols_allowed):
        for _ in range(max_iter):
            cand = [q for q in range(ncols_allowed) if T[M, q] < -tol]
            if not cand:
                return
            q = cand[0]                              # Bland: smallest index
            col = T[:M, q]
            best, r_best = None, None
            for r in range(M):
                if col[r] > tol:
                    ratio = T[r, -1] / col[r]
                    if best is None or ratio < best - 1e-15 or (abs(ratio - best) <= 1e-15 and basis[r] < basis[r_best]):
                        best, r_best = ratio, r
            if r_best is None:
                raise ValueError("LP unbounded")
            pivot(r_best, q)
        raise RuntimeError("simplex iteration limit")

    run(ncol + M)
    if T[M, -1] < -1e-9 * max(1.0, b.sum()):
        raise ValueError("LP infeasible")
    # drive artificials out of the basis
    for r in range(M):
        if basis[r] >= ncol:
            for q in range(ncol):
                if abs(T[r, q]) > tol:
                    pivot(r, q)
                    break
    # phase 2
    T[M, :] = 0.0
    T[M, :ncol] = -np.concatenate([c, np.zeros(mu)])
    for r in range(M):
        if basis[r] < ncol and T[M, basis[r]] != 0.0:
            T[M] -= T[M, basis[r]] * T[r]
    T[:, ncol:ncol + M] = 0.0                    # artificials never re-enter
    run(ncol)
    x = np.zeros(ncol + M)
    for r in range(M):
        x[basis[r]] = T[r, -1]
    return x[:n], float(c @ x[:n])


# ---------------------------------------------------------------- SBLP
def sblp_rows(inst):
    """Direct-form SBLP matrices (dense).  Variable order: per segment i,
    [y_i0, y_i,C_i[0], ...].  Returns (c, A_ub, b_ub, A_eq, b_eq, layout)."""
    m, N = inst.m, inst.N
    ks = np.diff(inst.seg_ptr)
    nvar = int(m + ks.sum())
    col0 = np.zeros(m, dtype=np.int64)           # column of y_i0
    col0[1:] = np.cumsum(ks[:-1] + 1)
    cost = np.zeros(nvar)
    cap_rows = np.zeros((N, nvar))
    bal = np.zeros((m, nvar))
    scale_rows = []
    for i in range(m):
        sl = inst.row(i)
        prod = inst.prod_idx[sl]
        v = inst.attract[sl]
        w = inst.shadow[sl]
        om = w / v
        vt0 = inst.no_purchase[i] + w.sum()
        c0 = col0[i]
        cols = c0 + 1 + np.arange(prod.shape[0])
        cost[cols] = inst.price[prod]
        cap_rows[prod, cols] = 1.0
        bal[i, c0] = 1.0
        bal[i, cols] = 1.0
        for q in range(prod.shape[0]):
            row = np.zeros(nvar)
            row[c0] = -v[q]
            row[cols] -= v[q] * om
            row[cols[q]] += vt0
            scale_rows.append(row)
    keep = inst.present
    A_ub = np.vstack([cap_rows[keep]] + ([np.array(scale_rows)] if scale_rows else []))
    b_ub = np.concatenate([inst.capacity[keep], np.zeros(len(scale_rows))])
    return cost, A_ub, b_ub, bal, inst.arrival.copy(), col0


def sblp_dense(inst, uncapacitated=False):
    """P* of the SBLP by the textbook dense simplex (tiny instances only)."""
    cost, A_ub, b_ub, A_eq, b_eq, col0 = sblp_rows(inst)
    if uncapacitated:
        ncap = int(inst.present.sum())
        A_ub, b_ub = A_ub[ncap:], b_ub[ncap:]
    x, obj = dense_simplex(cost, A_ub, b_ub, A_eq, b_eq)
    return obj, x


def sblp_highs(inst, uncapacitated=False):
    """P* of the SBLP through scipy.optimize.linprog(method='highs'), sparse
    U-auxiliary form.  Returns (objective, y, y0)."""
    import scipy.sparse as sp
    from scipy.optimize import linprog

    m, N, nnz = inst.m, inst.N, inst.nnz
    ks = np.diff(inst.seg_ptr)
    rows_of = np.repeat(np.arange(m), ks)
    om = inst.shadow / inst.attract
    vt0 = inst.no_purchase + np.add.reduceat(inst.shadow, inst.seg_ptr[:-1]) * (ks > 0)
    # variables: y [nnz], y0 [m], U [m]
    ny, n0 = nnz, m
    nv = ny + 2 * m
    iy = np.arange(ny)
    i0 = ny + np.arange(m)
    iU = ny + m + np.arange(m)
    cost = np.zeros(nv)
    cost[:ny] = -inst.price[inst.prod_idx]
    # equalities: balance, U definition
    r_bal = sp.coo_matrix((np.ones(ny + m), (np.concatenate([rows_of, np.arange(m)]),
                                             np.concatenate([iy, i0]))), shape=(m, nv))
    r_def = sp.coo_matrix((np.concatenate([om, np.ones(m), -vt0]),
                           (np.concatenate([rows_of, np.arange(m), np.arange(m)]),
                            np.concatenate([iy, i0, iU]))), shape=(m, nv))
    A_eq = sp.vstack([r_bal, r_def]).tocsr()
    b_eq = np.concatenate([inst.arrival, np.zeros(m)])
    # inequalities: y_ij - v_ij U_i <= 0 ; capacities
    r_sc = sp.coo_matrix((np.concatenate([np.ones(ny), -inst.attract]),
                          (np.concatenate([iy, iy]), np.concatenate([iy, iU[rows_of]]))), shape=(ny, nv))
    blocks = [r_sc]
    b_ub = [np.zeros(ny)]
    L = int(getattr(inst, "num_resources", 0) or 0)
    if not uncapacitated and L > 0:
        # bundles (Eq. 33): sum_i sum_j Bt_lj y_ij <= c_l
        bp, br = np.asarray(inst.bundle_ptr), np.asarray(inst.bundle_res)
        nres = np.diff(bp)[inst.prod_idx]                     # resources per entry
        rr = np.concatenate([br[bp[j]:bp[j + 1]] for j in inst.prod_idx]) if ny else np.zeros(0, int)
        cc = np.repeat(iy, nres)
        r_cap = sp.coo_matrix((np.ones(rr.size), (rr, cc)), shape=(L, nv))
        blocks.append(r_cap)
        b_ub.append(np.asarray(inst.resource_capacity, dtype=np.float64))
    elif not uncapacitated:
        keep = np.flatnonzero(inst.present)
        pos = np.full(N, -1)
        pos[keep] = np.arange(keep.size)
        r_cap = sp.coo_matrix((np.ones(ny), (pos[inst.prod_idx], iy)), shape=(keep.size, nv))
        blocks.append(r_cap)
        b_ub.append(inst.capacity[keep])
    A_ub = sp.vstack(blocks).tocsr()
    res = linprog(cost, A_ub=A_ub, b_ub=np.concatenate(b_ub), A_eq=A_eq, b_eq=b_eq,
                  bounds=(0, None), method="highs",
                  options=dict(primal_feasibility_tolerance=1e-10, dual_feasibility_tolerance=1e-10))
    if res.status != 0:
        raise RuntimeError(f"HiGHS: {res.message}")
    return -res.fun, res.x[:ny], res.x[ny:ny + n0]


# ---------------------------------------------------------------- CBLP
def gam_choice_prob(v, w, v0, S):
    """pi_j(S) for j in S (P:L202 with BASELINE names): v_j / (v0 + sum_S v + sum_{C\\S} w)."""
    S = np.asarray(S, dtype=bool)
    den = v0 + v[S].sum() + w[~S].sum()
    return np.where(S, v / den, 0.0)


def cblp_columns(inst):
    """Columns (i, S, revenue, usage-vector) of the CBLP P:L211-224."""
    cols = []
    for i in range(inst.m):
        sl = inst.row(i)
        prod, v, w = inst.prod_idx[sl], inst.attract[sl], inst.shadow[sl]
        k = prod.shape[0]
        for bits in itertools.product((False, True), repeat=k):
            S = np.array(bits, dtype=bool)
            pi = gam_choice_prob(v, w, inst.no_purchase[i], S)
            use = np.zeros(inst.N)
            use[prod] = pi
            cols.append((i, S, float((inst.price[prod] * pi).sum()), use))
    return cols


def cblp_lp(inst, uncapacitated=False, solver="dense"):
    """CBLP optimum by assortment enumeration (tiny instances, k <= ~8)."""
    cols = cblp_columns(inst)
    n = len(cols)
    cost = np.array([c[2] for c in cols])
    A_eq = np.zeros((inst.m, n))
    for q, (i, _S, _r, _u) in enumerate(cols):
        A_eq[i, q] = 1.0
    b_eq = inst.arrival.copy()
    if uncapacitated:
        A_ub, b_ub = None, None
    else:
        keep = inst.present
        A_ub = np.array([c[3][keep] for c in cols]).T
        b_ub = inst.capacity[keep]
    if solver == "dense":
        _x, obj = dense_simplex(cost, A_ub, b_ub, A_eq, b_eq)
        return obj
    from scipy.optimize import linprog
    res = linprog(-cost, A_ub=A_ub, b_ub=b_ub, A_eq=A_eq, b_eq=b_eq, bounds=(0, None), method="highs")
    return -res.fun


def best_assortment_value(g, v, w, v0, lam):
    """max over all S subset of C of lambda * sum_{j in S} g_j pi_j(S) (brute force, k <= ~14)."""
    k = len(g)
    best = 0.0
    for bits in itertools.product((False, True), repeat=k):
        S = np.array(bits, dtype=bool)
        val = lam * float((np.asarray(g) * gam_choice_prob(np.asarray(v), np.asarray(w), v0, S)).sum())
        best = max(best, val)
    return best
