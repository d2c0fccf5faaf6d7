/*
 * oracle/spfom_oracle.c -- plain single-threaded fp64 CPU oracle of SPFOM's
 * per-iteration primal-dual update for the GAM sales-based LP (SBLP).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with paper_2602_22421_b200/
 * (the CUDA path), and neither includes the other.
 *
 * Notation (BASELINE.json names; PAPER.md = P, SPEC.md = S, SURVEY.md = SV):
 *   m segments i, N products j, consideration set C_i (CSR row i),
 *   v_ij attraction, w_ij shadow attraction (GAM, 0 <= w < v),
 *   omega_ij = w_ij / v_ij, vt_ij = v_ij - w_ij, vt_i0 = v_i0 + sum_{C_i} w_ik,
 *   lambda_i arrival, r_j price, c_j capacity, eta_j capacity dual,
 *   y_ij sales, y_i0 no-purchase, s_j = sum_i y_ij usage (= (A y)_j).
 *
 * Functions and the passages they follow:
 *   oracle_project   Euclidean projection onto the segment polytope Y_i
 *                    (Eqs. 8-10 extended to GAM, P:L199-204;
 *                    readings c3/c5, SV App. A.1-A.2).  Semi-smooth Newton on
 *                    the 3-scalar KKT system, cold start, backtracking on the
 *                    residual infinity-norm; the result is accepted only after
 *                    a KKT check (feasibility, multiplier signs, residuals).
 *   oracle_argmax    exact inner maximisation z_i (reading c6):
 *                    enumerate the ratio-ordered prefixes, take the best value
 *                    z*, then S* = {j : g_j v_j > z* vt_j} (strict ties).
 *   oracle_fast_inner  Algorithm 1 FAST-INNER (MNL), with the
 *                    budget initialised to lambda_i - y_i0 (reading c6).
 *   oracle_golden    golden-section search over y_i0.
 *   oracle_iterate   one SPFOM iteration: primal block step (finite theta:
 *                    gradient step + projection; theta = inf: the
 *                    exact inner argmax, Alg. 2), usage sum
 *                    (P:L357), extrapolation (reading c8, NOT in the paper),
 *                    dual step Eq. 17 with per-product tau_j,
 *                    optional uniform averaging (reading c9, NOT in the paper).
 *   oracle_recover   SBLP -> CBLP policy recovery (P:L473-492 Lemma
 *                    "recover", GAM reading SV App. A.1):
 *                    nested assortments by y_j / v_j descending and their
 *                    offer probabilities alpha(S_l).
 *   bundles (NRM, Eq. 33): with L > 0 resources the
 *                    capacity rows are sum_i sum_j Bt_lj y_ij <= c_l; prices
 *                    g_j = r_j - sum_{l in B_j} eta_l (the Lagrangian
 *                    coefficient), the dual step runs over resources on
 *                    St_l = sum_{j : l in B_j} st_j, tau_l = tau / n_l with
 *                    n_l = sum_{j : l in B_j} n_j (reading c17).
 *   oracle_residuals objective (Eq. 6), Lagrangian dual bound
 *                    D(eta) = c^T eta + sum_i lambda_i z_i(r - eta),
 *                    infeasibility, certificate (reading c11).
 *
 * Sums are sequential in index order.  Build: gcc -O2 -ffp-contract=off.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENUMERIC 3

int oracle_version(void) { return 1; }

/* ------------------------------------------------------------------------ */
/* 3x3 linear solve, Gaussian elimination with partial pivoting.           */
static int solve3(double J[3][3], const double b[3], double x[3]) {
    double A[3][4];
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) A[r][c] = J[r][c];
        A[r][3] = b[r];
    }
    for (int c = 0; c < 3; ++c) {
        int p = c;
        for (int r = c + 1; r < 3; ++r)
            if (fabs(A[r][c]) > fabs(A[p][c])) p = r;
        if (A[p][c] == 0.0) return -1;
        if (p != c)
            for (int q = 0; q < 4; ++q) { double t = A[c][q]; A[c][q] = A[p][q]; A[p][q] = t; }
        for (int r = c + 1; r < 3; ++r) {
            double f = A[r][c] / A[c][c];
            for (int q = c; q < 4; ++q) A[r][q] -= f * A[c][q];
        }
    }
    for (int r = 2; r >= 0; --r) {
        double acc = A[r][3];
        for (int q = r + 1; q < 3; ++q) acc -= A[r][q] * x[q];
        x[r] = acc / A[r][r];
    }
    return 0;
}

/*
 * KKT of  min 1/2 (y0 - z0)^2 + 1/2 sum_j (y_j - z_j)^2  over Y_i:
 *   y0 + sum_j y_j = lambda                       (balance, multiplier nu)
 *   0 <= y_j <= v_j U,  U = (y0 + sum_k omega_k y_k) / vt0   (GAM scale)
 * Stationarity gives y0 = z0 - nu + kappa and y_j = clamp(a_j, 0, v_j U),
 * a_j = z_j - nu + omega_j kappa, with (nu, kappa, U) solving
 *   R1 = sum_j v_j (a_j - v_j U)^+ - vt0 kappa = 0
 *   R2 = y0 + sum_j omega_j y_j - vt0 U         = 0
 *   R3 = y0 + sum_j y_j - lambda                = 0.
 * eval_point computes y, R and the generalized Jacobian at x = (nu, kappa, U).
 */
typedef struct {
    double R[3];
    double J[3][3];
    double scale;   /* magnitude of the summed terms, for the stopping test */
} eval_t;

static void eval_point(int64_t k, double z0, const double *z, const double *v,
                       const double *om, double vt0, double lam, const double x[3],
                       double *y0, double *y, eval_t *e) {
    const double nu = x[0], ka = x[1], U = x[2];
    double r1 = 0.0, sy = 0.0, swy = 0.0, scale = fabs(lam) + fabs(z0) + fabs(nu) + fabs(ka);
    double cv = 0.0, cvw = 0.0, cvv = 0.0, fw = 0.0, fww = 0.0, nf = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        double a = z[j] - nu + om[j] * ka;
        double cap = v[j] * U;
        double yj;
        if (a >= cap) {            /* capped: y_j = v_j U, alpha_j = a_j - v_j U >= 0 */
            yj = cap;
            r1 += v[j] * (a - cap);
            cv += v[j];
            cvw += v[j] * om[j];
            cvv += v[j] * v[j];
        } else if (a > 0.0) {      /* free */
            yj = a;
            fw += om[j];
            fww += om[j] * om[j];
            nf += 1.0;
        } else {                   /* at zero */
            yj = 0.0;
        }
        y[j] = yj;
        sy += yj;
        swy += om[j] * yj;
        scale += fabs(z[j]) + fabs(cap);
    }
    *y0 = z0 - nu + ka;
    e->R[0] = r1 - vt0 * ka;
    e->R[1] = *y0 + swy - vt0 * U;
    e->R[2] = *y0 + sy - lam;
    /* d/d(nu, kappa, U) */
    e->J[0][0] = -cv;        e->J[0][1] = cvw - vt0;   e->J[0][2] = -cvv;
    e->J[1][0] = -1.0 - fw;  e->J[1][1] = 1.0 + fww;   e->J[1][2] = cvw - vt0;
    e->J[2][0] = -1.0 - nf;  e->J[2][1] = 1.0 + fw;    e->J[2][2] = cv;
    e->scale = scale * (1.0 + vt0);
}

static double rnorm(const double R[3]) {
    double a = fabs(R[0]), b = fabs(R[1]), c = fabs(R[2]);
    return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

/*
 * Euclidean projection (y0, y) = Pi_{Y_i}(z0, z).  Returns OR_OK, or
 * OR_ENUMERIC when Newton fails or the KKT check rejects the result.
 * mult (optional) receives (nu, kappa, U); iters (optional) the number of
 * residual evaluations.
 */
int oracle_project(int64_t k, double z0, const double *z, const double *v, const double *w,
                   double v0, double lam, double *y0, double *y, double *mult, int *iters) {
    if (k < 0 || !(lam > 0.0) || !(v0 > 0.0)) return OR_EINVAL;
    if (k == 0) {               /* empty consideration set: all mass on no-purchase */
        *y0 = lam;
        if (mult) { mult[0] = z0 - lam; mult[1] = 0.0; mult[2] = lam / v0; }
        if (iters) *iters = 0;
        return OR_OK;
    }
    double *om = (double *)malloc((size_t)k * sizeof(double));
    double *yt = (double *)malloc((size_t)k * sizeof(double));
    if (!om || !yt) { free(om); free(yt); return OR_EINVAL; }
    double vt0 = v0, sumz = 0.0, sumvt = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        om[j] = w[j] / v[j];
        vt0 += w[j];
        sumz += z[j];
        sumvt += v[j] - w[j];
    }
    /* cold start (SV App. A.2) */
    double x[3] = {(z0 + sumz - lam) / (double)(k + 1), 0.0, lam / (vt0 + sumvt)};
    eval_t e, et;
    double yt0;
    eval_point(k, z0, z, v, om, vt0, lam, x, y0, y, &e);
    int evals = 1, status = OR_ENUMERIC;
    const double eps = 1e-15;
    for (int it = 0; it < 500; ++it) {
        double nr = rnorm(e.R);
        if (nr <= 8.0 * eps * e.scale) { status = OR_OK; break; }
        double d[3], mR[3] = {-e.R[0], -e.R[1], -e.R[2]};
        if (solve3(e.J, mR, d) != 0) break;
        double step = 1.0, xt[3];
        int accepted = 0;
        for (int bt = 0; bt < 60; ++bt) {
            xt[0] = x[0] + step * d[0];
            xt[1] = x[1] + step * d[1];
            xt[2] = x[2] + step * d[2];
            eval_point(k, z0, z, v, om, vt0, lam, xt, &yt0, yt, &et);
            ++evals;
            double nt = rnorm(et.R);
            if (nt <= (1.0 - 1e-4 * step) * nr || nt <= 8.0 * eps * et.scale) { accepted = 1; break; }
            step *= 0.5;
        }
        if (!accepted) {
            /* Full Newton step on the current piece; if the residual cannot be
             * reduced we are at rounding level: stop and let the KKT check decide. */
            status = OR_OK;
            break;
        }
        x[0] = xt[0]; x[1] = xt[1]; x[2] = xt[2];
        e = et;
        *y0 = yt0;
        memcpy(y, yt, (size_t)k * sizeof(double));
    }
    if (status == OR_OK) {
        /* KKT check in the original variables: balance, 0 <= y_j <= v_j U(y),
         * kappa >= 0, U > 0, and the residuals of the multiplier equations. */
        double sy = 0.0, swy = 0.0, ymax = lam;
        for (int64_t j = 0; j < k; ++j) { sy += y[j]; swy += om[j] * y[j]; }
        double Uy = (*y0 + swy) / vt0;
        double tol = 1e-12 * (e.scale > ymax ? e.scale : ymax);
        if (fabs(*y0 + sy - lam) > tol) status = OR_ENUMERIC;
        if (x[1] < -tol || !(x[2] > 0.0)) status = OR_ENUMERIC;
        for (int64_t j = 0; j < k; ++j)
            if (y[j] < 0.0 || y[j] > v[j] * Uy + tol) status = OR_ENUMERIC;
        if (rnorm(e.R) > tol) status = OR_ENUMERIC;
    }
    if (mult) { mult[0] = x[0]; mult[1] = x[1]; mult[2] = x[2]; }
    if (iters) *iters = evals;
    free(om);
    free(yt);
    return status;
}

/* ------------------------------------------------------------------------ */
/* Exact inner argmax (theta = inf).                                       */
typedef struct { double q; int64_t j; } ratio_t;

static int cmp_ratio(const void *pa, const void *pb) {
    const ratio_t *a = (const ratio_t *)pa, *b = (const ratio_t *)pb;
    if (a->q > b->q) return -1;
    if (a->q < b->q) return 1;
    return (a->j < b->j) ? -1 : (a->j > b->j);
}

/*
 * max sum_j g_j y_j over Y_i.  In (U, u_j = y_j / v_j) coordinates Y_i is
 * {0 <= u_j <= U, vt0 U + sum_j vt_j u_j = lambda}; its vertices are the
 * assortments S with y_j = lambda v_j / (vt0 + sum_S vt) (SV App. A.1), and
 * the best assortment is a prefix of the order g_j v_j / vt_j descending.
 * Returns lambda * z* (z* = best prefix value, >= 0 via the empty set);
 * writes y, y0 for S* = {j : g_j v_j > z* vt_j}; margin (optional) receives
 * min_j |g_j v_j - z* vt_j| / (|g_j v_j| + z* vt_j) over j with g_j > 0
 * (the tie distance, reading c13).
 */
double oracle_argmax(int64_t k, const double *g, const double *v, const double *w, double v0,
                     double lam, double *y0, double *y, double *margin) {
    double vt0 = v0;
    for (int64_t j = 0; j < k; ++j) vt0 += w[j];
    ratio_t *ord = (ratio_t *)malloc((size_t)(k > 0 ? k : 1) * sizeof(ratio_t));
    int64_t nc = 0;
    for (int64_t j = 0; j < k; ++j)
        if (g[j] > 0.0) { ord[nc].q = g[j] * v[j] / (v[j] - w[j]); ord[nc].j = j; ++nc; }
    qsort(ord, (size_t)nc, sizeof(ratio_t), cmp_ratio);
    double zs = 0.0, num = 0.0, den = vt0;
    for (int64_t t = 0; t < nc; ++t) {
        int64_t j = ord[t].j;
        num += g[j] * v[j];
        den += v[j] - w[j];
        double val = num / den;
        if (val > zs) zs = val;
    }
    free(ord);
    double dS = vt0, mg = INFINITY;
    for (int64_t j = 0; j < k; ++j) {
        double lhs = g[j] * v[j], rhs = zs * (v[j] - w[j]);
        if (g[j] > 0.0) {
            double d = fabs(lhs - rhs) / (fabs(lhs) + rhs);
            if (d < mg) mg = d;
        }
        if (lhs > rhs) dS += v[j] - w[j];
    }
    double U = lam / dS, sy = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        double lhs = g[j] * v[j], rhs = zs * (v[j] - w[j]);
        y[j] = (lhs > rhs) ? v[j] * U : 0.0;
        sy += y[j];
    }
    *y0 = lam - sy;
    if (margin) *margin = mg;
    return lam * zs;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1 FAST-INNER (MNL: attraction v, no-purchase v0) for fixed y0. */
typedef struct { double g; int64_t j; } coef_t;

static int cmp_coef(const void *pa, const void *pb) {
    const coef_t *a = (const coef_t *)pa, *b = (const coef_t *)pb;
    if (a->g > b->g) return -1;
    if (a->g < b->g) return 1;
    return (a->j < b->j) ? -1 : (a->j > b->j);
}

/* Returns z_i = sum_j y_j g_j; OR-style failure is signalled by NAN
 * (y0 below the feasibility bound lambda v0 / (v0 + sum v)). */
double oracle_fast_inner(int64_t k, const double *g, const double *v, double v0, double lam,
                         double y0, double *y) {
    coef_t *ord = (coef_t *)malloc((size_t)(k > 0 ? k : 1) * sizeof(coef_t));
    for (int64_t j = 0; j < k; ++j) { ord[j].g = g[j]; ord[j].j = j; y[j] = 0.0; }
    qsort(ord, (size_t)k, sizeof(coef_t), cmp_coef);   /* descending (r_j - eta_j) */
    double budget = lam - y0;                          /* S:L217 correction */
    for (int64_t t = 0; t < k && budget > 0.0; ++t) {
        int64_t j = ord[t].j;
        double cap = v[j] * y0 / v0;
        double yj = cap < budget ? cap : budget;
        y[j] = yj;
        budget -= yj;
    }
    free(ord);
    if (budget > 1e-12 * lam) return NAN;
    double zval = 0.0;
    for (int64_t j = 0; j < k; ++j) zval += y[j] * g[j];
    return zval;
}

/* Golden-section search over y0 in [lambda v0/(v0+sum v), lambda] maximising
 * FAST-INNER's value; stops when the bracket is <= tol*lambda.
 * Writes the best evaluated point's y0, y. */
double oracle_golden(int64_t k, const double *g, const double *v, double v0, double lam,
                     double tol, double *y0, double *y) {
    double sv = 0.0;
    for (int64_t j = 0; j < k; ++j) sv += v[j];
    double lo = lam * v0 / (v0 + sv), hi = lam;
    const double ig = (sqrt(5.0) - 1.0) / 2.0;
    double *tmp = (double *)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
    double a = hi - ig * (hi - lo), b = lo + ig * (hi - lo);
    /* guard the lower endpoint against rounding below the feasibility bound */
    double fa = oracle_fast_inner(k, g, v, v0, lam, a, tmp);
    double fb = oracle_fast_inner(k, g, v, v0, lam, b, tmp);
    while (hi - lo > tol * lam) {
        if (fa >= fb) { hi = b; b = a; fb = fa; a = hi - ig * (hi - lo); fa = oracle_fast_inner(k, g, v, v0, lam, a, tmp); }
        else          { lo = a; a = b; fa = fb; b = lo + ig * (hi - lo); fb = oracle_fast_inner(k, g, v, v0, lam, b, tmp); }
    }
    double best = fa >= fb ? a : b;
    double val = oracle_fast_inner(k, g, v, v0, lam, best, y);
    *y0 = best;
    free(tmp);
    return val;
}

/* ------------------------------------------------------------------------ */
/* One SPFOM iteration.                                                    */
typedef struct {
    int64_t m, N;
    const int64_t *seg_ptr;
    const int32_t *prod_idx;
    const double *v, *w, *v0, *lam, *r, *c;
    /* bundles (L > 0): resources of bundle j = bres[bptr[j] .. bptr[j+1]), capacities cres[L];
     * eta / tau then have length L and c is unused */
    int64_t L;
    const int64_t *bptr;
    const int32_t *bres;
    const double *cres;
} oracle_instance;

static int64_t n_duals(const oracle_instance *in) { return in->L > 0 ? in->L : in->N; }

/* g_j = r_j - (A^T eta)_j: eta_j per product, or sum_{l in B_j} eta_l (bundles) */
static void prices(const oracle_instance *in, const double *eta, double *g) {
    for (int64_t j = 0; j < in->N; ++j) {
        if (in->L > 0) {
            double b = 0.0;
            for (int64_t e = in->bptr[j]; e < in->bptr[j + 1]; ++e) b += eta[in->bres[e]];
            g[j] = in->r[j] - b;
        } else {
            g[j] = in->r[j] - eta[j];
        }
    }
}

/* public: g = r - A^T eta (test access to the effective bundle prices) */
void oracle_prices(const oracle_instance *in, const double *eta, double *g) { prices(in, eta, g); }

/* resource usage St_l = sum_{j : l in B_j} x_j (j ascending) */
static void resource_sum(const oracle_instance *in, const double *x, double *St) {
    for (int64_t l = 0; l < in->L; ++l) St[l] = 0.0;
    for (int64_t j = 0; j < in->N; ++j)
        for (int64_t e = in->bptr[j]; e < in->bptr[j + 1]; ++e) St[in->bres[e]] += x[j];
}

typedef struct {
    double theta;          /* > 0; INFINITY => exact inner argmax (Alg. 2)   */
    double mu;             /* Eq. 17 penalty, >= 0                            */
    double extrapolation;  /* omega_x in [0, 1]; 0 = paper                    */
    int32_t averaging;     /* 0 = off (paper)                                 */
    int32_t pad_;
    int64_t refresh_every; /* sampled mode: recompute s from y every K its    */
} oracle_params;

typedef struct {
    double *y, *y0, *eta, *s;      /* iterate; s = A y (stale rows included) */
    double *ybar, *y0bar, *etabar; /* running averages (may be NULL if off)  */
    int64_t t;                     /* completed iterations                    */
} oracle_state;

/* tau_j = tau (mode 0) or tau / n_j (mode 1; n_j = #segments considering j,
 * tau for n_j = 0).  Reading c8 (per-product steps are NOT in the paper). */
void oracle_tau(const oracle_instance *in, double tau, int mode, double *tau_j) {
    int64_t *n = (int64_t *)calloc((size_t)in->N, sizeof(int64_t));
    for (int64_t e = 0; e < in->seg_ptr[in->m]; ++e) n[in->prod_idx[e]] += 1;
    if (in->L > 0) {               /* bundles: n_l = sum_{j : l in B_j} n_j, one tau per resource */
        int64_t *nl = (int64_t *)calloc((size_t)in->L, sizeof(int64_t));
        for (int64_t j = 0; j < in->N; ++j)
            for (int64_t e = in->bptr[j]; e < in->bptr[j + 1]; ++e) nl[in->bres[e]] += n[j];
        for (int64_t l = 0; l < in->L; ++l)
            tau_j[l] = (mode == 1 && nl[l] > 0) ? tau / (double)nl[l] : tau;
        free(nl);
    } else {
        for (int64_t j = 0; j < in->N; ++j)
            tau_j[j] = (mode == 1 && n[j] > 0) ? tau / (double)n[j] : tau;
    }
    free(n);
}

/* Initial state (reading c10): y = 0, y0 = lambda, eta = 0, s = 0. */
void oracle_init(const oracle_instance *in, oracle_state *st) {
    for (int64_t e = 0; e < in->seg_ptr[in->m]; ++e) st->y[e] = 0.0;
    for (int64_t i = 0; i < in->m; ++i) st->y0[i] = in->lam[i];
    for (int64_t j = 0; j < in->N; ++j) st->s[j] = 0.0;
    for (int64_t j = 0; j < n_duals(in); ++j) st->eta[j] = 0.0;
    if (st->ybar) {
        for (int64_t e = 0; e < in->seg_ptr[in->m]; ++e) st->ybar[e] = 0.0;
        for (int64_t i = 0; i < in->m; ++i) st->y0bar[i] = in->lam[i];
        for (int64_t j = 0; j < n_duals(in); ++j) st->etabar[j] = 0.0;
    }
    st->t = 0;
}

/* Projected dual step, Eq. 17 (mu = 0 gives Alg. 2's step
 * P:L357) on the extrapolated usage st = s_new + omega_x (s_new - s_old):
 *   eta_j <- max{0, (1 - tau_j mu) eta_j - tau_j (c_j - st_j)}. */
void oracle_dual_step(int64_t N, double *eta, const double *s_new, const double *s_old,
                      const double *c, const double *tau_j, double mu, double omega_x) {
    for (int64_t j = 0; j < N; ++j) {
        double sx = s_new[j] + omega_x * (s_new[j] - s_old[j]);
        double e = (1.0 - tau_j[j] * mu) * eta[j] - tau_j[j] * (c[j] - sx);
        eta[j] = e > 0.0 ? e : 0.0;
    }
}

/* Dual step of either form: per product (Eq. 17) or, with bundles, per
 * resource on St = sum_{j in bundles(l)} (s_new + omega_x (s_new - s_old))_j. */
static void dual_step_any(const oracle_instance *in, const oracle_params *p, const double *tau,
                          double *eta, const double *s_new, const double *s_old) {
    if (in->L == 0) {
        oracle_dual_step(in->N, eta, s_new, s_old, in->c, tau, p->mu, p->extrapolation);
        return;
    }
    double *sx = (double *)malloc((size_t)in->N * sizeof(double));
    double *St = (double *)malloc((size_t)in->L * sizeof(double));
    for (int64_t j = 0; j < in->N; ++j) sx[j] = s_new[j] + p->extrapolation * (s_new[j] - s_old[j]);
    resource_sum(in, sx, St);
    for (int64_t l = 0; l < in->L; ++l) {
        double e = (1.0 - tau[l] * p->mu) * eta[l] - tau[l] * (in->cres[l] - St[l]);
        eta[l] = e > 0.0 ? e : 0.0;
    }
    free(sx);
    free(St);
}

static int update_segment(const oracle_instance *in, const oracle_params *p, const double *g,
                          int64_t i, oracle_state *st, double *zbuf, double *gbuf, double *yb) {
    int64_t a = in->seg_ptr[i], k = in->seg_ptr[i + 1] - a;
    const int32_t *idx = in->prod_idx + a;
    for (int64_t q = 0; q < k; ++q) gbuf[q] = g[idx[q]];          /* A^T eta gather */
    if (isinf(p->theta)) {
        double y0n;
        oracle_argmax(k, gbuf, in->v + a, in->w + a, in->v0[i], in->lam[i], &y0n, yb, NULL);
        st->y0[i] = y0n;
    } else {
        for (int64_t q = 0; q < k; ++q) zbuf[q] = st->y[a + q] + p->theta * gbuf[q];  /* z_i0 = y_i0 */
        double y0n;
        int rc = oracle_project(k, st->y0[i], zbuf, in->v + a, in->w + a, in->v0[i], in->lam[i],
                                &y0n, yb, NULL, NULL);
        if (rc != OR_OK) return rc;
        st->y0[i] = y0n;
    }
    memcpy(st->y + a, yb, (size_t)k * sizeof(double));
    return OR_OK;
}

static void fresh_usage(const oracle_instance *in, const double *y, double *s) {
    for (int64_t j = 0; j < in->N; ++j) s[j] = 0.0;
    for (int64_t i = 0; i < in->m; ++i)
        for (int64_t e = in->seg_ptr[i]; e < in->seg_ptr[i + 1]; ++e) s[in->prod_idx[e]] += y[e];
}

/*
 * One iteration t -> t+1 (SV §8(c) oracle algorithm):
 *   for i in I_t ascending: z0 = y0_i, z_j = y_ij + theta (r_j - eta_j); project
 *                           (theta = inf: exact inner argmax with g = r - eta)
 *   s_new = A y  (full sweep: fresh sum in i order; sampled: s + sum of row deltas)
 *   st = s_new + omega_x (s_new - s);  eta_j = max(0, (1 - tau_j mu) eta_j - tau_j (c_j - st_j))
 * block == NULL or B == m => full sweep.
 */
int oracle_iterate(const oracle_instance *in, const oracle_params *p, const double *tau_j,
                   const int32_t *block, int64_t B, oracle_state *st) {
    int64_t m = in->m, N = in->N, kmax = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t k = in->seg_ptr[i + 1] - in->seg_ptr[i];
        if (k > kmax) kmax = k;
    }
    double *g = (double *)malloc((size_t)N * sizeof(double));
    double *zb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    double *gb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    double *yb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    double *yold = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    double *snew = (double *)malloc((size_t)N * sizeof(double));
    int rc = OR_OK;
    prices(in, st->eta, g);
    int full = (block == NULL || B == m);
    if (full) {
        for (int64_t i = 0; i < m && rc == OR_OK; ++i) rc = update_segment(in, p, g, i, st, zb, gb, yb);
        fresh_usage(in, st->y, snew);
    } else {
        for (int64_t j = 0; j < N; ++j) snew[j] = st->s[j];
        for (int64_t b = 0; b < B && rc == OR_OK; ++b) {
            int64_t i = block[b], a = in->seg_ptr[i], k = in->seg_ptr[i + 1] - a;
            memcpy(yold, st->y + a, (size_t)k * sizeof(double));
            rc = update_segment(in, p, g, i, st, zb, gb, yb);
            for (int64_t q = 0; q < k; ++q) snew[in->prod_idx[a + q]] += st->y[a + q] - yold[q];
        }
        if (p->refresh_every > 0 && (st->t + 1) % p->refresh_every == 0) fresh_usage(in, st->y, snew);
    }
    if (rc == OR_OK) {
        dual_step_any(in, p, tau_j, st->eta, snew, st->s);
        for (int64_t j = 0; j < N; ++j) st->s[j] = snew[j];
        st->t += 1;
        if (p->averaging && st->ybar) {
            double inv = 1.0 / (double)st->t;
            for (int64_t e = 0; e < in->seg_ptr[m]; ++e) st->ybar[e] += (st->y[e] - st->ybar[e]) * inv;
            for (int64_t i = 0; i < m; ++i) st->y0bar[i] += (st->y0[i] - st->y0bar[i]) * inv;
            for (int64_t j = 0; j < n_duals(in); ++j) st->etabar[j] += (st->eta[j] - st->etabar[j]) * inv;
        }
    }
    free(g); free(zb); free(gb); free(yb); free(yold); free(snew);
    return rc;
}

/* Sharded emulation (Alg. 3): a rank owns a
 * contiguous segment range (`in` is that shard).  oracle_primal_shard runs the
 * full-sweep primal step of its segments and writes the shard's usage
 * s_local = sum_{i in shard} y_i (i order); the caller sums the ranks' s_local
 * and oracle_dual_apply performs the dual step every rank performs identically
 * with that global usage.  Composed on one rank they are oracle_iterate's full
 * sweep without averaging. */
int oracle_primal_shard(const oracle_instance *in, const oracle_params *p, oracle_state *st, double *s_local) {
    int64_t m = in->m, N = in->N, kmax = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t k = in->seg_ptr[i + 1] - in->seg_ptr[i];
        if (k > kmax) kmax = k;
    }
    double *g = (double *)malloc((size_t)N * sizeof(double));
    double *zb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    double *gb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    double *yb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    int rc = OR_OK;
    prices(in, st->eta, g);
    for (int64_t i = 0; i < m && rc == OR_OK; ++i) rc = update_segment(in, p, g, i, st, zb, gb, yb);
    fresh_usage(in, st->y, s_local);
    free(g); free(zb); free(gb); free(yb);
    return rc;
}

void oracle_dual_apply(const oracle_instance *in, const oracle_params *p, const double *tau_j,
                       const double *s_new, oracle_state *st) {
    dual_step_any(in, p, tau_j, st->eta, s_new, st->s);
    for (int64_t j = 0; j < in->N; ++j) st->s[j] = s_new[j];
    st->t += 1;
}

/* ------------------------------------------------------------------------ */
/* Residuals and certificate (reading c11).  out[0..12]:
 *  0 primal_obj P = sum_j r_j s_j (s = fresh A y)
 *  1 dual_obj   D = sum_j c_j eta_j + sum_i lambda_i z_i*(r - eta)
 *  2 rel_gap    (D - P) / (1 + |P| + |D|)
 *  3 infeas_abs max_j (s_j - c_j)^+
 *  4 infeas_rel max_j (s_j - c_j)^+ / max(1, c_j)
 *  5 infeas_rel_l2 ||(s - c)^+||_2 / (1 + ||c||_2)
 *  6 balance_rel_max max_i |y0_i + sum_j y_ij - lambda_i| / lambda_i
 *  7 scale_rel_max   max_ij (y_ij - v_ij U_i)^+ / lambda_i, U_i = (y0_i + sum omega y)/vt0_i
 *  8 neg_max         max(-y)^+ over y_ij and y_i0
 *  9 compl_slack     sum_j eta_j |c_j - s_j| / (1 + |P|)
 * 10 cert_lower      (1 - alpha) P, alpha = max_j (s_j - c_j)^+ / s_j
 * 11 cert_upper      D
 * 12 alpha
 * `present` (optional, length N) excludes products no segment considers.
 * Bundles (L > 0): P = sum_j r_j s_j over bundles, the capacity terms (D's
 * c^T eta, infeasibility, complementary slackness, alpha) run over resources
 * on S_l = sum_{j : l in B_j} s_j.
 */
int oracle_residuals(const oracle_instance *in, const double *eta, const double *y, const double *y0,
                     const uint8_t *present, double *out) {
    int64_t m = in->m, N = in->N, kmax = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t k = in->seg_ptr[i + 1] - in->seg_ptr[i];
        if (k > kmax) kmax = k;
    }
    double *s = (double *)malloc((size_t)N * sizeof(double));
    double *g = (double *)malloc((size_t)N * sizeof(double));
    double *gb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    double *yb = (double *)malloc((size_t)(kmax + 1) * sizeof(double));
    fresh_usage(in, y, s);
    double P = 0.0, D = 0.0, ia = 0.0, ir = 0.0, il2 = 0.0, cn2 = 0.0, cs = 0.0, alpha = 0.0;
    prices(in, eta, g);
    for (int64_t j = 0; j < N; ++j)
        if (!present || present[j]) P += in->r[j] * s[j];
    /* capacity rows: products (c, s) or resources (cres, S = Bt s) */
    const int64_t nr = n_duals(in);
    double *S = s;
    if (in->L > 0) {
        S = (double *)malloc((size_t)in->L * sizeof(double));
        resource_sum(in, s, S);
    }
    const double *cap = in->L > 0 ? in->cres : in->c;
    for (int64_t j = 0; j < nr; ++j) {
        if (in->L == 0 && present && !present[j]) continue;
        D += cap[j] * eta[j];
        double over = S[j] - cap[j];
        if (over < 0.0) over = 0.0;
        if (over > ia) ia = over;
        double rel = over / (cap[j] > 1.0 ? cap[j] : 1.0);
        if (rel > ir) ir = rel;
        il2 += over * over;
        cn2 += cap[j] * cap[j];
        cs += eta[j] * fabs(cap[j] - S[j]);
        if (S[j] > 0.0 && over / S[j] > alpha) alpha = over / S[j];
    }
    if (in->L > 0) free(S);
    double bal = 0.0, scl = 0.0, neg = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t a = in->seg_ptr[i], k = in->seg_ptr[i + 1] - a;
        for (int64_t q = 0; q < k; ++q) gb[q] = g[in->prod_idx[a + q]];
        double y0d;
        D += oracle_argmax(k, gb, in->v + a, in->w + a, in->v0[i], in->lam[i], &y0d, yb, NULL);
        double sy = 0.0, swy = 0.0, vt0 = in->v0[i];
        for (int64_t q = 0; q < k; ++q) {
            sy += y[a + q];
            swy += in->w[a + q] / in->v[a + q] * y[a + q];
            vt0 += in->w[a + q];
            if (-y[a + q] > neg) neg = -y[a + q];
        }
        if (-y0[i] > neg) neg = -y0[i];
        double b = fabs(y0[i] + sy - in->lam[i]) / in->lam[i];
        if (b > bal) bal = b;
        double U = (y0[i] + swy) / vt0;
        for (int64_t q = 0; q < k; ++q) {
            double o = (y[a + q] - in->v[a + q] * U) / in->lam[i];
            if (o > scl) scl = o;
        }
    }
    out[0] = P;
    out[1] = D;
    out[2] = (D - P) / (1.0 + fabs(P) + fabs(D));
    out[3] = ia;
    out[4] = ir;
    out[5] = sqrt(il2) / (1.0 + sqrt(cn2));
    out[6] = bal;
    out[7] = scl;
    out[8] = neg;
    out[9] = cs / (1.0 + fabs(P));
    out[10] = (1.0 - alpha) * P;
    out[11] = D;
    out[12] = alpha;
    free(s); free(g); free(gb); free(yb);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* SBLP -> CBLP recovery (GAM: SV App. A.1).                    */
typedef struct { double u; int32_t id; int64_t j; } urank_t;

static int cmp_urank(const void *pa, const void *pb) {
    const urank_t *a = (const urank_t *)pa, *b = (const urank_t *)pb;
    if (a->u > b->u) return -1;
    if (a->u < b->u) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id);     /* ties: ascending product index */
}

/*
 * One feasible row (y0, y_1..y_k) of segment i with attraction v, shadow
 * attraction w, no-purchase weight v0 and arrival lambda.  Sort the products
 * by u_j = y_j / v_j descending (ties by ascending product id prod[j]); the
 * nested sets S_l are the first l of them (S_0: no product, only the
 * no-purchase option), l = 0..k.  With vt0 = v0 + sum_j w_j,
 * U = u_(0) = (y0 + sum_j (w_j / v_j) y_j) / vt0 and u_(k+1) = 0,
 *     alpha(S_l) = (u_(l) - u_(l+1)) * D(S_l) / lambda,
 *     D(S) = vt0 + sum_{j in S} (v_j - w_j)
 * -- the lemma's (y_l / w_l - y_{l+1} / w_{l+1}) * sum_{j in S_l} w_j / lambda
 * (paper letters: w = attraction, the sum includes option 0) with the GAM
 * normaliser D(S) = v0 + sum_S v + sum_{C \ S} w.  order[l - 1] receives the
 * row position j of the l-th product; alpha[0..k] the probabilities.
 */
void oracle_recover(int64_t k, double y0, const double *y, const double *v, const double *w, double v0,
                    double lam, const int32_t *prod, int64_t *order, double *alpha) {
    urank_t *r = (urank_t *)malloc((size_t)(k > 0 ? k : 1) * sizeof(urank_t));
    double vt0 = v0, swy = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        vt0 += w[j];
        swy += w[j] / v[j] * y[j];
        r[j].u = y[j] / v[j];
        r[j].id = prod[j];
        r[j].j = j;
    }
    qsort(r, (size_t)k, sizeof(urank_t), cmp_urank);
    double D = vt0, prev = (y0 + swy) / vt0;
    for (int64_t l = 0; l <= k; ++l) {
        const double next = (l < k) ? r[l].u : 0.0;
        alpha[l] = (prev - next) * D / lam;
        if (l < k) {
            const int64_t j = r[l].j;
            order[l] = j;
            D += v[j] - w[j];
            prev = next;
        }
    }
    free(r);
}
