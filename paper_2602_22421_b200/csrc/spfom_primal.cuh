// spfom_primal.cuh -- K1, the fused primal kernels of one SPFOM iteration.
//
//   a2 gather g_ij = r_j - eta_j (head of g staged in shared memory)
//   a3 gradient step z_ij = y_ij + theta g_ij, z_i0 = y_i0
//   a4 projection of (z_i0, z_i) onto Y_i (GAM polytope, reading c3/c5): semi-
//      smooth Newton on the 3-scalar KKT system in (nu, kappa, U), warm-started
//      from the segment's previous multipliers; theta = inf: exact inner argmax
//      by Dinkelbach (reading c6)
//   a5 usage scatter s_j += y_ij (sampled: y_new - y_old): the Zipf head
//      j < HH goes to group-private shared-memory histograms, flushed once per
//      persistent block; the tail uses global fp64 reductions.
//
// Two kernels share the per-segment device code:
//   k_primal_stream  full sweep over a contiguous bin (the hot path).  Every
//                    warp owns a contiguous range of rounds (GPW consecutive
//                    segments each); a round's rows are contiguous in every
//                    array, so the warp fetches round r+1 with six TMA bulk
//                    copies (cp.async.bulk, mbarrier completion) into its
//                    shared-memory slot while it computes round r.
//   k_primal         segment lists (sampled blocks, bins longer than 256
//                    entries): register-direct 128/256-bit loads.
//
// Thread mapping: a group of G lanes owns one segment; lane l holds quads
// l, l+G, .. (Q of them) of the padded row; a quad = 4 entries.
//
// KKT system: with a_j = z_j - nu + omega_j kappa and the
// piece C = {a_j >= v_j U} (capped), F = {0 < a_j < v_j U} (free):
//   R1 = sum_C v_j (a_j - v_j U) - vt0 kappa
//   R2 = y0 + sum_j omega_j y_j - vt0 U,   R3 = y0 + sum_j y_j - lambda,
//   y0 = z0 - nu + kappa, y_j = clamp(a_j, 0, v_j U).
// Per piece everything is affine, so the group sums are kept in piece-constant
// form: sum_C v a, sum_C v, sum_C v omega, sum_C v^2, |F|, sum_F a,
// sum_F omega a, sum_F omega, sum_F omega^2 (then sum_j y = U sum_C v + sum_F a,
// sum_j omega y = U sum_C v omega + sum_F omega a).
//
// Newton schedule per segment: a FULL pass evaluates the piece, R and the
// Jacobian and takes the Newton step; the next pass is a CHECK pass that only
// re-classifies: if no entry of the group changed class, R is affine on that
// piece, so the new point solves R = 0 exactly and the segment is done without
// any reduction.  Otherwise a FULL pass follows at the same point
// (sufficient-decrease test, backtracking on ||R||_inf).
//
// Head scatter: each G-lane group has its own histogram of the head products
// (ids are distinct within a segment, so a group's updates never collide and
// need no atomics); the block sums the histograms once at the end.
#pragma once

#include "spfom_common.cuh"

namespace spfom {

#ifndef SPFOM_FAST_RCP
#define SPFOM_FAST_RCP 1
#endif
// 1 / x to full double precision (within an ulp, not correctly rounded): the
// MUFU seed refined by two Newton steps -- ~50 cycles of dependent latency
// instead of ~130 for the IEEE division (B200, exp/ubench_fp64.cu).  Used for
// the Newton direction only, a search step, not an output.
__device__ __forceinline__ double fast_rcp(double x) {
#if SPFOM_FAST_RCP
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
#else
    return 1.0 / x;
#endif
}

// Solve J d = -R (3x3) by cofactors; false if singular / non-finite.
__device__ __forceinline__ bool newton_dir(const double J[3][3], const double R[3], double d[3]) {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    if (!(fabs(det) > 0.0) || !isfinite(det)) return false;
    const double inv = fast_rcp(det);
    const double c10 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    const double c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    const double c12 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    const double c20 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    const double c21 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    const double c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    d[0] = -(c00 * R[0] + c10 * R[1] + c20 * R[2]) * inv;   // J^{-1} = adj(J) / det
    d[1] = -(c01 * R[0] + c11 * R[1] + c21 * R[2]) * inv;
    d[2] = -(c02 * R[0] + c12 * R[1] + c22 * R[2]) * inv;
    return isfinite(d[0] + d[1] + d[2]);                    // one test: inf / NaN propagate into the sum
}

// max without the NaN-aware fmax expansion (callers test finiteness themselves)
__device__ __forceinline__ double dmax_sel(double a, double b) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}" : "=d"(r) : "d"(a), "d"(b));
    return r;
}

struct PieceSums {
    double sfa, sfwa, rva, cv, cvw, cvv, fw, fww;
    int nf;
};

// FULL pass, one entry: classify at (x0, x1, x2) = (nu, kappa, U), set the
// class bits and accumulate the piece-constant sums.  Branch-free: the inputs
// are selected (3 fp64 selects) and the 8 sums are plain fp64 adds -- ptxas
// if-converts predicated fp64 into selects of the results, which costs more.
// |F| is popc(fm) after the entry loop.
__device__ __forceinline__ void full_entry(double z, double v, double om, double x0, double x1, double x2,
                                           uint32_t bit, PieceSums &s, uint32_t &cm, uint32_t &fm) {
    const double a = fma(om, x1, z - x0);     // a = omega kappa + (z - nu)
    const double cap = v * x2;                // v U
    const bool isC = a >= cap;
    const bool isF = !isC && (a > 0.0);
    cm |= isC ? bit : 0u;
    fm |= isF ? bit : 0u;
    const double vc = isC ? v : 0.0;
    const double af = isF ? a : 0.0;
    const double wf = isF ? om : 0.0;
    s.rva = fma(vc, a, s.rva);                // sum_C v a
    s.cv += vc;                               // sum_C v
    s.cvw = fma(vc, om, s.cvw);               // sum_C v omega
    s.cvv = fma(vc, v, s.cvv);                // sum_C v^2
    s.sfa += af;                              // sum_F a
    s.sfwa = fma(om, af, s.sfwa);             // sum_F omega a
    s.fw += wf;                               // sum_F omega
    s.fww = fma(wf, om, s.fww);               // sum_F omega^2
}

// CHECK pass, one entry: class bits at (x0, x1, x2) only.
__device__ __forceinline__ void check_bits(double z, double v, double om, double x0, double x1, double x2,
                                           uint32_t bit, uint32_t &cm, uint32_t &fm) {
    const double a = fma(om, x1, z - x0);
    const double cap = v * x2;
    asm("{\n\t.reg .pred pc, pf;\n\t"
        "setp.ge.f64 pc, %2, %3;\n\t"
        "setp.gt.and.f64 pf, %2, 0d0000000000000000, !pc;\n\t"
        "@pc or.b32 %0, %0, %4;\n\t"
        "@pf or.b32 %1, %1, %4;\n\t"
        "}"
        : "+r"(cm), "+r"(fm)
        : "d"(a), "d"(cap), "r"(bit));
}

// Output, one entry: y_j = clamp(a_j, 0, v_j U) at (x0, x1, x2).
__device__ __forceinline__ double y_entry(double z, double v, double om, double x0, double x1, double x2) {
    const double a = fma(om, x1, z - x0);
    const double cap = v * x2;
    double y;
    // explicit selects (the C form is pattern-matched into a NaN-aware fmax)
    asm("{\n\t.reg .pred pc, pp;\n\t.reg .f64 t;\n\t"
        "setp.ge.f64 pc, %1, %2;\n\t"
        "setp.gt.f64 pp, %1, 0d0000000000000000;\n\t"
        "selp.f64 t, %1, 0d0000000000000000, pp;\n\t"
        "selp.f64 %0, %2, t, pc;\n\t}"
        : "=d"(y) : "d"(a), "d"(cap));
    return y;
}

#ifndef SPFOM_CHECK_OUT
#define SPFOM_CHECK_OUT 1
#endif
// CHECK pass + output, one entry: class bits at (x0, x1, x2) and
// y_j = clamp(a_j, 0, v_j U) from the same two comparisons (entry-mapped
// stream kernels; in the 168-register 12-warp layouts the extra live y values
// spill, so they keep the separate output pass).
__device__ __forceinline__ double check_out(double z, double v, double om, double x0, double x1, double x2,
                                            uint32_t bit, uint32_t &cm, uint32_t &fm) {
    const double a = fma(om, x1, z - x0);
    const double cap = v * x2;
    double y;
    asm("{\n\t.reg .pred pc, pf;\n\t.reg .f64 t;\n\t"
        "setp.ge.f64 pc, %3, %4;\n\t"
        "setp.gt.and.f64 pf, %3, 0d0000000000000000, !pc;\n\t"
        "@pc or.b32 %0, %0, %5;\n\t"
        "@pf or.b32 %1, %1, %5;\n\t"
        "selp.f64 t, %3, 0d0000000000000000, pf;\n\t"
        "selp.f64 %2, %4, t, pc;\n\t}"
        : "+r"(cm), "+r"(fm), "=d"(y)
        : "d"(a), "d"(cap), "r"(bit));
    return y;
}

// Diagnostics (exp/phase.py, exp/k1var.py; never in the product build):
//   SPFOM_DIAG_PHASE        cycles per phase of a K1 stream round (g_diag_phase)
//   SPFOM_DIAG_SKIP_PROJECT no projection (y <- a function of z): data movement only
//   SPFOM_DIAG_SKIP_RED     no global reductions in the stream kernel
//   SPFOM_DIAG_RED_FROM=j0  global reductions only for products >= j0
//   SPFOM_DIAG_SEP_USAGE    no usage scatter in K1; A y recomputed by k_usage before K3
//                           (+ SPFOM_DIAG_SEP_DUMMY: K1 still scatters, into discarded copies)
#ifdef SPFOM_DIAG_SPAN
// diagnostic: per block of the last K1 launch, %globaltimer at entry, after
// the block setup, the latest warp's loop end, and exit (after the flush)
// (indexed by %smid -- one persistent block per SM -- so that concurrent bin
// launches do not collide; g_diag_key[sm] = the bin's G * 10000 + Q * 100 + EQ)
__device__ unsigned long long g_diag_span[4 * 160];
__device__ unsigned int g_diag_key[160];
#define SPAN_MARK(k) do { unsigned long long t_; unsigned s_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s_)); \
    if ((k) == 2) atomicMax(&g_diag_span[4 * s_ + 2], t_); else if (threadIdx.x == 0) { g_diag_span[4 * s_ + (k)] = t_; \
    if ((k) == 0) g_diag_key[s_] = G * 10000 + Q * 100 + EQ; } } while (0)
#else
#define SPAN_MARK(k) do { } while (0)
#endif
#ifdef SPFOM_DIAG_PHASE
// [0] mbarrier wait, [1] slot read + gather + step, [2] projection, [3] y /
// state write-back, [4] head histograms, [5] global reductions, [6] rounds,
// [7] loop / claim, [8] TMA issue
__device__ unsigned long long g_diag_phase[10];
#define PH_MARK(k) do { const long long t_ = clock64(); ph[k] += t_ - ph_t; ph_t = t_; } while (0)
#else
#define PH_MARK(k) do { } while (0)
#endif
#ifdef SPFOM_DIAG_TIME
__device__ uint64_t g_diag_time[2 * 148 * 16];   // diagnostic: per-warp start / end of the last K1 launch
__device__ uint32_t g_diag_loops[4 * 148 * 16];  // diagnostic: per warp: mbarrier-wait, scatter kcycles, smid
#endif
struct ProjStats {
    unsigned long long passes = 0, failures = 0, restarts = 0;
};

// a4, theta < inf: Euclidean projection of (z0, z) onto Y_i for the segment of
// this G-lane group (reading c5).  (x0, x1, x2) holds the warm
// start (nu, kappa, U) on entry and the final multipliers on exit; yv / y0new
// receive the projected point.  Must be called by the whole warp.
template <int G, int NE, bool CO = false>
__device__ __forceinline__ void project_group(const double (&z)[NE], const double (&v)[NE], const double (&om)[NE],
                                              double z0, double lam, double vt0, bool active, unsigned gmask,
                                              int max_newton, double &x0, double &x1, double &x2,
                                              double (&yv)[NE], double &y0new, ProjStats &st) {
    double sabs = 0.0;
#pragma unroll
    for (int e = 0; e < NE; ++e) sabs += fabs(z[e]);
    sabs = group_sum<G>(sabs);
    const double tol = 1e-13 * (lam + fabs(z0) + sabs) * fmax(1.0, vt0);

    double a0 = x0, a1 = x1, a2 = x2;                   // last accepted point
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, step = 1.0, Ra = 0.0;
    uint32_t cA = 0, fA = 0;                            // class bitmasks at the accepted point
    bool go = active, full = true, first = true, failed = false, restarted = false;
    bool have_y = false;                                // yv formed by the final CHECK pass
    int passes = 0;
    const int restart_at = max_newton / 2;
    while (__any_sync(0xffffffffu, go)) {
#ifdef SPFOM_DIAG_TIME
        if ((threadIdx.x & 31) == 0) g_diag_loops[4 * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) + 3] += 1u;
#endif
        // safeguard: a segment still unconverged after half the budget restarts
        // from the cold point (nu, kappa, U) = ((z0 + sum z - lam)/(k+1), 0, lam/(vt0 + sum vt))
        if (__any_sync(0xffffffffu, go && passes == restart_at)) {
            double sz = 0.0, svt = 0.0, nk = 0.0;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                // opaque copies: keep this rare path from being hoisted out of the loop
                double ve = v[e], oe = om[e];
                asm volatile("" : "+d"(ve), "+d"(oe));
                sz += z[e];
                svt += fma(-ve, oe, ve);
                nk += ve > 0.0 ? 1.0 : 0.0;
            }
            sz = group_sum<G>(sz);
            svt = group_sum<G>(svt);
            nk = group_sum<G>(nk);
            if (go && passes == restart_at) {
                x0 = (z0 + sz - lam) / (nk + 1.0);
                x1 = 0.0;
                x2 = lam / (vt0 + svt);
                full = true;
                first = true;
                step = 1.0;
                restarted = true;
            }
        }
        const bool need = __any_sync(0xffffffffu, go && full);   // warp-uniform
        uint32_t cm = 0, fm = 0;
        if (!need) {
            // CHECK pass for every unfinished group of the warp
            if constexpr (CO && SPFOM_CHECK_OUT) {
                // ... which also forms y at the point (the same a and cap): when it
                // ends the loop for every group of the warp, that is the output
                // (groups finished earlier re-evaluate at their final multipliers)
#pragma unroll
                for (int e = 0; e < NE; ++e) yv[e] = check_out(z[e], v[e], om[e], x0, x1, x2, 1u << e, cm, fm);
            } else {
#pragma unroll
                for (int e = 0; e < NE; ++e) check_bits(z[e], v[e], om[e], x0, x1, x2, 1u << e, cm, fm);
            }
            const bool changed = (__ballot_sync(0xffffffffu, (cm != cA) || (fm != fA)) & gmask) != 0u;
            if (go) {
                ++passes;
                if (!changed) go = false;     // same piece: R(x) = 0 exactly
                else full = true;             // piece moved: evaluate R, J here
            }
            if constexpr (CO && SPFOM_CHECK_OUT) {
                if (!__any_sync(0xffffffffu, go)) {
                    have_y = true;
                    break;
                }
            }
            continue;
        }
        PieceSums ps = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0};
#pragma unroll
        for (int e = 0; e < NE; ++e) full_entry(z[e], v[e], om[e], x0, x1, x2, 1u << e, ps, cm, fm);
        ps.nf = __popc(fm);
        ps.sfa = group_sum<G>(ps.sfa);   ps.sfwa = group_sum<G>(ps.sfwa);
        ps.rva = group_sum<G>(ps.rva);   ps.cv = group_sum<G>(ps.cv);
        ps.cvw = group_sum<G>(ps.cvw);   ps.cvv = group_sum<G>(ps.cvv);
        ps.fw = group_sum<G>(ps.fw);     ps.fww = group_sum<G>(ps.fww);
#pragma unroll
        for (int o = G / 2; o >= 1; o >>= 1) ps.nf += __shfl_xor_sync(0xffffffffu, ps.nf, o);
        const bool changed = (__ballot_sync(0xffffffffu, (cm != cA) || (fm != fA)) & gmask) != 0u;
        if (go) {
            ++passes;
            if (!full) {
                // CHECK pass (evaluated as a full pass because another group needed one)
                if (!changed) go = false;
                else full = true;
            } else {
                const double y0c = z0 - x0 + x1;
                const double sy = fma(x2, ps.cv, ps.sfa);
                const double swy = fma(x2, ps.cvw, ps.sfwa);
                const double r1 = fma(-x2, ps.cvv, ps.rva);
                const double R[3] = {r1 - vt0 * x1, y0c + swy - vt0 * x2, y0c + sy - lam};
                const double nr = dmax_sel(fabs(R[0]), dmax_sel(fabs(R[1]), fabs(R[2])));   // NaN -> caught below
                // within tol at the warm start (an extrapolated warm start can be that
                // close): still one Newton step, so that the output is the exact
                // solution on its piece (balance / scale residuals at rounding level)
                bool done = !(nr > tol) && !first;
                if (!isfinite(nr)) { done = true; failed = true; }
                if (!done) {
                    if (first || nr <= (1.0 - 1e-4 * step) * Ra) {
                        const double dnf = (double)ps.nf;
                        const double J[3][3] = {{-ps.cv, ps.cvw - vt0, -ps.cvv},
                                                {-1.0 - ps.fw, 1.0 + ps.fww, ps.cvw - vt0},
                                                {-1.0 - dnf, 1.0 + ps.fw, ps.cv}};
                        double d[3];
                        if (!newton_dir(J, R, d)) {
                            done = true;
                            failed = !(nr <= tol);
                        } else {
                            a0 = x0; a1 = x1; a2 = x2;
                            d0 = d[0]; d1 = d[1]; d2 = d[2];
                            Ra = nr;
                            cA = cm;
                            fA = fm;
                            step = 1.0;
                            full = false;
                        }
                    } else {
                        step *= 0.5;
                        full = true;
                        if (step < 1e-12) { done = true; failed = true; }
                    }
                    if (!done && passes >= max_newton) {
                        done = true;                  // budget spent: keep the last evaluated point
                        failed = true;
                    }
                    if (!done) {
                        x0 = a0 + step * d0;
                        x1 = a1 + step * d1;
                        x2 = a2 + step * d2;
                        first = false;
                    }
                }
                if (done) go = false;
            }
        }
    }
    if (active && (threadIdx.x & (G - 1)) == 0) {
        st.passes += (unsigned long long)passes;
        st.failures += failed ? 1ull : 0ull;
#ifdef SPFOM_DIAG_LONG
        st.restarts += (passes > SPFOM_DIAG_LONG) ? 1ull : 0ull;   // diagnostic: segments needing many passes
#else
        st.restarts += restarted ? 1ull : 0ull;
#endif
    }
    if (!have_y) {
#pragma unroll
        for (int e = 0; e < NE; ++e) yv[e] = y_entry(z[e], v[e], om[e], x0, x1, x2);
    }
    y0new = z0 - x0 + x1;
}

// a4, theta = inf: exact inner argmax by Dinkelbach from z = 0 (reading c6;
// SURVEY App. A.3).  g holds the prices g_ij of the group's entries.
template <int G, int NE>
__device__ __forceinline__ void argmax_group(const double (&g)[NE], const double (&v)[NE], const double (&om)[NE],
                                             double lam, double vt0, bool active, double (&yv)[NE],
                                             double &y0new) {
    double zs = 0.0, den = 0.0, sv_in = 0.0;
    bool go = active;
    for (int it = 0; it < 64; ++it) {
        double num = 0.0, dd = 0.0, sv = 0.0;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const double gv = g[e] * v[e], vt = fma(-v[e], om[e], v[e]);
            const bool in = gv > zs * vt;
            num += in ? gv : 0.0;
            dd += in ? vt : 0.0;
            sv += in ? v[e] : 0.0;
        }
        num = group_sum<G>(num);
        dd = group_sum<G>(dd);
        sv = group_sum<G>(sv);
        den = dd;
        sv_in = sv;
        const double zn = num / (vt0 + dd);
        const bool more = go && (zn > zs);
        if (more) zs = zn;
        go = more;
        if (!__any_sync(0xffffffffu, go)) break;
    }
    const double U = lam / (vt0 + den);
#pragma unroll
    for (int e = 0; e < NE; ++e) yv[e] = (g[e] * v[e] > zs * fma(-v[e], om[e], v[e])) ? v[e] * U : 0.0;
    y0new = lam - U * sv_in;
}

// a5, one group: head entries into the group's private histogram, tail
// entries (and no pads: pads carry id N) into s by fp64 reductions.
// Warm head [HH, spread_n) goes to this warp's spread copy (offset spread_rel
// from s), the rest of the tail to s itself.
template <int NE>
__device__ __forceinline__ void scatter_group(const int (&idx)[NE], const double (&c)[NE], double *hg, int HH,
                                              double *s, int N, int spread_n, int spread_rel) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const int j = idx[e];
        if (j < HH) hg[j] += c[e];
        const int off = j < spread_n ? spread_rel + j : j;
        red_add_if(s + off, c[e], j >= HH && j < N);
    }
}

// Block-wide flush of the group histograms (nh of them, stride hs doubles).
__device__ __forceinline__ void flush_hists(const double *hist, int nh, int hs, int HH, int N, double *s) {
    const int lim = HH < N ? HH : N;
    for (int j = threadIdx.x; j < lim; j += blockDim.x) {
        double sum = 0.0;
        for (int h = 0; h < nh; ++h) sum += hist[h * hs + j];
        if (sum != 0.0) atomicAdd(s + j, sum);
    }
}

// group histogram stride: HH + 1 doubles, so that the same product of two
// groups falls in different banks
__host__ __device__ constexpr int hist_stride(int HH) { return HH + 1; }

// Dynamic round claims: work[0] is the claim counter of the launch, work[1]
// counts exited blocks; the last block resets both for the next launch (so
// the iteration graph needs no memset node before K1).
__device__ __forceinline__ void release_work(unsigned long long *work) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(work + 1, 1ull) == (unsigned long long)gridDim.x - 1ull) {
            work[0] = 0ull;
            work[1] = 0ull;
        }
    }
}

// Block setup: the head of g (products [0, HG)) into shared memory as one TMA
// bulk copy on its own mbarrier (thread 0 issues it; every thread waits on
// gbar after the block's setup barrier).  A strided copy loop was ~7 us of
// every launch's prologue (exp/span.py).
__device__ __forceinline__ void ghead_issue(double *ghead, const double *g, int HG, uint64_t *gbar) {
    if (threadIdx.x == 0 && HG > 0) {
        mbar_init(gbar, 1);
        fence_mbar_init();
        const uint32_t bytes = ((uint32_t)HG * 8u + 15u) & ~15u;   // g holds >= N + 2 slots
        mbar_arrive_expect_tx(gbar, bytes);
        bulk_g2s(ghead, g, bytes, gbar);
    }
}
__device__ __forceinline__ void ghead_wait(int HG, uint64_t *gbar) {
    if (HG > 0) mbar_wait(gbar, 0);
}

// ============================================================== k_primal_stream
// Full sweep over segments [first, first + count) of one bin (contiguous).
#ifndef SPFOM_SPREAD_C
#define SPFOM_SPREAD_C 8
#endif
#ifndef SPFOM_HIST_TOTAL
#define SPFOM_HIST_TOTAL 1024      // head products privatised per warp (split over its groups)
#endif
#ifndef SPFOM_SAMP_BULK
#define SPFOM_SAMP_BULK 1   // sampled rounds: 1 = one bulk copy per (row, array); 0 = 16-B cp.async over the lanes
#endif
#ifndef SPFOM_DYN_CH
#define SPFOM_DYN_CH 2   // rounds per dynamically claimed chunk (0: static contiguous partition per warp)
#endif
#ifndef SPFOM_EXTRAP
// full-sweep stream kernels: the projection's warm start is the segment's last
// multipliers (nu, kappa, U) plus their last change (linear extrapolation),
// from iteration SPFOM_EXTRAP_FROM on.  Newton passes in iterations 6-25 of
// huge (exp/warm_sim.py, a host replica of project_group on the GPU's
// iterates): 2.28 -> 2.01 per segment, 3.42 -> 2.07 per warp round (the max
// over its 8 segments, which is what a warp pays).  The projection is exact
// from any start: only the pass count changes.
#define SPFOM_EXTRAP 1
#endif
#ifndef SPFOM_EXTRAP_FROM
#define SPFOM_EXTRAP_FROM 5
#endif
#ifndef SPFOM_EXTRAP_UNTIL
#define SPFOM_EXTRAP_UNTIL 1000000000LL   // iterations >= UNTIL: no extrapolation, no history kept
#endif
#ifndef SPFOM_DYN_CH_MP
#define SPFOM_DYN_CH_MP 1   // multi-period kernel: rounds (x T periods) per dynamically claimed chunk
#endif
#ifndef SPFOM_HIST_TOTAL_E
#define SPFOM_HIST_TOTAL_E SPFOM_HIST_TOTAL   // entry-mapped layouts have a smaller slot: room for more
#endif
#ifndef SPFOM_STREAM_WARPS
#define SPFOM_STREAM_WARPS 12        // 8 entries per lane: 168 registers -> 12 warps per SM
#endif
#ifndef SPFOM_STREAM_WARPS_E
#define SPFOM_STREAM_WARPS_E 8       // entry mapping (registers: 2 warps per scheduler)
#endif
#ifndef SPFOM_STREAM_WARPS_WIDE
#define SPFOM_STREAM_WARPS_WIDE 8    // 16 entries per lane
#endif
// EQ > 0: entry mapping, EQ entries per lane for rows of at most EQ G
// entries (RQ = EQ G / 4 quads): lane l of a G-lane group takes entries l,
// l + G, l + 2 G, .. of the row (entry e = element e % 4 of quad e / 4).  With
// G = 4 that is entry l of every quad, and no lane computes on pad quads when
// the rows are EQ quads long (huge: k = 50 -> 13 quads, 19% less per-entry
// work than the (4, 4) bin); G = 8 / 16 serve rows of up to 104 / 208 entries
// with the same 13 entries per lane (medium).
// TA (sampled uniform rows, TMA gather4 into the slot): every gather4
// destination 128-B aligned -- the quad arrays start on 128 B, segc rows 4..7
// and ids rows 4..7 sit 64 B further (the compute adds the shift), and the
// inert ids move past them.
template <int G, int Q, int EQ = 0, bool TA = false>
struct StreamLayout {
    static_assert(EQ == 0 || G % 4 == 0, "entry mapping: a multiple of 4 lanes per segment");
    static constexpr int NE = EQ ? EQ : 4 * Q;         // entries per lane
    static constexpr int RQ = EQ ? EQ * G / 4 : G * Q; // quads per row, at most
    // one persistent block per SM; warps per block from the register budget
    static constexpr int WARPS = EQ ? SPFOM_STREAM_WARPS_E : ((4 * Q >= 16) ? SPFOM_STREAM_WARPS_WIDE : SPFOM_STREAM_WARPS);
    static constexpr int GPW = 32 / G;                 // segments per round (per warp)
    static constexpr int QMAX = GPW * RQ;              // quads per round, at most
    static constexpr int QW = ((GPW + 8) + 3) & ~3;    // qoff window of the next round (ints)
    static constexpr uint32_t OFF_SEGV = 0;                            // double4 x GPW
    static constexpr uint32_t OFF_SEGC = 32u * GPW;                    // double2 x GPW
    static constexpr uint32_t SHIFT = TA ? 64u : 0u;                   // segc / ids rows 4..7 (TA)
    static constexpr uint32_t OFF_QW = OFF_SEGC + 16u * GPW + SHIFT;   // int x QW
    static constexpr uint32_t OFF_SEGD = OFF_QW + 4u * QW;              // float4 x GPW (full sweep)
    // quad arrays hold QMAX + NI quads: quads QMAX .. QMAX + NI - 1 are inert
    // zero quads (id N, v = omega = y = 0) that lanes without a quad read
    // instead of branching (NI = EQ for the entry mapping on 4 lanes, so that a
    // whole row of an inactive group maps onto them with constant offsets)
    static constexpr int NI = (EQ > 0 && G == 4) ? EQ : 1;
    static constexpr uint32_t AL = TA ? 127u : 0u;
    static constexpr uint32_t OFF_V = ((OFF_SEGD + 16u * GPW) + 63u + AL) & ~(63u + AL);   // double4 x (QMAX + NI)
    static constexpr uint32_t OFF_OM = (OFF_V + 32u * (QMAX + NI) + AL) & ~AL;          // double4 x (QMAX + NI)
    static constexpr uint32_t OFF_Y = (OFF_OM + 32u * (QMAX + NI) + AL) & ~AL;          // double4 x (QMAX + NI)
    static constexpr uint32_t OFF_IDS = (OFF_Y + 32u * (QMAX + NI) + AL) & ~AL;         // int4 x (QMAX + NI) (+ SHIFT)
    static constexpr uint32_t SLOT = ((OFF_IDS + 16u * (QMAX + NI) + SHIFT) + 127u) & ~127u;
    // one head histogram per group (ids are distinct within a segment: no atomics)
    static constexpr int NHIST = GPW;
    static constexpr int HH = (EQ ? SPFOM_HIST_TOTAL_E : SPFOM_HIST_TOTAL) / NHIST;
    static constexpr uint32_t HIST = (uint32_t)NHIST * hist_stride(HH) * 8u;   // bytes per warp
    static constexpr uint32_t PER_WARP = SLOT + ((HIST + 127u) & ~127u);
};


struct StreamList {
    int64_t first, count;   // segments [first, first + count), all of one bin
    int32_t ghead;          // g staged in shared memory for products [0, ghead)
    int32_t hh;             // group histograms cover products [0, hh) (<= Layout::HH)
    unsigned long long *work;   // dynamic round chunks: counter zeroed before the launch
    int32_t uni;            // entry mapping, G = 4: every row of the bin has exactly EQ quads
    int32_t qbase;          // qoff[first] (host copy: no load on the launch's critical path)
    // sampled blocks (SAMP instantiations): this iteration's segments of the
    // bin are ids[row_off[r][bin] .. row_off[r][bin + 1]), r = t mod block_iters
    // (device slots of the bin, count = an upper bound for the grid)
    const int32_t *ids;
    const int32_t *row_off;
    int32_t bin, nbins;
    int64_t block_iters;
    // uniform bins: 6 TMA tensor maps (128 B each, global memory) over the
    // bin's rows -- ids, v, omega, y as [rows][4 EQ], segv [rows][4], segc
    // [rows][2] -- for tile::gather4 (null: per-row copies)
    const void *tm;
};

// + mbarriers; SAMP: + each warp's copy of y_old (NE x 32 lanes) for the usage delta
template <int G, int Q, int EQ = 0, bool SAMP = false, bool UNI = false>
__host__ __device__ constexpr size_t stream_smem_fixed() {
    using LY = StreamLayout<G, Q, EQ, SAMP && UNI>;
    return (size_t)LY::WARPS * LY::PER_WARP + 128 + (SAMP ? (size_t)LY::WARPS * LY::NE * 256 : 0);
}

// UNI (entry mapping on 4 lanes, every row of the bin exactly EQ quads): slot
// positions are compile-time offsets from one per-lane base (an inactive group
// of the last round points at the inert quads), so the round has no per-entry
// bounds tests at all -- a separate instantiation, so that the compiler cannot
// fold the ragged path's index arithmetic into it.
//
// SAMP (sampled blocks, "Randomly generate a subset of customers I"):
// the rounds are GPW consecutive entries of this iteration's block list of the
// bin instead of GPW consecutive device slots.  The rows are not contiguous,
// so the slot is filled by 16-B cp.async copies (each row's quads are
// contiguous: a few copies per row and array, spread over the lanes) instead
// of one bulk copy per array; the compute is the same, and the usage scatter
// adds y_new - y_old (Alg. 2's sum over [n] keeps the rows outside I_t).
template <int G, int Q, bool ARGMAX, int EQ = 0, bool UNI = false, bool SAMP = false>
__global__ void __launch_bounds__(32 * StreamLayout<G, Q, EQ>::WARPS, 1) k_primal_stream(DevState S, StreamList L) {
    SPAN_MARK(0);
    using LY = StreamLayout<G, Q, EQ, SAMP && UNI>;
    constexpr int NE = LY::NE;
    constexpr int GPW = LY::GPW;
    static_assert(NE <= 32, "class bitmasks hold at most 32 entries per lane");
    static_assert(GPW + 1 <= 32, "qoff lanes");

    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int gidx = lane / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gidx * G));
    const int N = (int)S.N;
    const int HG = L.ghead, HH = L.hh;
    constexpr int HS = hist_stride(LY::HH);
    // warm-start extrapolation (full sweep, projection): this iteration is *S.t + 1
    constexpr bool EX = SPFOM_EXTRAP && !SAMP && !ARGMAX;
    const int64_t it_ = *S.t + 1;
    const bool ex_on = EX && it_ >= SPFOM_EXTRAP_FROM && it_ < SPFOM_EXTRAP_UNTIL;   // extrapolate (segd read)
    const bool ex_rec = EX && it_ < SPFOM_EXTRAP_UNTIL;                              // keep the history (segd written)

    unsigned char *slot = smem + (size_t)warp * LY::PER_WARP;
    double *hist_all = reinterpret_cast<double *>(smem + LY::SLOT);   // warp w's hists at w * PER_WARP
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + (size_t)LY::WARPS * LY::PER_WARP) + warp;
    double *ghead = reinterpret_cast<double *>(smem + stream_smem_fixed<G, Q, EQ, SAMP, UNI>());
    double *hg = reinterpret_cast<double *>(smem + (size_t)warp * LY::PER_WARP + LY::SLOT) + gidx * HS;
    // SAMP: entry e of this lane's y_old at yo_s + 256 e (conflict-free)
    const uint32_t yo_s = smem_u32(smem + (size_t)LY::WARPS * LY::PER_WARP + 128) + (uint32_t)warp * (NE * 256u) + 8u * lane;
    (void)yo_s;
    const uint32_t ghead_s = smem_u32(ghead), hg_s = smem_u32(hg);
    const int spread_n = S.spread_n;
    const int spread_rel = S.spread_off + ((blockIdx.x * LY::WARPS + warp) % (S.spread_c > 0 ? S.spread_c : 1)) * spread_n;

    for (int e = lane; e < 4 * LY::NI; e += 32) {   // this warp's inert zero quads (past the quads the copies write)
        reinterpret_cast<double *>(slot + LY::OFF_V + 32u * LY::QMAX)[e] = 0.0;
        reinterpret_cast<double *>(slot + LY::OFF_OM + 32u * LY::QMAX)[e] = 0.0;
        reinterpret_cast<double *>(slot + LY::OFF_Y + 32u * LY::QMAX)[e] = 0.0;
        reinterpret_cast<int *>(slot + LY::OFF_IDS + 16u * LY::QMAX + LY::SHIFT)[e] = N;
    }
    if (lane == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncwarp();
    (void)hist_all;
#ifdef SPFOM_DIAG_TIME
    uint64_t t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    long long wait_cycles = 0, red_cycles = 0;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
#endif

    // Rounds of GPW consecutive segments.  SPFOM_DYN_CH > 0: warps claim
    // chunks of CH rounds from a global counter (the SMs of the two dies do
    // not run at the same speed: a static split leaves one die idle at the
    // end); the next chunk is claimed one chunk ahead, so the atomic's latency
    // is hidden.  Rounds come from a 3-deep queue q0 (current), q1 (its TMA
    // is issued during q0), q2 (q1's copy also fetches q2's offsets).
    int64_t count = L.count;
    const int32_t *sids = nullptr;
    if constexpr (SAMP) {
        const int64_t row = (*S.t) % L.block_iters;
        const int32_t *ro = L.row_off + row * (L.nbins + 1);
        const int32_t a = ro[L.bin];
        count = ro[L.bin + 1] - a;
        sids = L.ids + a;
    }
    const int32_t rounds = (int32_t)((count + GPW - 1) / GPW);
    constexpr int CH = SPFOM_DYN_CH;
    const int32_t nch = CH > 0 ? (rounds + CH - 1) / CH : 0;
    // the claimed chunk id stays in lane 0's register until the warp moves to
    // that chunk (the broadcast is the first use: the atomic's latency is
    // hidden behind the current chunk's rounds)
    auto grab = [&]() -> unsigned long long { return claim_chunk(L.work, lane); };
    auto bcast = [&](unsigned long long c) -> int32_t {
        return __shfl_sync(0xffffffffu, (int32_t)(c < 0x7fffffffull ? c : 0x7fffffffull), 0);
    };
    int32_t fpos = 0, fend = 0;
    unsigned long long fpend = 0;
    if constexpr (CH > 0) {
        fpend = grab();
    } else {
        const int64_t W = (int64_t)gridDim.x * LY::WARPS;
        const int64_t gw = (int64_t)blockIdx.x * LY::WARPS + warp;
        fpos = (int32_t)(rounds * gw / W);
        fend = (int32_t)(rounds * (gw + 1) / W);
    }
    auto fnext = [&]() -> int32_t {
        if constexpr (CH > 0) {
            if (fpos >= fend) {
                const int32_t c = bcast(fpend);
                if (c >= nch) return -1;
                fpos = c * CH;
                fend = min(fpos + CH, rounds);
                fpend = grab();
            }
        } else {
            if (fpos >= fend) return -1;
        }
        return fpos++;
    };

    // uniform entry-mapped bin: every row has EQ quads, so a segment's quad
    // offset is arithmetic (no qoff reads, no window copy per round)
    static_assert(!UNI || (EQ > 0 && G == 4), "uniform rows: entry mapping on 4 lanes");
    constexpr bool uni = UNI;
    const int32_t qbase = uni ? L.qbase : 0;
    // lane l <= GPW: qoff of segment GPW r + l of the bin (clamped to the bin end)
    auto qload = [&](int64_t r) -> int32_t {
        int64_t k = GPW * r + (lane < GPW ? lane : GPW);
        k = k < count ? k : count;
        return uni ? qbase + (int32_t)(EQ * k) : S.qoff[L.first + k];
    };
    // SAMP: lane l < GPW: device slot of round r's segment l (-1: none)
    auto sload = [&](int64_t r) -> int32_t {
        const int64_t k = GPW * r + lane;
        return (lane < GPW && k < count) ? __ldg(sids + k) : -1;
    };
    // SAMP: quad range [gq, ge) of slot sid (loads only: the first use is in issue_s)
    auto sdesc = [&](int32_t sid, int32_t &gq, int32_t &ge) {
        if (sid < 0) {
            gq = 0;
            ge = 0;
        } else if constexpr (UNI) {
            gq = qbase + EQ * (sid - (int32_t)L.first);
            ge = gq + EQ;
        } else {
            gq = __ldg(S.qoff + sid);
            ge = __ldg(S.qoff + sid + 1);
        }
    };
    // SAMP: gather round's rows into the slot: row l at local quad lq (the
    // exclusive prefix of the row lengths; EQ l for uniform rows)
    auto issue_s = [&](int32_t sid, int32_t gq, int32_t ge, int32_t &lq) {
        if constexpr (UNI) {
            if (L.tm != nullptr) {
                // uniform rows: 4 rows per TMA gather4 per array (rows past the
                // round's last are copies of its first: the compute masks them)
                lq = EQ * lane;
                const int32_t rl = sid - (int32_t)L.first;
                const int nrows = __popc(__ballot_sync(0xffffffffu, sid >= 0));
                int32_t rr[GPW];
#pragma unroll
                for (int j = 0; j < GPW; ++j) rr[j] = __shfl_sync(0xffffffffu, rl, j < nrows ? j : 0);
                if (lane == 0) {
                    constexpr uint32_t ROWB = 16u * EQ + 3u * 32u * EQ + 48u;   // ids, v, om, y, segv, segc
                    const int ng = (nrows + 3) >> 2;
                    mbar_arrive_expect_tx(bar, (uint32_t)ng * 4u * ROWB);
                    const uint64_t pol = l2_evict_first_policy();
                    const unsigned char *tm = reinterpret_cast<const unsigned char *>(L.tm);
                    const uint32_t sb = smem_u32(slot);
#pragma unroll
                    for (int g4 = 0; g4 < GPW / 4; ++g4) {
                        if (g4 < ng) {
                            const int32_t a = rr[4 * g4], b = rr[4 * g4 + 1], c = rr[4 * g4 + 2], d = rr[4 * g4 + 3];
                            const uint32_t r0 = 4u * g4;
                            tma_gather4(sb + LY::OFF_IDS + 16u * EQ * r0 + (g4 ? LY::SHIFT : 0u), tm + 0 * 128, a, b, c, d, bar, pol);
                            tma_gather4(sb + LY::OFF_V + 32u * EQ * r0, tm + 1 * 128, a, b, c, d, bar, pol);
                            tma_gather4(sb + LY::OFF_OM + 32u * EQ * r0, tm + 2 * 128, a, b, c, d, bar, pol);
                            tma_gather4(sb + LY::OFF_Y + 32u * EQ * r0, tm + 3 * 128, a, b, c, d, bar, pol);
                            tma_gather4(sb + LY::OFF_SEGV + 32u * r0, tm + 4 * 128, a, b, c, d, bar, pol);
                            tma_gather4(sb + LY::OFF_SEGC + 16u * r0 + (g4 ? LY::SHIFT : 0u), tm + 5 * 128, a, b, c, d, bar, pol);
                        }
                    }
                }
                return;
            }
        }
        const int32_t nq = ge - gq;
        if constexpr (UNI) {
            lq = EQ * lane;
        } else {
            int32_t inc = nq;
#pragma unroll
            for (int d = 1; d < GPW; d <<= 1) {
                const int32_t t = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += t;
            }
            lq = inc - nq;
        }
#if SPFOM_SAMP_BULK
        // one bulk copy per (row, array), issued by the row's lane; lane 0
        // arms the barrier with the round's bytes first
        const int32_t totq = __shfl_sync(0xffffffffu, lq + nq, GPW - 1);
        const uint32_t nrows = (uint32_t)__popc(__ballot_sync(0xffffffffu, sid >= 0));
        if (lane == 0) mbar_arrive_expect_tx(bar, 48u * nrows + 112u * (uint32_t)totq);
        __syncwarp();
        if (sid >= 0) {
            const uint32_t rsh = lane >= 4 ? LY::SHIFT : 0u;     // TA layout: rows 4..7 of segc / ids
            bulk_g2s(slot + LY::OFF_SEGV + 32u * lane, S.segv + sid, 32u, bar);
            bulk_g2s(slot + LY::OFF_SEGC + 16u * lane + rsh, S.segc + sid, 16u, bar);
            if (nq > 0) {
                const uint64_t pol = l2_evict_first_policy();
                bulk_g2s_hint(slot + LY::OFF_IDS + 16u * lq + rsh, S.pidx + gq, 16u * nq, bar, pol);
                bulk_g2s_hint(slot + LY::OFF_V + 32u * lq, S.v + 4 * (int64_t)gq, 32u * nq, bar, pol);
                bulk_g2s_hint(slot + LY::OFF_OM + 32u * lq, S.om + 4 * (int64_t)gq, 32u * nq, bar, pol);
                bulk_g2s_hint(slot + LY::OFF_Y + 32u * lq, S.y + 4 * (int64_t)gq, 32u * nq, bar, pol);
            }
        }
#else
        const uint32_t sb = smem_u32(slot);
        if (sid >= 0) {
            const double *sv = reinterpret_cast<const double *>(S.segv + sid);
            cp16_g2s(sb + LY::OFF_SEGV + 32u * lane, sv);
            cp16_g2s(sb + LY::OFF_SEGV + 32u * lane + 16u, sv + 2);
            cp16_g2s(sb + LY::OFF_SEGC + 16u * lane + (lane >= 4 ? LY::SHIFT : 0u), S.segc + sid);
        }
#pragma unroll 1
        for (int j = 0; j < GPW; ++j) {
            const int32_t gj = __shfl_sync(0xffffffffu, gq, j);
            const int32_t nj = __shfl_sync(0xffffffffu, nq, j);
            const int32_t lj = __shfl_sync(0xffffffffu, lq, j);
            if (nj == 0) continue;         // empty row (k = 0) or no row
            SPFOM_DCHECK(S, nj <= LY::RQ && lj + nj <= LY::QMAX && gj >= 0 && (int64_t)gj + nj <= S.nq);
            for (int c = lane; c < nj; c += 32)
                cp16_g2s(sb + LY::OFF_IDS + 16u * (uint32_t)(lj + c) + (j >= 4 ? LY::SHIFT : 0u), S.pidx + gj + c);
            for (int c = lane; c < 2 * nj; c += 32) {
                const int64_t o = 4 * (int64_t)gj + 2 * c;
                const uint32_t d = 32u * (uint32_t)lj + 16u * (uint32_t)c;
                cp16_g2s(sb + LY::OFF_V + d, S.v + o);
                cp16_g2s(sb + LY::OFF_OM + d, S.om + o);
                cp16_g2s(sb + LY::OFF_Y + d, S.y + o);
            }
        }
        cp_commit();
#endif
    };
    // lane 0 issues the bulk copies of round r (q: this lane's qoff of round r):
    // segment state, quads, and (rw >= 0) the 16-B aligned qoff window that
    // holds round rw's offsets
    auto issue = [&](int64_t r, int32_t q, int64_t rw) {
        const int32_t qa = __shfl_sync(0xffffffffu, q, 0), qb = __shfl_sync(0xffffffffu, q, GPW);
        const int64_t s0 = L.first + GPW * r;
        const int64_t left = count - GPW * r;
        const uint32_t n = (uint32_t)(left < GPW ? left : GPW);
        const uint32_t nq = (uint32_t)(qb - qa);
        const int64_t w0 = (L.first + GPW * rw) & ~(int64_t)3;        // window of round rw
        SPFOM_DCHECK(S, qb >= qa && nq <= (uint32_t)LY::QMAX && qa >= 0 && (int64_t)qb <= S.nq * S.T);
        SPFOM_DCHECK(S, left > 0 && s0 + n <= S.m);
        const uint32_t wbytes = (rw >= 0 && !uni) ? 4u * LY::QW : 0u;
        // one elected lane, straight-line: the copies take uniform operands
        if (lane == 0) {
            mbar_arrive_expect_tx(bar, (ex_on ? 64u : 48u) * n + 112u * nq + wbytes);
            bulk_g2s(slot + LY::OFF_SEGV, S.segv + s0, 32u * n, bar);
            bulk_g2s(slot + LY::OFF_SEGC, S.segc + s0, 16u * n, bar);
            if (ex_on) bulk_g2s(slot + LY::OFF_SEGD, S.segd + s0, 16u * n, bar);
            if (wbytes) bulk_g2s(slot + LY::OFF_QW, S.qoff + w0, wbytes, bar);
            if (nq > 0) {
                const uint64_t pol = l2_evict_first_policy();
                bulk_g2s_hint(slot + LY::OFF_IDS, S.pidx + qa, 16u * nq, bar, pol);
                bulk_g2s_hint(slot + LY::OFF_V, S.v + 4 * (int64_t)qa, 32u * nq, bar, pol);
                bulk_g2s_hint(slot + LY::OFF_OM, S.om + 4 * (int64_t)qa, 32u * nq, bar, pol);
                bulk_g2s_hint(slot + LY::OFF_Y, S.y + 4 * (int64_t)qa, 32u * nq, bar, pol);
            }
        }
    };


    ProjStats st;
    int32_t qc = 0;
    int32_t q0 = fnext(), q1 = fnext(), q2 = fnext();
    // SAMP: per lane (< GPW), round q0: slot ss0, quads [sg0, se0), local sl0;
    // round q1: ss1, [sg1, se1), sl1; round q2: ss2
    int32_t ss0 = -1, sg0 = 0, se0 = 0, sl0 = 0, ss1 = -1, sg1 = 0, se1 = 0, sl1 = 0, ss2 = -1;
    if constexpr (SAMP) {
        if (q0 >= 0) {
            ss0 = sload(q0);
            sdesc(ss0, sg0, se0);
            issue_s(ss0, sg0, se0, sl0);
        }
        if (q1 >= 0) ss1 = sload(q1);
    } else if (q0 >= 0) {
        qc = qload(q0);
        issue(q0, qc, q1);
    }
    // block setup while the first round is in flight: the head of g and
    // zeroed group histograms
    uint64_t *gbar = reinterpret_cast<uint64_t *>(smem + (size_t)LY::WARPS * LY::PER_WARP) + LY::WARPS;
    ghead_issue(ghead, S.g, HG, gbar);
    for (int w = 0; w < LY::WARPS; ++w) {
        double *h = reinterpret_cast<double *>(smem + (size_t)w * LY::PER_WARP + LY::SLOT);
        for (int j = threadIdx.x; j < LY::NHIST * HS; j += blockDim.x) h[j] = 0.0;
    }
    __syncthreads();
    ghead_wait(HG, gbar);
    SPAN_MARK(1);
#ifdef SPFOM_DIAG_TIME
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    uint32_t phase = 0;
#ifdef SPFOM_DIAG_PHASE
    long long ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long ph_t = clock64();
#endif
    for (; q0 >= 0; q0 = q1, q1 = q2, q2 = fnext(), phase ^= 1u) {
        const int64_t r = q0;
        PH_MARK(7);
#ifdef SPFOM_DIAG_TIME
        const long long tw0 = clock64();
#endif
        if (SAMP && !SPFOM_SAMP_BULK && !(UNI && L.tm != nullptr)) {
            cp_wait_all();
            __syncwarp();
        } else {
            mbar_wait(bar, phase);
        }
#ifdef SPFOM_DIAG_TIME
        wait_cycles += clock64() - tw0;
        const long long tr0 = clock64();
#endif
        PH_MARK(0);
        if constexpr (SAMP) {
            // ids of round q2 and the quad ranges of round q1 (used by issue_s)
            ss2 = q2 >= 0 ? sload(q2) : -1;
            sdesc(ss1, sg1, se1);
        }
        // round q1's offsets from the window that arrived with this round
        int32_t qn = 0;
        if (!SAMP && q1 >= 0) {
            const int64_t s1 = L.first + GPW * (int64_t)q1;
            int64_t k = GPW * (int64_t)q1 + (lane < GPW ? lane : GPW);
            k = k < count ? k : count;
            qn = uni ? qbase + (int32_t)(EQ * k)
                     : reinterpret_cast<const int32_t *>(slot + LY::OFF_QW)[L.first + k - (s1 & ~(int64_t)3)];
        }
        int32_t base, qa, qb;
        int64_t i;
        if constexpr (SAMP) {
            // group gidx: row ss0 of lane gidx, global quads [qa, qb), local from qa - base
            qa = __shfl_sync(0xffffffffu, sg0, gidx);
            qb = __shfl_sync(0xffffffffu, se0, gidx);
            base = qa - __shfl_sync(0xffffffffu, sl0, gidx);
            i = __shfl_sync(0xffffffffu, ss0, gidx);
        } else {
            base = __shfl_sync(0xffffffffu, qc, 0);
            qa = __shfl_sync(0xffffffffu, qc, gidx);
            qb = __shfl_sync(0xffffffffu, qc, gidx + 1);
            i = L.first + GPW * r + gidx;
        }
        const int64_t left = count - GPW * r;
        const bool active = gidx < left;

        // ---- segment state and this lane's quads, from the slot
        double lam = 1.0, vt0 = 1.0;
        double4 sv = make_double4(1.0, 0.0, 0.0, 1.0);
        float4 sd = make_float4(0.f, 0.f, 0.f, 0.f);
        if (active) {
            sv = reinterpret_cast<const double4 *>(slot + LY::OFF_SEGV)[gidx];
            if (ex_on) sd = reinterpret_cast<const float4 *>(slot + LY::OFF_SEGD)[gidx];
            const double2 sc = *reinterpret_cast<const double2 *>(slot + LY::OFF_SEGC + 16u * gidx + (gidx >= 4 ? LY::SHIFT : 0u));
            lam = sc.x;
            vt0 = sc.y;
        }
        const double z0 = sv.x;
        int idx[NE];
        double v[NE], om[NE], z[NE];
        double gpre[EQ > 0 ? NE : 1];
        if constexpr (EQ > 0) {
            // entry mapping: entry gl of quads qa, qa + 1, .. of the row.  The
            // ids first and the price gather right away (a2), so the L2 reads
            // of the tail prices are in flight while v, omega and y are read
            int pos[NE];
            if constexpr (UNI) {
                // uniform rows: group g's row is quads [EQ g, EQ g + EQ) of the slot; an
                // inactive group (last round) reads the EQ inert quads instead
                const int pb = 4 * (active ? EQ * gidx : LY::QMAX) + gl;
#pragma unroll
                for (int t = 0; t < EQ; ++t) pos[t] = pb + 4 * t;
            } else {
                // entry gl + G t of the row: quad qa + gl / 4 + (G / 4) t, element gl % 4
#pragma unroll
                for (int t = 0; t < EQ; ++t) {
                    const int32_t q = qa + gl / 4 + (G / 4) * t;
                    pos[t] = 4 * (q < qb ? q - base : LY::QMAX) + (gl & 3);   // no quad: the inert zero quad
                }
            }
            // TA layout: ids of rows 4..7 and the inert ids sit SHIFT bytes further
            const int ish = (LY::SHIFT != 0 && (gidx >= 4 || !active)) ? (int)(LY::SHIFT / 4) : 0;
#pragma unroll
            for (int t = 0; t < EQ; ++t) idx[t] = reinterpret_cast<const int *>(slot + LY::OFF_IDS)[pos[t] + ish];
            uint32_t gh_s = ghead_s;
            const double *gglob = S.g;
            asm volatile("" : "+r"(gh_s), "+l"(gglob));
#pragma unroll
            for (int t = 0; t < EQ; ++t) {
                const int j = idx[t];
                gpre[t] = (j < HG) ? lds_f64(gh_s + 8u * (uint32_t)j) : __ldg(gglob + j);
            }
#pragma unroll
            for (int t = 0; t < EQ; ++t) {
                v[t] = reinterpret_cast<const double *>(slot + LY::OFF_V)[pos[t]];
                om[t] = reinterpret_cast<const double *>(slot + LY::OFF_OM)[pos[t]];
                z[t] = reinterpret_cast<const double *>(slot + LY::OFF_Y)[pos[t]];
            }
        } else
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int32_t q = qa + gl + G * t;
            const int p = q < qb ? q - base : LY::QMAX;          // no quad: the inert zero quad
            const int4 id4 = reinterpret_cast<const int4 *>(slot + LY::OFF_IDS)[p];
            idx[4 * t + 0] = id4.x; idx[4 * t + 1] = id4.y; idx[4 * t + 2] = id4.z; idx[4 * t + 3] = id4.w;
            const double2 *vp = reinterpret_cast<const double2 *>(slot + LY::OFF_V) + 2 * p;
            const double2 *wp = reinterpret_cast<const double2 *>(slot + LY::OFF_OM) + 2 * p;
            const double2 *yp = reinterpret_cast<const double2 *>(slot + LY::OFF_Y) + 2 * p;
            const double2 v01 = vp[0], v23 = vp[1], w01 = wp[0], w23 = wp[1], y01 = yp[0], y23 = yp[1];
            v[4 * t + 0] = v01.x; v[4 * t + 1] = v01.y; v[4 * t + 2] = v23.x; v[4 * t + 3] = v23.y;
            om[4 * t + 0] = w01.x; om[4 * t + 1] = w01.y; om[4 * t + 2] = w23.x; om[4 * t + 3] = w23.y;
            z[4 * t + 0] = y01.x; z[4 * t + 1] = y01.y; z[4 * t + 2] = y23.x; z[4 * t + 3] = y23.y;
        }
        if constexpr (SAMP) {
#pragma unroll
            for (int e = 0; e < NE; ++e) sts_f64(yo_s + 256u * e, z[e]);   // y_old (z is y until a3)
        }
        // the slot is free: fetch round r + 1 into it while this round computes.
        // The warp barrier orders every lane's slot reads before the copy is
        // issued (the consumer-release pattern of TMA pipelines); a
        // fence.proxy.async here compiles to MEMBAR.ALL.CTA, which would also
        // wait for the previous round's global reductions to drain.
        PH_MARK(1);
        __syncwarp();
        if constexpr (SAMP) {
            if (q1 >= 0) issue_s(ss1, sg1, se1, sl1);
        } else if (q1 >= 0) {
            issue(q1, qn, q2);
        }
        PH_MARK(8);

#ifdef SPFOM_DEVICE_CHECKS
#pragma unroll
        for (int e = 0; e < NE; ++e) SPFOM_DCHECK(S, idx[e] >= 0 && idx[e] <= N);
        SPFOM_DCHECK(S, qb - qa <= LY::RQ && qa >= base && qb - base <= LY::QMAX);
#endif
        // a2: price gather (g[N] = 0 for pads; head from shared memory).  The
        // opaque copies keep the two bases in registers (otherwise ptxas
        // rebuilds the shared window base and reloads S.g for every entry).
        uint32_t gh_s = ghead_s;
        const double *gglob = S.g;
        asm volatile("" : "+r"(gh_s), "+l"(gglob));
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int j = idx[e];
            double gj;
            if constexpr (EQ > 0) gj = gpre[e];
            else gj = (j < HG) ? lds_f64(gh_s + 8u * (uint32_t)j) : __ldg(gglob + j);
            if constexpr (ARGMAX) z[e] = gj;             // theta = inf: keep g itself
            else z[e] = fma(S.theta, gj, z[e]);          // a3: z = y + theta g
        }

        double yv[NE];
        double y0new;
        double x0 = sv.y, x1 = sv.z, x2 = sv.w;
        if (EX && ex_on) {
            x0 += (double)sd.x;
            x1 += (double)sd.y;
            x2 = fmax(x2 + (double)sd.z, 0.5 * x2);
        }
        PH_MARK(1);
#ifdef SPFOM_DIAG_SKIP_PROJECT
#pragma unroll
        for (int e = 0; e < NE; ++e) yv[e] = z[e] * v[e] + om[e];
        y0new = z0;
        (void)lam; (void)vt0;
#else
        if constexpr (ARGMAX) argmax_group<G, NE>(z, v, om, lam, vt0, active, yv, y0new);
        else project_group<G, NE, (EQ > 0)>(z, v, om, z0, lam, vt0, active, gmask, S.max_newton, x0, x1, x2, yv, y0new, st);
#endif
        PH_MARK(2);

        // ---- write back (y, segment state), a5 usage scatter
        if constexpr (EQ > 0) {
            // each quad's 32-B sector is written by 4 lanes of the group
            double *yp = S.y + 4 * ((int64_t)qa + gl / 4) + (gl & 3);
            SPFOM_DCHECK(S, !active || (int64_t)qb <= S.nq);
            if constexpr (UNI) {
                if (active) {
#pragma unroll
                    for (int t = 0; t < EQ; ++t) yp[4 * t] = yv[t];
                }
            } else {
#pragma unroll
                for (int t = 0; t < EQ; ++t)
                    if (qa + gl / 4 + (G / 4) * t < qb) yp[G * t] = yv[t];
            }
        } else
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int32_t q = qa + gl + G * t;
            if (q < qb) st256_stream(S.y + 4 * (int64_t)q, yv[4 * t], yv[4 * t + 1], yv[4 * t + 2], yv[4 * t + 3]);
        }
        if (active && gl == 0) {
            st256(reinterpret_cast<double *>(S.segv + i), y0new, x0, x1, x2);
            if (ex_rec) S.segd[i] = make_float4((float)(x0 - sv.y), (float)(x1 - sv.z), (float)(x2 - sv.w), 0.f);
        }
        if constexpr (SAMP) {
#pragma unroll
            for (int e = 0; e < NE; ++e) yv[e] -= lds_f64_v(yo_s + 256u * e);   // a5 delta: y_new - y_old
        }
        PH_MARK(3);
#ifdef SPFOM_DIAG_TIME
        const long long ts0 = clock64();
#endif
        // a5: head -> histogram, warm head -> spread copies, tail -> s
        // ids are distinct within a segment and every group has its own
        // histogram: all loads first, then all stores (no serial RMW chain)
#if !defined(SPFOM_DIAG_SEP_USAGE) || defined(SPFOM_DIAG_SEP_DUMMY)
        {
            double hv[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) hv[e] = idx[e] < HH ? lds_f64_v(hg_s + 8u * (uint32_t)idx[e]) : 0.0;
#pragma unroll
            for (int e = 0; e < NE; ++e)
                if (idx[e] < HH) sts_f64(hg_s + 8u * (uint32_t)idx[e], hv[e] + yv[e]);
        }
#endif
        PH_MARK(4);
#if !defined(SPFOM_DIAG_SKIP_RED) && (!defined(SPFOM_DIAG_SEP_USAGE) || defined(SPFOM_DIAG_SEP_DUMMY))
#ifndef SPFOM_DIAG_RED_FROM
#define SPFOM_DIAG_RED_FROM HH
#endif
        // entries with y = 0 (products not sold to the segment: ~38% of them in
        // the first iterations on huge, ~0 near the optimum) add nothing
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int j = idx[e];
            const int off = j < spread_n ? spread_rel + j : j;     // warm head -> this warp's spread copy
            SPFOM_DCHECK(S, off >= 0 && off < S.spread_off + S.spread_c * spread_n);
            red_add_if(S.s + off, yv[e], j >= SPFOM_DIAG_RED_FROM && j < N && yv[e] != 0.0);
        }
#endif
#ifdef SPFOM_DIAG_TIME
        red_cycles += clock64() - ts0;
        (void)tr0;
#endif
        qc = qn;
        if constexpr (SAMP) {
            ss0 = ss1; sg0 = sg1; se0 = se1; sl0 = sl1;
            ss1 = ss2;
        }
        PH_MARK(5);
#ifdef SPFOM_DIAG_PHASE
        ph[6] += 1;
#endif
    }
#ifdef SPFOM_DIAG_PHASE
    if (lane == 0)
        for (int k = 0; k < 10; ++k) atomicAdd(&g_diag_phase[k], (unsigned long long)ph[k]);
#endif
    if (lane == 0) SPAN_MARK(2);
#ifdef SPFOM_DIAG_TIME
    if (lane == 0) {
        g_diag_loops[4 * (blockIdx.x * LY::WARPS + warp)] = (uint32_t)(wait_cycles >> 10);
        g_diag_loops[4 * (blockIdx.x * LY::WARPS + warp) + 1] = (uint32_t)(red_cycles >> 10);
        g_diag_loops[4 * (blockIdx.x * LY::WARPS + warp) + 2] = smid;
        uint64_t t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        g_diag_time[2 * (blockIdx.x * LY::WARPS + warp)] = t_start;
        g_diag_time[2 * (blockIdx.x * LY::WARPS + warp) + 1] = t_end;
    }
#endif
    if constexpr (!ARGMAX) {
        if (st.passes) {
            atomicAdd(S.counters + 1, st.passes);
            if (st.failures) atomicAdd(S.counters + 0, st.failures);
            if (st.restarts) atomicAdd(S.counters + 2, st.restarts);
        }
    }
    if constexpr (CH > 0) release_work(L.work);
    __syncthreads();
    // flush: histogram h of warp w lives at w * PER_WARP + SLOT + h * HS
    {
        const int lim = HH < N ? HH : N;
        for (int j = threadIdx.x; j < lim; j += blockDim.x) {
            double sum = 0.0;
            for (int w = 0; w < LY::WARPS; ++w) {
                const double *h = reinterpret_cast<const double *>(smem + (size_t)w * LY::PER_WARP + LY::SLOT);
#pragma unroll
                for (int g2 = 0; g2 < LY::NHIST; ++g2) sum += h[g2 * HS + j];
            }
            if (sum != 0.0) atomicAdd(S.s + j, sum);
        }
    }
    SPAN_MARK(3);
}

// ============================================================== k_primal_mp
// Multi-period shared structure (reading c15; SURVEY §8(a) layout contract):
// segment (t, i) shares C_i, v_i. and omega_i. with every period; only
// lambda_{i,t}, y_{.,t}, y0 and the warm start are per period.  The work unit
// is (round r, period t); units in round-major order are split evenly over the
// warps.  A warp loads a round's structure (ids, v, omega) once, stages
// theta g once, then projects each of its periods of that round; the per-entry
// usage sum_t y_ijt accumulates in shared memory and is scattered once per
// round, so the structure bytes, the gather and the scatter are T times rarer
// than in the stacked layout.  Two TMA slots per warp: the structure of round
// r + 1 and the per-period data of the next unit are fetched while the current
// unit computes.
template <int G, int Q, int EQ = 0>
struct MPLayout {
    static_assert(EQ == 0 || G == 4, "entry mapping: 4 lanes per segment");
    static constexpr int WARPS = (EQ > 0 || 4 * Q >= 16) ? SPFOM_STREAM_WARPS_WIDE : SPFOM_STREAM_WARPS;
    static constexpr int GPW = 32 / G;
    static constexpr int NE = EQ ? EQ : 4 * Q;          // entries per lane (EQ: entry mapping, as K1 stream)
    static constexpr int QMAX = GPW * (EQ ? EQ : G * Q);
    static constexpr int QW = ((GPW + 8) + 3) & ~3;
    // structure slot (index QMAX of each quad array: inert zero quad)
    static constexpr uint32_t S_QW = 0;
    static constexpr uint32_t S_V = ((4u * QW) + 63u) & ~63u;
    static constexpr uint32_t S_OM = S_V + 32u * (QMAX + 1);
    static constexpr uint32_t S_IDS = S_OM + 32u * (QMAX + 1);
    static constexpr uint32_t S_END = ((S_IDS + 16u * (QMAX + 1)) + 127u) & ~127u;
    // period slot
    static constexpr uint32_t P_SEGV = S_END;                              // double4 x GPW
    static constexpr uint32_t P_SEGC = P_SEGV + 32u * GPW;                 // double2 x GPW
    static constexpr uint32_t P_SEGD = P_SEGC + 16u * GPW;                 // float4 x GPW (warm-start change)
    static constexpr uint32_t P_Y = ((P_SEGD + 16u * GPW) + 63u) & ~63u;   // double4 x (QMAX + 1)
    static constexpr uint32_t P_END = ((P_Y + 32u * (QMAX + 1)) + 127u) & ~127u;
    // per-lane theta g and usage accumulators, [NE][32 lanes] doubles
    static constexpr uint32_t GT = P_END;
    static constexpr uint32_t YS = GT + 256u * NE;
    static constexpr uint32_t PER_WARP = YS + 256u * NE;
};

template <int G, int Q, int EQ = 0>
__host__ __device__ constexpr size_t mp_smem_fixed() {
    return (size_t)MPLayout<G, Q, EQ>::WARPS * MPLayout<G, Q, EQ>::PER_WARP + 256;   // + 2 mbarriers per warp
}

template <int G, int Q, bool ARGMAX, int EQ = 0>
__global__ void __launch_bounds__(32 * MPLayout<G, Q, EQ>::WARPS, 1) k_primal_mp(DevState S, StreamList L) {
    // warm-start extrapolation (SPFOM_EXTRAP): this iteration is *S.t + 1
#ifndef SPFOM_EXTRAP_MP
#define SPFOM_EXTRAP_MP 1
#endif
    constexpr bool EX = SPFOM_EXTRAP && SPFOM_EXTRAP_MP && !ARGMAX;
    const int64_t it_ = *S.t + 1;
    const bool ex_on = EX && it_ >= SPFOM_EXTRAP_FROM && it_ < SPFOM_EXTRAP_UNTIL;   // extrapolate (segd read)
    const bool ex_rec = EX && it_ < SPFOM_EXTRAP_UNTIL;                              // keep the history (segd written)
    using LY = MPLayout<G, Q, EQ>;
    constexpr int NE = LY::NE;
    constexpr int GPW = LY::GPW;
    static_assert(NE <= 32, "class bitmasks hold at most 32 entries per lane");

    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int gidx = lane / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gidx * G));
    const int N = (int)S.N;
    const int HG = L.ghead;
    const int64_t T = S.T, nqb = S.nq, mb = S.m;

    unsigned char *ws = smem + (size_t)warp * LY::PER_WARP;
    uint64_t *barS = reinterpret_cast<uint64_t *>(smem + (size_t)LY::WARPS * LY::PER_WARP) + 2 * warp;
    uint64_t *barP = barS + 1;
    double *ghead = reinterpret_cast<double *>(smem + mp_smem_fixed<G, Q, EQ>());
    const uint32_t ghead_s = smem_u32(ghead);
    const uint32_t gt_s = smem_u32(ws + LY::GT) + 8u * lane, ys_s = smem_u32(ws + LY::YS) + 8u * lane;
    const int spread_n = S.spread_n;
    const int spread_rel = S.spread_off + ((blockIdx.x * LY::WARPS + warp) % (S.spread_c > 0 ? S.spread_c : 1)) * spread_n;

    uint64_t *gbar = reinterpret_cast<uint64_t *>(smem + (size_t)LY::WARPS * LY::PER_WARP) + 2 * LY::WARPS;
    ghead_issue(ghead, S.g, HG, gbar);
    if (lane < 4) {   // inert zero quads
        reinterpret_cast<double *>(ws + LY::S_V + 32u * LY::QMAX)[lane] = 0.0;
        reinterpret_cast<double *>(ws + LY::S_OM + 32u * LY::QMAX)[lane] = 0.0;
        reinterpret_cast<int *>(ws + LY::S_IDS + 16u * LY::QMAX)[lane] = N;
        reinterpret_cast<double *>(ws + LY::P_Y + 32u * LY::QMAX)[lane] = 0.0;
    }
    if (lane == 0) {
        mbar_init(barS, 1);
        mbar_init(barP, 1);
        fence_mbar_init();
    }
    __syncthreads();
    ghead_wait(HG, gbar);

    // Whole rounds (all T periods of GPW base segments) per claim: warps take
    // rounds from a global counter (SPFOM_DYN_CH_MP > 0; see k_primal_stream)
    // or a static contiguous split; q0 / q1 / q2 as in k_primal_stream.
    const int32_t rounds = (int32_t)((L.count + GPW - 1) / GPW);
    constexpr int CH = SPFOM_DYN_CH_MP;
    const int32_t nch = CH > 0 ? (rounds + CH - 1) / CH : 0;
    auto grab = [&]() -> unsigned long long { return claim_chunk(L.work, lane); };
    auto bcast = [&](unsigned long long c) -> int32_t {
        return __shfl_sync(0xffffffffu, (int32_t)(c < 0x7fffffffull ? c : 0x7fffffffull), 0);
    };
    int32_t fpos = 0, fend = 0;
    unsigned long long fpend = 0;
    if constexpr (CH > 0) {
        fpend = grab();
    } else {
        const int64_t W = (int64_t)gridDim.x * LY::WARPS;
        const int64_t gw = (int64_t)blockIdx.x * LY::WARPS + warp;
        fpos = (int32_t)(rounds * gw / W);
        fend = (int32_t)(rounds * (gw + 1) / W);
    }
    auto fnext = [&]() -> int32_t {
        if constexpr (CH > 0) {
            if (fpos >= fend) {
                const int32_t c = bcast(fpend);
                if (c >= nch) return -1;
                fpos = c * CH;
                fend = min(fpos + CH, rounds);
                fpend = grab();
            }
        } else {
            if (fpos >= fend) return -1;
        }
        return fpos++;
    };

    auto qload = [&](int64_t r) -> int32_t {
        int64_t k = GPW * r + (lane < GPW ? lane : GPW);
        k = k < L.count ? k : L.count;
        return S.qoff[L.first + k];
    };
    // structure of round r (+ the qoff window of round rw >= 0)
    auto issueS = [&](int64_t r, int32_t q, int64_t rw) {
        const int32_t qa = __shfl_sync(0xffffffffu, q, 0), qb = __shfl_sync(0xffffffffu, q, GPW);
        const uint32_t nq = (uint32_t)(qb - qa);
        const int64_t w0 = (L.first + GPW * rw) & ~(int64_t)3;
        SPFOM_DCHECK(S, qb >= qa && nq <= (uint32_t)LY::QMAX && (int64_t)qb <= S.nq);
        const uint32_t wbytes = rw >= 0 ? 4u * LY::QW : 0u;
        if (lane == 0) {
            mbar_arrive_expect_tx(barS, 80u * nq + wbytes);
            if (wbytes) bulk_g2s(ws + LY::S_QW, S.qoff + w0, wbytes, barS);
            if (nq > 0) {
                bulk_g2s(ws + LY::S_IDS, S.pidx + qa, 16u * nq, barS);
                bulk_g2s(ws + LY::S_V, S.v + 4 * (int64_t)qa, 32u * nq, barS);
                bulk_g2s(ws + LY::S_OM, S.om + 4 * (int64_t)qa, 32u * nq, barS);
            }
        }
    };
    // period t of round r: segment state and y_t
    auto issueP = [&](int64_t r, int64_t t, int32_t q) {
        const int32_t qa = __shfl_sync(0xffffffffu, q, 0), qb = __shfl_sync(0xffffffffu, q, GPW);
        const int64_t s0 = L.first + GPW * r;
        const int64_t left = L.count - GPW * r;
        const uint32_t n = (uint32_t)(left < GPW ? left : GPW);
        const uint32_t nq = (uint32_t)(qb - qa);
        if (lane == 0) {
            mbar_arrive_expect_tx(barP, (ex_on ? 64u : 48u) * n + 32u * nq);
            bulk_g2s(ws + LY::P_SEGV, S.segv + t * mb + s0, 32u * n, barP);
            bulk_g2s(ws + LY::P_SEGC, S.segc + t * mb + s0, 16u * n, barP);
            if (ex_on) bulk_g2s(ws + LY::P_SEGD, S.segd + t * mb + s0, 16u * n, barP);
            if (nq > 0) bulk_g2s(ws + LY::P_Y, S.y + 4 * (t * nqb + qa), 32u * nq, barP);
        }
    };

    ProjStats st;
    int32_t qc = 0, qn = 0;
    int32_t q0 = fnext(), q1 = fnext(), q2 = fnext();
    if (q0 >= 0) {
        qc = qload(q0);
        issueS(q0, qc, q1);
        issueP(q0, 0, qc);
    }
    uint32_t phS = 0, phP = 0;
    int idx[NE];
    double v[NE], om[NE];
    for (; q0 >= 0; q0 = q1, q1 = q2, q2 = fnext()) {
        const int64_t r = q0;
        // ---- new round: structure into registers, theta g into shared memory
        mbar_wait(barS, phS);
        phS ^= 1u;
        qn = 0;
        if (q1 >= 0) {
            const int64_t s1 = L.first + GPW * (int64_t)q1;
            int64_t k = GPW * (int64_t)q1 + (lane < GPW ? lane : GPW);
            k = k < L.count ? k : L.count;
            qn = reinterpret_cast<const int32_t *>(ws + LY::S_QW)[L.first + k - (s1 & ~(int64_t)3)];
        }
        const int32_t base = __shfl_sync(0xffffffffu, qc, 0);
        const int32_t qa = __shfl_sync(0xffffffffu, qc, gidx);
        const int32_t qb = __shfl_sync(0xffffffffu, qc, gidx + 1);
        int epos[EQ > 0 ? NE : 1];                     // entry mapping: slot entry of each of this lane's entries
        if constexpr (EQ > 0) {
#pragma unroll
            for (int t = 0; t < EQ; ++t) {
                const int32_t q = qa + t;
                epos[t] = 4 * (q < qb ? q - base : LY::QMAX) + gl;
                idx[t] = reinterpret_cast<const int *>(ws + LY::S_IDS)[epos[t]];
                v[t] = reinterpret_cast<const double *>(ws + LY::S_V)[epos[t]];
                om[t] = reinterpret_cast<const double *>(ws + LY::S_OM)[epos[t]];
            }
        } else
#pragma unroll
        for (int tq = 0; tq < Q; ++tq) {
            const int32_t q = qa + gl + G * tq;
            const int p = q < qb ? q - base : LY::QMAX;
            const int4 id4 = reinterpret_cast<const int4 *>(ws + LY::S_IDS)[p];
            idx[4 * tq + 0] = id4.x; idx[4 * tq + 1] = id4.y; idx[4 * tq + 2] = id4.z; idx[4 * tq + 3] = id4.w;
            const double2 *vp = reinterpret_cast<const double2 *>(ws + LY::S_V) + 2 * p;
            const double2 *wp = reinterpret_cast<const double2 *>(ws + LY::S_OM) + 2 * p;
            const double2 v01 = vp[0], v23 = vp[1], w01 = wp[0], w23 = wp[1];
            v[4 * tq + 0] = v01.x; v[4 * tq + 1] = v01.y; v[4 * tq + 2] = v23.x; v[4 * tq + 3] = v23.y;
            om[4 * tq + 0] = w01.x; om[4 * tq + 1] = w01.y; om[4 * tq + 2] = w23.x; om[4 * tq + 3] = w23.y;
        }
        __syncwarp();                                  // slot reads before the copy (see k_primal_stream)
        if (q1 >= 0) issueS(q1, qn, q2);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int j = idx[e];
            const double gj = (j < HG) ? lds_f64(ghead_s + 8u * (uint32_t)j) : __ldg(S.g + j);
            sts_f64(gt_s + 256u * e, ARGMAX ? gj : S.theta * gj);   // a2 (+ the theta of a3)
            sts_f64(ys_s + 256u * e, 0.0);
        }
        const int64_t left = L.count - GPW * r;
        const bool active = gidx < left;
        const int64_t i = L.first + GPW * r + gidx;      // device base slot
        for (int64_t t = 0; t < T; ++t) {
            // ---- period t of round r
            mbar_wait(barP, phP);
            phP ^= 1u;
            double lam = 1.0, vt0 = 1.0;
            double4 sv = make_double4(1.0, 0.0, 0.0, 1.0);
            float4 sd = make_float4(0.f, 0.f, 0.f, 0.f);
            if (active) {
                sv = reinterpret_cast<const double4 *>(ws + LY::P_SEGV)[gidx];
                if (ex_on) sd = reinterpret_cast<const float4 *>(ws + LY::P_SEGD)[gidx];
                const double2 sc = reinterpret_cast<const double2 *>(ws + LY::P_SEGC)[gidx];
                lam = sc.x;
                vt0 = sc.y;
            }
            double z[NE];
            if constexpr (EQ > 0) {
#pragma unroll
                for (int t = 0; t < EQ; ++t) z[t] = reinterpret_cast<const double *>(ws + LY::P_Y)[epos[t]];
            } else
#pragma unroll
            for (int tq = 0; tq < Q; ++tq) {
                const int32_t q = qa + gl + G * tq;
                const int p = q < qb ? q - base : LY::QMAX;
                const double2 *yp = reinterpret_cast<const double2 *>(ws + LY::P_Y) + 2 * p;
                const double2 y01 = yp[0], y23 = yp[1];
                z[4 * tq + 0] = y01.x; z[4 * tq + 1] = y01.y; z[4 * tq + 2] = y23.x; z[4 * tq + 3] = y23.y;
            }
            __syncwarp();
            if (t + 1 < T) issueP(r, t + 1, qc);
            else if (q1 >= 0) issueP(q1, 0, qn);
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const double gt = lds_f64_v(gt_s + 256u * e);
                z[e] = ARGMAX ? gt : z[e] + gt;                  // a3: z = y + theta g
            }
            double yv[NE];
            double y0new;
            double x0 = sv.y, x1 = sv.z, x2 = sv.w;
            if (EX && ex_on) {      // warm start extrapolated along the last change (SPFOM_EXTRAP)
                x0 += (double)sd.x;
                x1 += (double)sd.y;
                x2 = fmax(x2 + (double)sd.z, 0.5 * x2);
            }
            if constexpr (ARGMAX) argmax_group<G, NE>(z, v, om, lam, vt0, active, yv, y0new);
            else project_group<G, NE>(z, v, om, sv.x, lam, vt0, active, gmask, S.max_newton, x0, x1, x2, yv, y0new, st);

            // ---- write back y_t and the segment state; accumulate sum_t y
            if constexpr (EQ > 0) {
#pragma unroll
                for (int tt = 0; tt < EQ; ++tt)
                    if (qa + tt < qb) S.y[4 * (t * nqb + qa + tt) + gl] = yv[tt];
            } else
#pragma unroll
            for (int tq = 0; tq < Q; ++tq) {
                const int32_t q = qa + gl + G * tq;
                if (q < qb)
                    st256(S.y + 4 * (t * nqb + q), yv[4 * tq], yv[4 * tq + 1], yv[4 * tq + 2], yv[4 * tq + 3]);
            }
            if (active && gl == 0) {
                st256(reinterpret_cast<double *>(S.segv + t * mb + i), y0new, x0, x1, x2);
                if (ex_rec) S.segd[t * mb + i] = make_float4((float)(x0 - sv.y), (float)(x1 - sv.z), (float)(x2 - sv.w), 0.f);
            }
            {
                double hv[NE];                                 // loads first: no serial RMW chain
#pragma unroll
                for (int e = 0; e < NE; ++e) hv[e] = lds_f64_v(ys_s + 256u * e);
#pragma unroll
                for (int e = 0; e < NE; ++e) sts_f64(ys_s + 256u * e, hv[e] + yv[e]);
            }
        }
        // ---- end of round r: a5 scatter of sum_t y
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int j = idx[e];
            const int off = j < spread_n ? spread_rel + j : j;
            red_add_if(S.s + off, lds_f64_v(ys_s + 256u * e), j < N);
        }
        qc = qn;
    }
    if constexpr (!ARGMAX) {
        if (st.passes) {
            atomicAdd(S.counters + 1, st.passes);
            if (st.failures) atomicAdd(S.counters + 0, st.failures);
            if (st.restarts) atomicAdd(S.counters + 2, st.restarts);
        }
    }
    if constexpr (CH > 0) release_work(L.work);
}

// ============================================================== k_primal (lists)
// Segments from a list (sampled blocks) or long-row bins: register-direct loads.
template <int Q, int G>
struct ListSmem {
    static constexpr int WARPS = kPrimalThreads / 32;
    static constexpr int GPW = 32 / G;
    static constexpr int HH = 1024 / GPW;
    double hist[WARPS * GPW * hist_stride(HH)];   // group histograms of the head products
    double ghead[kHeadMax];                       // price vector g on the head products
};

// 16+ entries per lane: trade resident blocks for registers (no spills)
template <int Q>
constexpr int list_min_blocks() { return Q >= 4 ? 1 : kPrimalMinBlocks; }

template <int G, int Q, bool ARGMAX, bool SAMPLED>
__global__ void __launch_bounds__(kPrimalThreads, list_min_blocks<Q>()) k_primal(DevState S, SegList L) {
    using SM = ListSmem<Q, G>;
    constexpr int NE = 4 * Q;               // entries per lane
    constexpr int GPW = 32 / G;             // segments per warp
    constexpr int WARPS = kPrimalThreads / 32;
    constexpr int HS = hist_stride(SM::HH);
    static_assert(NE <= 32, "class bitmasks hold at most 32 entries per lane");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    SM &sm = *reinterpret_cast<SM *>(smem_raw);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int gidx = lane / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gidx * G));
    const int N = (int)S.N;
    const int H = L.head;                    // ghead and histogram coverage
    const int HH = H < SM::HH ? H : SM::HH;

    for (int j = threadIdx.x; j < H; j += kPrimalThreads) sm.ghead[j] = S.g[j];
    for (int j = threadIdx.x; j < WARPS * GPW * HS; j += kPrimalThreads) sm.hist[j] = 0.0;
    __syncthreads();
    double *hg = sm.hist + (warp * GPW + gidx) * HS;
    const int spread_n = S.spread_n;
    const int spread_rel = S.spread_off +
        (int)((((int64_t)blockIdx.x * WARPS + warp)) % (S.spread_c > 0 ? S.spread_c : 1)) * spread_n;

    const int64_t groups_per_block = kPrimalThreads / G;
    const SegSpan span = seg_span(L, S);              // row of the block table resolved once
    const int64_t total = span.count;
    const int64_t stride = (int64_t)gridDim.x * groups_per_block;
    const int64_t slot_end = ((total + stride - 1) / stride) * stride;   // warp-uniform trip count
    ProjStats st;

    for (int64_t slot = (int64_t)blockIdx.x * groups_per_block + threadIdx.x / G; slot < slot_end; slot += stride) {
        int64_t i = 0;
        const bool active = span_slot(span, slot, i);

        // ---- segment state and this lane's quads
        double lam = 1.0, vt0 = 1.0;
        double4 sv = make_double4(1.0, 0.0, 0.0, 1.0);
        int32_t q0 = 0, q1 = 0;
        if (active) {
            const double2 sc = S.segc[i];
            lam = sc.x;
            vt0 = sc.y;
            sv = S.segv[i];
            q0 = S.qoff[i];
            q1 = S.qoff[i + 1];
        }
        const double z0 = sv.x;
        int idx[NE];
        double v[NE], om[NE], z[NE];
        double yold[SAMPLED ? NE : 1];
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int32_t q = q0 + gl + G * t;
            double y4[4] = {0.0, 0.0, 0.0, 0.0};
            if (q < q1) {
                const int4 id4 = ld128_nc(S.pidx + q);
                idx[4 * t + 0] = id4.x; idx[4 * t + 1] = id4.y; idx[4 * t + 2] = id4.z; idx[4 * t + 3] = id4.w;
                ld256_nc(S.v + 4 * (int64_t)q, v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]);
                ld256_nc(S.om + 4 * (int64_t)q, om[4 * t], om[4 * t + 1], om[4 * t + 2], om[4 * t + 3]);
                ld256(S.y + 4 * (int64_t)q, y4[0], y4[1], y4[2], y4[3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    idx[4 * t + e] = N;
                    v[4 * t + e] = 0.0;
                    om[4 * t + e] = 0.0;
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                z[4 * t + e] = y4[e];                     // y_old until the gradient step
                if constexpr (SAMPLED) yold[4 * t + e] = y4[e];
            }
        }
        // a2: price gather (g[N] = 0 for pads; head from shared memory)
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int j = idx[e];
            const double gj = (j < H) ? sm.ghead[j] : __ldg(S.g + j);
            if constexpr (ARGMAX) z[e] = gj;             // theta = inf: keep g itself
            else z[e] = fma(S.theta, gj, z[e]);          // a3: z = y + theta g
        }

        double yv[NE];
        double y0new;
        double x0 = sv.y, x1 = sv.z, x2 = sv.w;
        if constexpr (ARGMAX) argmax_group<G, NE>(z, v, om, lam, vt0, active, yv, y0new);
        else project_group<G, NE>(z, v, om, z0, lam, vt0, active, gmask, S.max_newton, x0, x1, x2, yv, y0new, st);

        // ---- write back, a5 usage scatter
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int32_t q = q0 + gl + G * t;
            if (active && q < q1) st256(S.y + 4 * (int64_t)q, yv[4 * t], yv[4 * t + 1], yv[4 * t + 2], yv[4 * t + 3]);
        }
        if (active && gl == 0) st256(reinterpret_cast<double *>(S.segv + i), y0new, x0, x1, x2);
        if constexpr (SAMPLED) {
#pragma unroll
            for (int e = 0; e < NE; ++e) yv[e] -= yold[e];
        }
        scatter_group<NE>(idx, yv, hg, HH, S.s, N, spread_n, spread_rel);
    }
    if constexpr (!ARGMAX) {
        if (st.passes) {
            atomicAdd(S.counters + 1, st.passes);
            if (st.failures) atomicAdd(S.counters + 0, st.failures);
            if (st.restarts) atomicAdd(S.counters + 2, st.restarts);
        }
    }
    __syncthreads();
    flush_hists(sm.hist, WARPS * GPW, HS, HH, N, S.s);
}

}  // namespace spfom
