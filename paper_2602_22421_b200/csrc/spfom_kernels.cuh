// spfom_kernels.cuh -- sm_100a kernels of one SPFOM iteration (GAM SBLP).
//
// K1  k_primal<G,Q,ARGMAX>   a2 gather g = r - eta, a3 gradient step, a4 the
//                            segment projection (semi-smooth Newton on the
//                            3-scalar KKT system) or, ARGMAX,
//                            the exact inner argmax (Dinkelbach), fused with
//                            a5 the usage scatter s_j += y_ij.
// K3  k_dual                 a7 extrapolated projected dual step (Eq. 17) and
//                            the next price vector g = r - eta; a8 averaging.
// K5/K6 residual kernels     D(eta), audits, per-product residuals.
//
// Thread mapping: a group of G lanes owns one segment; lane l holds the
// row's quads q = l, l+G, ..., (Q of them); a quad is 4 consecutive padded
// entries loaded with one 128-bit (int32 ids) and three 256-bit (v, omega, y)
// loads.  Group sums use xor-butterflies inside the group.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

namespace spfom {

constexpr int kThreads = 256;

struct DevState {
    // per quad (4 padded entries), relabelled product ids, rows sorted by new id
    const int4 *pidx;     // [nq]
    const double *v;      // [4 nq]  attraction (0 on pads)
    const double *om;     // [4 nq]  omega = w / v (0 on pads)
    double *y;            // [4 nq]  sales iterate
    double *ybar;         // [4 nq]  average (averaging on) or null
    // per local segment
    const int32_t *qoff;  // [m+1] quad offsets
    const double2 *seg;   // [m]   (lambda, vt0 = v0 + sum w)
    double *y0;           // [m]   no-purchase iterate
    double *y0bar;        // [m]   or null
    double4 *warm;        // [m]   (nu, kappa, U, -) of the last projection
    // per product, N + 1 slots (slot N = dummy of the pads: g = 0)
    const double *r, *c, *tau;
    double *eta, *g, *s, *s_prev, *etabar;
    // counters (device)
    unsigned long long *counters;  // [0] newton failures, [1] passes, [2] non-finite
    int64_t *t;                    // completed iterations
    int64_t m, N;
    double theta, mu, omega_x;
    int32_t max_newton;
    int32_t sampled;               // 1 => scatter y_new - y_old into s (stale rows kept)
};

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ void ld256_nc(const double *p, double &a, double &b, double &c, double &d) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void ld256(const double *p, double &a, double &b, double &c, double &d) {
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void st256(double *p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}
__device__ __forceinline__ int4 ld128_nc(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ int idx_of(const int4 &q, int e) {
    return e == 0 ? q.x : (e == 1 ? q.y : (e == 2 ? q.z : q.w));
}

template <int G>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
template <int G>
__device__ __forceinline__ double group_max(double x) {
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// Solve J d = -R (3x3) by cofactors; returns false if singular / non-finite.
__device__ __forceinline__ bool newton_dir(const double J[3][3], const double R[3], double d[3]) {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    if (!(fabs(det) > 0.0) || !isfinite(det)) return false;
    const double inv = 1.0 / det;
    const double c10 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    const double c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    const double c12 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    const double c20 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    const double c21 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    const double c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    // J^{-1} = adj / det, adj[i][j] = cofactor[j][i]
    d[0] = -(c00 * R[0] + c10 * R[1] + c20 * R[2]) * inv;
    d[1] = -(c01 * R[0] + c11 * R[1] + c21 * R[2]) * inv;
    d[2] = -(c02 * R[0] + c12 * R[1] + c22 * R[2]) * inv;
    return isfinite(d[0]) && isfinite(d[1]) && isfinite(d[2]);
}

// ----------------------------------------------------------------- K1
// Segments processed by a launch: list[0..count) (local ids) or, list == null,
// the contiguous range [first, first + count).  In sampled mode the list is
// the (iteration row, bin) slice of the block table, found from *t.
struct SegList {
    const int32_t *ids;          // null => contiguous
    int64_t first, count;        // full sweep
    const int32_t *row_off;      // sampled: [block_iters][nbins+1] offsets into ids
    int32_t bin, nbins;
    int64_t block_iters;
};

__device__ __forceinline__ bool seg_slot(const SegList &L, const DevState &S, int64_t slot, int64_t &i) {
    if (L.row_off) {
        const int64_t row = (*S.t) % L.block_iters;
        const int32_t *ro = L.row_off + row * (L.nbins + 1);
        const int64_t a = ro[L.bin], b = ro[L.bin + 1];
        if (slot >= b - a) return false;
        i = L.ids[a + slot];
        return true;
    }
    if (slot >= L.count) return false;
    i = L.ids ? (int64_t)L.ids[L.first + slot] : L.first + slot;
    return true;
}

__device__ __forceinline__ int64_t seg_count(const SegList &L, const DevState &S) {
    if (L.row_off) {
        const int64_t row = (*S.t) % L.block_iters;
        const int32_t *ro = L.row_off + row * (L.nbins + 1);
        return ro[L.bin + 1] - ro[L.bin];
    }
    return L.count;
}

template <int G, int Q, bool ARGMAX>
__global__ void __launch_bounds__(kThreads) k_primal(DevState S, SegList L) {
    constexpr int NE = 4 * Q;                      // entries per lane
    // 2-bit class (0 at zero, 1 free, 2 capped) per entry: the lane's piece signature
    using PieceT = typename std::conditional<(2 * NE <= 32), uint32_t, unsigned long long>::type;
    static_assert(2 * NE <= 64, "piece signature holds at most 32 entries per lane");
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);                 // lane within group
    const int gidx = lane / G;                     // group within warp
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gidx * G));
    const int64_t groups_per_block = (int64_t)kThreads / G;
    const int64_t total = seg_count(L, S);
    const int64_t stride = (int64_t)gridDim.x * groups_per_block;
    int64_t slot = (int64_t)blockIdx.x * groups_per_block + threadIdx.x / G;
    const int64_t slot_end = ((total + stride - 1) / stride) * stride;   // warp-uniform trip count

    for (; slot < slot_end; slot += stride) {
        int64_t i = 0;
        const bool active = seg_slot(L, S, slot, i);

        // ---- segment scalars and this lane's quads
        double lam = 1.0, vt0 = 1.0, z0 = 1.0;
        int32_t q0 = 0, q1 = 0;
        if (active) {
            const double2 sv = S.seg[i];
            lam = sv.x;
            vt0 = sv.y;
            z0 = S.y0[i];
            q0 = S.qoff[i];
            q1 = S.qoff[i + 1];
        }
        int idx[NE];
        double v[NE], om[NE], z[NE], yold[NE];
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int32_t q = q0 + gl + G * t;
            if (q < q1) {
                const int4 id4 = ld128_nc(S.pidx + q);
                idx[4 * t + 0] = id4.x; idx[4 * t + 1] = id4.y; idx[4 * t + 2] = id4.z; idx[4 * t + 3] = id4.w;
                ld256_nc(S.v + 4 * (int64_t)q, v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]);
                ld256_nc(S.om + 4 * (int64_t)q, om[4 * t], om[4 * t + 1], om[4 * t + 2], om[4 * t + 3]);
                ld256(S.y + 4 * (int64_t)q, yold[4 * t], yold[4 * t + 1], yold[4 * t + 2], yold[4 * t + 3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    idx[4 * t + e] = (int)S.N;
                    v[4 * t + e] = 0.0; om[4 * t + e] = 0.0; yold[4 * t + e] = 0.0;
                }
            }
        }
        // a2: price gather (g[N] = 0 for pads)
        double gj[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) gj[e] = __ldg(S.g + idx[e]);

        double ynew[NE];
        double y0new = z0;

        if constexpr (ARGMAX) {
            // ---- exact inner argmax (theta = inf), Dinkelbach from z = 0
            double gv[NE], vt[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                gv[e] = gj[e] * v[e];
                vt[e] = fma(-v[e], om[e], v[e]);
            }
            double zs = 0.0, den = 0.0, sv_in = 0.0;
            bool go = active;
            for (int it = 0; it < 64; ++it) {
                double num = 0.0, dd = 0.0, sv = 0.0;
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    const bool in = gv[e] > zs * vt[e];
                    num += in ? gv[e] : 0.0;
                    dd += in ? vt[e] : 0.0;
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
            for (int e = 0; e < NE; ++e) ynew[e] = (gv[e] > zs * vt[e]) ? v[e] * U : 0.0;
            y0new = lam - U * sv_in;
        } else {
            // ---- a3 gradient step and a4 projection (semi-smooth Newton)
            const double theta = S.theta;
            double w[NE];
            double sabs = 0.0;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                z[e] = fma(theta, gj[e], yold[e]);
                w[e] = v[e] * om[e];
                sabs += fabs(z[e]);
            }
            sabs = group_sum<G>(sabs);
            const double tol = 1e-13 * (lam + fabs(z0) + sabs) * fmax(1.0, vt0);

            double4 wm = active ? S.warm[i] : make_double4(0.0, 0.0, 1.0, 0.0);
            double x0 = wm.x, x1 = wm.y, x2 = wm.z;       // trial point (nu, kappa, U)
            double a0 = x0, a1 = x1, a2 = x2;             // last accepted point
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, step = 1.0, Ra = 0.0;
            PieceT pieceA = 0;
            bool go = active, first = true;
            int passes = 0;
            bool failed = false;
            while (__any_sync(0xffffffffu, go)) {
                // evaluate classification, y and the 9 group sums at x
                double r1 = 0.0, sy = 0.0, swy = 0.0, cv = 0.0, cvw = 0.0, cvv = 0.0, fw = 0.0, fww = 0.0, nf = 0.0;
                PieceT piece = 0;
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    const double a = fma(om[e], x1, z[e] - x0);
                    const double cap = v[e] * x2;
                    const bool isC = a >= cap;
                    const bool isF = !isC && (a > 0.0);
                    const double ye = isC ? cap : (isF ? a : 0.0);
                    sy += ye;
                    swy = fma(om[e], ye, swy);
                    if (isC) {
                        r1 = fma(v[e], a - cap, r1);
                        cv += v[e];
                        cvw += w[e];
                        cvv = fma(v[e], v[e], cvv);
                    }
                    if (isF) {
                        fw += om[e];
                        fww = fma(om[e], om[e], fww);
                        nf += 1.0;
                    }
                    piece |= (PieceT)(isC ? 2u : (isF ? 1u : 0u)) << (2 * e);
                }
                r1 = group_sum<G>(r1);   sy = group_sum<G>(sy);   swy = group_sum<G>(swy);
                cv = group_sum<G>(cv);   cvw = group_sum<G>(cvw); cvv = group_sum<G>(cvv);
                fw = group_sum<G>(fw);   fww = group_sum<G>(fww); nf = group_sum<G>(nf);
                const bool same_piece = (__ballot_sync(0xffffffffu, piece != pieceA) & gmask) == 0u;
                if (go) {
                    ++passes;
                    const double y0c = z0 - x0 + x1;
                    double R[3] = {r1 - vt0 * x1, y0c + swy - vt0 * x2, y0c + sy - lam};
                    const double nr = fmax(fabs(R[0]), fmax(fabs(R[1]), fabs(R[2])));
                    bool done = !(nr > tol) || (!first && step == 1.0 && same_piece);
                    if (!isfinite(nr)) { done = true; failed = true; }
                    if (!done) {
                        const bool accept = first || nr <= (1.0 - 1e-4 * step) * Ra;
                        if (accept) {
                            const double J[3][3] = {{-cv, cvw - vt0, -cvv},
                                                    {-1.0 - fw, 1.0 + fww, cvw - vt0},
                                                    {-1.0 - nf, 1.0 + fw, cv}};
                            double d[3];
                            if (!newton_dir(J, R, d)) {
                                done = true;
                                failed = true;
                            } else {
                                a0 = x0; a1 = x1; a2 = x2;
                                d0 = d[0]; d1 = d[1]; d2 = d[2];
                                Ra = nr;
                                pieceA = piece;
                                step = 1.0;
                            }
                        } else {
                            step *= 0.5;
                            if (step < 1e-12) { done = true; failed = true; }
                        }
                        if (!done) {
                            x0 = a0 + step * d0;
                            x1 = a1 + step * d1;
                            x2 = a2 + step * d2;
                            first = false;
                            if (passes >= S.max_newton) { done = true; failed = true; }
                        }
                    }
                    if (done) go = false;
                }
            }
            if (active && gl == 0) {
                atomicAdd(S.counters + 1, (unsigned long long)passes);
                if (failed) atomicAdd(S.counters + 0, 1ull);
            }
            // y at the final point
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const double a = fma(om[e], x1, z[e] - x0);
                const double cap = v[e] * x2;
                ynew[e] = a >= cap ? cap : (a > 0.0 ? a : 0.0);
            }
            y0new = z0 - x0 + x1;
            if (active && gl == 0) S.warm[i] = make_double4(x0, x1, x2, 0.0);
        }

        // ---- write back, a5 usage scatter
        if (active) {
#pragma unroll
            for (int t = 0; t < Q; ++t) {
                const int32_t q = q0 + gl + G * t;
                if (q < q1) {
                    st256(S.y + 4 * (int64_t)q, ynew[4 * t], ynew[4 * t + 1], ynew[4 * t + 2], ynew[4 * t + 3]);
#pragma unroll
                    for (int e = 4 * t; e < 4 * t + 4; ++e) {
                        if (idx[e] < S.N) {
                            const double contrib = S.sampled ? ynew[e] - yold[e] : ynew[e];
                            atomicAdd(S.s + idx[e], contrib);
                        }
                    }
                }
            }
            if (gl == 0) S.y0[i] = y0new;
        }
    }
}

// ----------------------------------------------------------------- K3
// S.s is this iteration's scatter accumulator, S.s_prev the usage of the
// previous iterate (s = A y).  s_new = full ? acc : s_prev + acc (sampled:
// stale rows kept); st = s_new + omega_x (s_new - s_prev);
// eta = max(0, (1 - tau mu) eta - tau (c - st)); g = r - eta; s_prev = s_new;
// acc = 0.  a8 (averaging): etabar += (eta - etabar) / t.
__global__ void __launch_bounds__(kThreads) k_dual(DevState S, int32_t full) {
    const int64_t t_next = *S.t + 1;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.N; j += (int64_t)gridDim.x * blockDim.x) {
        const double sn = full ? S.s[j] : S.s_prev[j] + S.s[j];
        const double sx = fma(S.omega_x, sn - S.s_prev[j], sn);
        const double tj = S.tau[j];
        const double e = fmax(0.0, fma(-tj, S.c[j] - sx, (1.0 - tj * S.mu) * S.eta[j]));
        S.eta[j] = e;
        S.g[j] = S.r[j] - e;
        S.s_prev[j] = sn;
        S.s[j] = 0.0;
        if (S.etabar) S.etabar[j] += (e - S.etabar[j]) / (double)t_next;
    }
}

__global__ void k_tick(int64_t *t) { *t += 1; }

// a8 averaging of the primal (all rows, so that stale rows count in sampled mode)
__global__ void __launch_bounds__(kThreads) k_average(DevState S, int64_t nq) {
    const double inv = 1.0 / (double)(*S.t + 1);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        double a, b, c, d, ea, eb, ec, ed;
        ld256(S.y + 4 * q, a, b, c, d);
        ld256(S.ybar + 4 * q, ea, eb, ec, ed);
        st256(S.ybar + 4 * q, ea + (a - ea) * inv, eb + (b - eb) * inv, ec + (c - ec) * inv, ed + (d - ed) * inv);
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S.m; i += (int64_t)gridDim.x * blockDim.x)
        S.y0bar[i] += (S.y0[i] - S.y0bar[i]) * inv;
}

// fresh usage: out[j] = sum_i y_ij (out zeroed by the caller)
__global__ void __launch_bounds__(kThreads) k_usage(DevState S, int64_t nq, double *out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        const int4 id = S.pidx[q];
        double a, b, c, d;
        ld256(S.y + 4 * q, a, b, c, d);
        if (id.x < S.N) atomicAdd(out + id.x, a);
        if (id.y < S.N) atomicAdd(out + id.y, b);
        if (id.z < S.N) atomicAdd(out + id.z, c);
        if (id.w < S.N) atomicAdd(out + id.w, d);
    }
}

// ----------------------------------------------------------------- residuals
// Per segment: lambda_i z_i*(r - eta) (Dinkelbach on g = r - eta, the price
// vector k_dual maintains) and the balance / scale / negativity audits of the
// current iterate; per-block partials [4] = (sum D_seg, max bal, max scale, max neg).
template <int G, int Q>
__global__ void __launch_bounds__(kThreads) k_resid_seg(DevState S, SegList L, double *partials) {
    constexpr int NE = 4 * Q;
    __shared__ double red[kThreads / 32][4];
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int64_t groups_per_block = (int64_t)kThreads / G;
    const int64_t total = seg_count(L, S);
    const int64_t stride = (int64_t)gridDim.x * groups_per_block;
    const int64_t slot_end = ((total + stride - 1) / stride) * stride;
    double dsum = 0.0, bmax = 0.0, smax = 0.0, nmax = 0.0;
    for (int64_t slot = (int64_t)blockIdx.x * groups_per_block + threadIdx.x / G; slot < slot_end; slot += stride) {
        int64_t i = 0;
        const bool active = seg_slot(L, S, slot, i);
        double lam = 1.0, vt0 = 1.0, y0 = 1.0;
        int32_t q0 = 0, q1 = 0;
        if (active) {
            lam = S.seg[i].x; vt0 = S.seg[i].y; y0 = S.y0[i]; q0 = S.qoff[i]; q1 = S.qoff[i + 1];
        }
        double v[NE], om[NE], y[NE], gj[NE];
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int32_t q = q0 + gl + G * t;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool ok = q < q1;
                const int64_t p = 4 * (int64_t)q + e;
                v[4 * t + e] = ok ? S.v[p] : 0.0;
                om[4 * t + e] = ok ? S.om[p] : 0.0;
                y[4 * t + e] = ok ? S.y[p] : 0.0;
                gj[4 * t + e] = ok ? S.g[idx_of(S.pidx[q], e)] : 0.0;
            }
        }
        double sy = 0.0, swy = 0.0, neg = fmax(0.0, -y0);
#pragma unroll
        for (int e = 0; e < NE; ++e) { sy += y[e]; swy = fma(om[e], y[e], swy); neg = fmax(neg, -y[e]); }
        sy = group_sum<G>(sy);
        swy = group_sum<G>(swy);
        const double U = (y0 + swy) / vt0;
        double sc = 0.0;
#pragma unroll
        for (int e = 0; e < NE; ++e) sc = fmax(sc, (y[e] - v[e] * U) / lam);
        sc = group_max<G>(sc);
        neg = group_max<G>(neg);
        // Dinkelbach
        double zs = 0.0;
        bool go = active;
        for (int it = 0; it < 64; ++it) {
            double num = 0.0, dd = 0.0;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const double gv = gj[e] * v[e], vt = fma(-v[e], om[e], v[e]);
                const bool in = gv > zs * vt;
                num += in ? gv : 0.0;
                dd += in ? vt : 0.0;
            }
            num = group_sum<G>(num);
            dd = group_sum<G>(dd);
            const double zn = num / (vt0 + dd);
            const bool more = go && (zn > zs);
            if (more) zs = zn;
            go = more;
            if (!__any_sync(0xffffffffu, go)) break;
        }
        if (active && gl == 0) {
            dsum += lam * zs;
            bmax = fmax(bmax, fabs(y0 + sy - lam) / lam);
            smax = fmax(smax, sc);
            nmax = fmax(nmax, neg);
        }
    }
    // block reduction (deterministic order)
    for (int o = 16; o >= 1; o >>= 1) {
        dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
        smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
        nmax = fmax(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    }
    if (lane == 0) {
        red[threadIdx.x / 32][0] = dsum; red[threadIdx.x / 32][1] = bmax;
        red[threadIdx.x / 32][2] = smax; red[threadIdx.x / 32][3] = nmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
        for (int k = 0; k < kThreads / 32; ++k) {
            a += red[k][0]; b = fmax(b, red[k][1]); c = fmax(c, red[k][2]); d = fmax(d, red[k][3]);
        }
        partials[4 * blockIdx.x + 0] = a;
        partials[4 * blockIdx.x + 1] = b;
        partials[4 * blockIdx.x + 2] = c;
        partials[4 * blockIdx.x + 3] = d;
    }
}

// Per product (j < n_present): partials[8] per block =
// (sum r s, sum c eta, max over, max over/max(1,c), sum over^2, sum c^2, sum eta |c - s|, max over/s)
__global__ void __launch_bounds__(kThreads) k_resid_prod(DevState S, const double *sfresh, int64_t n_present,
                                                         double *partials) {
    __shared__ double red[kThreads / 32][8];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_present; j += (int64_t)gridDim.x * blockDim.x) {
        const double s = sfresh[j], c = S.c[j], e = S.eta[j];
        const double over = fmax(0.0, s - c);
        acc[0] += S.r[j] * s;
        acc[1] += c * e;
        acc[2] = fmax(acc[2], over);
        acc[3] = fmax(acc[3], over / fmax(1.0, c));
        acc[4] += over * over;
        acc[5] += c * c;
        acc[6] += e * fabs(c - s);
        if (s > 0.0) acc[7] = fmax(acc[7], over / s);
    }
    const int lane = threadIdx.x & 31;
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double other = __shfl_xor_sync(0xffffffffu, acc[k], o);
            acc[k] = (k == 2 || k == 3 || k == 7) ? fmax(acc[k], other) : acc[k] + other;
        }
    }
    if (lane == 0)
        for (int k = 0; k < 8; ++k) red[threadIdx.x / 32][k] = acc[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        double out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int w = 0; w < kThreads / 32; ++w)
            for (int k = 0; k < 8; ++k)
                out[k] = (k == 2 || k == 3 || k == 7) ? fmax(out[k], red[w][k]) : out[k] + red[w][k];
        for (int k = 0; k < 8; ++k) partials[8 * blockIdx.x + k] = out[k];
    }
}

}  // namespace spfom
