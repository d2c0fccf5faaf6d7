// spfom_kernels.cuh -- sm_100a kernels of one SPFOM iteration (GAM SBLP).
//
// K1  k_primal<G,Q,ARGMAX,SAMPLED>   spfom_primal.cuh: a2 gather, a3 gradient
//                                    step, a4 projection / exact argmax, a5 scatter
// K3  k_dual                         a7 extrapolated projected dual step (Eq. 17)
//                                    and the next price vector g = r - eta; a8
// K5/K6 residual kernels             D(eta), audits, per-product residuals
#pragma once

#include "spfom_common.cuh"
#include "spfom_primal.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace spfom {

// ----------------------------------------------------------------- K3
// S.s is this iteration's scatter accumulator, S.s_prev the usage of the
// previous iterate (s = A y).  s_new = full ? acc : s_prev + acc (sampled:
// stale rows kept); st = s_new + omega_x (s_new - s_prev);
// eta = max(0, (1 - tau mu) eta - tau (c - st)); g = r - eta; s_prev = s_new;
// acc = 0.  a8 (averaging): etabar += (eta - etabar) / t.
// tick != 0 (no averaging): the kernel also advances the iteration counter
// (one launch less per iteration than a separate k_tick).
__global__ void k_tick(int64_t *t) { *t += 1; }

// Fused tick: the kernels that tick never read *S.t themselves (only the
// averaging path reads it, and that path ticks in a separate k_tick), and the
// next reader is a later kernel on the same stream, so one thread of block 0
// can advance the counter without waiting for the other blocks (no fence, no
// arrival counter).
__device__ __forceinline__ void tick_once(const DevState &S) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *S.t += 1;
}

// a7 for one product j (Eq. 17 with extrapolation and per-product tau_j)
// fold of K1's spread copies of product j into acc, in fixed copy order
// (deterministic); all copies are loaded before any is cleared, so the loads
// are independent (one memory latency, not spread_c of them)
__device__ __forceinline__ double fold_spread(const DevState &S, int64_t j, double acc) {
    double part[SPFOM_SPREAD_C];
#pragma unroll
    for (int c = 0; c < SPFOM_SPREAD_C; ++c)
        part[c] = c < S.spread_c ? S.spread[(size_t)c * S.spread_n + j] : 0.0;
#pragma unroll
    for (int c = 0; c < SPFOM_SPREAD_C; ++c) acc += part[c];
#pragma unroll
    for (int c = 0; c < SPFOM_SPREAD_C; ++c)
        if (c < S.spread_c) S.spread[(size_t)c * S.spread_n + j] = 0.0;
    return acc;
}

__device__ __forceinline__ void dual_update(const DevState &S, int64_t j, int32_t full, int64_t t_next) {
    double acc = S.s[j];
    if (S.fold_in_dual && j < S.spread_n) acc = fold_spread(S, j, acc);
    const double sn = full ? acc : S.s_prev[j] + acc;
    const double sx = fma(S.omega_x, sn - S.s_prev[j], sn);
    const double tj = S.tau[j];
    const double e = fmax(0.0, fma(-tj, S.c[j] - sx, (1.0 - tj * S.mu) * S.eta[j]));
    S.eta[j] = e;
    S.g[j] = S.r[j] - e;
    S.s_prev[j] = sn;
    S.s[j] = 0.0;
    if (S.etabar) S.etabar[j] += (e - S.etabar[j]) / (double)t_next;
}

__global__ void __launch_bounds__(kThreads) k_dual(DevState S, int32_t full, int32_t tick) {
    const int64_t t_next = tick ? 0 : *S.t + 1;     // t is only needed for averaging (tick == 0)
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.N; j += (int64_t)gridDim.x * blockDim.x)
        dual_update(S, j, full, t_next);
    if (tick) tick_once(S);
}

// K3 on this rank's slice (world > 1, ReduceScatter -> K3 -> AllGather): the
// ReduceScatter left the summed usage of products [lo, lo + chunk) in
// acc[lo .. lo + chunk); this rank updates their eta, s_prev (and etabar)
// and prices g (slots >= N: g = 0, the pads' dummy); the AllGather that follows
// shares g.  eta / s_prev stay sliced (the getters gather them).  Every acc
// slot of the padded length np is cleared for the next scatter.
__global__ void __launch_bounds__(kThreads) k_dual_slice(DevState S, int32_t full, int32_t tick, int64_t lo,
                                                         int64_t chunk, int64_t np) {
    const int64_t t_next = tick ? 0 : *S.t + 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < lo + chunk; j += stride) {
        if (j < S.N) {
            dual_update(S, j, full, t_next);
        } else {
            S.g[j] = 0.0;
            S.s[j] = 0.0;
        }
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < np; j += stride)
        if (j < lo || j >= lo + chunk) S.s[j] = 0.0;
    if (tick) tick_once(S);
}

// ----------------------------------------------------------------- bundles (a7, NRM)
// P:L719-741 Eq. 33: the dual step runs over the L resources.
// 1) per bundle: s_new, st = s_new + omega_x (s_new - s_prev), s_prev = s_new
__global__ void __launch_bounds__(kThreads) k_bundle_usage(DevState S, int32_t full) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.N; j += (int64_t)gridDim.x * blockDim.x) {
        double acc = S.s[j];
        if (S.fold_in_dual && j < S.spread_n) acc = fold_spread(S, j, acc);
        const double sn = full ? acc : S.s_prev[j] + acc;
        S.stilde[j] = fma(S.omega_x, sn - S.s_prev[j], sn);
        S.s_prev[j] = sn;
        S.s[j] = 0.0;
    }
}
// 2) per resource: St_l = sum_{j uses l} st_j (ascending original bundle id),
//    eta_l = max{0, (1 - tau_l mu) eta_l - tau_l (c_l - St_l)}
__global__ void __launch_bounds__(kThreads) k_bundle_dual(DevState S, int32_t averaging) {
    const int64_t t_next = averaging ? *S.t + 1 : 0;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < S.L; l += (int64_t)gridDim.x * blockDim.x) {
        double st = 0.0;
        for (int32_t e = S.rptr[l]; e < S.rptr[l + 1]; ++e) st += S.stilde[S.rbun[e]];
        const double tl = S.tau[l];
        const double e = fmax(0.0, fma(-tl, S.c[l] - st, (1.0 - tl * S.mu) * S.eta[l]));
        S.eta[l] = e;
        if (S.etabar) S.etabar[l] += (e - S.etabar[l]) / (double)t_next;
    }
}
// 3) per bundle: g_j = r_j - sum_{l in B_j} eta_l; optional tick
__global__ void __launch_bounds__(kThreads) k_bundle_prices(DevState S, int32_t tick) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.N; j += (int64_t)gridDim.x * blockDim.x) {
        double b = 0.0;
        for (int32_t e = S.bptr[j]; e < S.bptr[j + 1]; ++e) b += S.eta[S.bres[e]];
        S.g[j] = S.r[j] - b;
    }
    if (tick) tick_once(S);
}

// Residual terms of the resource rows (bundles): partials[8] per block as in
// k_resid_prod with slot 0 (objective) left 0.
__global__ void __launch_bounds__(kThreads) k_resid_res(DevState S, const double *sfresh, double *partials) {
    __shared__ double red[kThreads / 32][8];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < S.L; l += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int32_t e = S.rptr[l]; e < S.rptr[l + 1]; ++e) s += sfresh[S.rbun[e]];
        const double c = S.c[l], et = S.eta[l];
        const double over = fmax(0.0, s - c);
        acc[1] += c * et;
        acc[2] = fmax(acc[2], over);
        acc[3] = fmax(acc[3], over / fmax(1.0, c));
        acc[4] += over * over;
        acc[5] += c * c;
        acc[6] += et * fabs(c - s);
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

// world > 1: fold K1's spread copies into the usage accumulator before the allreduce
__global__ void __launch_bounds__(kThreads) k_fold(DevState S) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S.spread_n) return;
    S.s[j] = fold_spread(S, j, S.s[j]);
}

// ----------------------------------------------------------------- small regime
// Persistent cooperative kernel running `iters` whole iterations in one launch
// (world == 1, no averaging / refresh): per iteration, a1-a5 over this
// iteration's segments (one warp per segment, 4 Q entries per lane), grid-wide
// barrier, a7 over all products, barrier.  Replaces 2 graph nodes + their
// launch latency per iteration when the per-iteration work is a few thousand
// segments (small instances, the paper's small sampled blocks).
struct SmallArgs {
    const int32_t *ids;        // sampled: block table (device slots), else null (full sweep over [0, m))
    const int32_t *row_off;    // sampled: [block_iters][nbins + 1]
    int64_t block_iters;
    int32_t nbins;
    int32_t full_mode;         // 1: s = acc (full sweep); 0: s = s_prev + acc (sampled)
    int64_t t0, iters;         // first iteration index, iterations in this launch
};
constexpr int kSmallThreads = 256;

template <int Q, bool ARGMAX, bool SAMPLED>
__global__ void __launch_bounds__(kSmallThreads, 1) k_small(DevState S, SmallArgs A) {
    constexpr int G = 32, NE = 4 * Q;
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int N = (int)S.N;
    const int spread_n = S.spread_n;
    const int spread_rel = S.spread_off + (int)(gwarp % (S.spread_c > 0 ? S.spread_c : 1)) * spread_n;
    ProjStats st;
    for (int64_t it = 0; it < A.iters; ++it) {
        const int64_t t = A.t0 + it;
        const int32_t *ids = nullptr;
        int64_t cnt = S.m;
        if constexpr (SAMPLED) {
            const int32_t *ro = A.row_off + (t % A.block_iters) * (A.nbins + 1);
            ids = A.ids + ro[0];
            cnt = ro[A.nbins] - ro[0];
        }
        for (int64_t k = gwarp; k < cnt; k += nwarps) {
            const int64_t i = SAMPLED ? (int64_t)ids[k] : k;
            const double2 sc = S.segc[i];
            const double4 sv = S.segv[i];
            const int32_t q0 = S.qoff[i], q1 = S.qoff[i + 1];
            int idx[NE];
            double v[NE], om[NE], z[NE];
            double yold[SAMPLED ? NE : 1];
#pragma unroll
            for (int tq = 0; tq < Q; ++tq) {
                const int32_t q = q0 + lane + G * tq;
                double y4[4] = {0.0, 0.0, 0.0, 0.0};
                if (q < q1) {
                    const int4 id4 = ld128_nc(S.pidx + q);
                    idx[4 * tq + 0] = id4.x; idx[4 * tq + 1] = id4.y; idx[4 * tq + 2] = id4.z; idx[4 * tq + 3] = id4.w;
                    ld256_nc(S.v + 4 * (int64_t)q, v[4 * tq], v[4 * tq + 1], v[4 * tq + 2], v[4 * tq + 3]);
                    ld256_nc(S.om + 4 * (int64_t)q, om[4 * tq], om[4 * tq + 1], om[4 * tq + 2], om[4 * tq + 3]);
                    ld256(S.y + 4 * (int64_t)q, y4[0], y4[1], y4[2], y4[3]);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        idx[4 * tq + e] = N;
                        v[4 * tq + e] = 0.0;
                        om[4 * tq + e] = 0.0;
                    }
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    z[4 * tq + e] = y4[e];
                    if constexpr (SAMPLED) yold[4 * tq + e] = y4[e];
                }
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const double gj = S.g[idx[e]];                 // a2 (g[N] = 0 for pads)
                if constexpr (ARGMAX) z[e] = gj;
                else z[e] = fma(S.theta, gj, z[e]);            // a3
            }
            double yv[NE];
            double y0new;
            double x0 = sv.y, x1 = sv.z, x2 = sv.w;
            constexpr bool EX = SPFOM_EXTRAP && !SAMPLED && !ARGMAX;   // extrapolated warm start (spfom_primal.cuh)
            float4 sd = make_float4(0.f, 0.f, 0.f, 0.f);
            if (EX && t + 1 >= SPFOM_EXTRAP_FROM && t + 1 < SPFOM_EXTRAP_UNTIL) {
                sd = S.segd[i];
                x0 += (double)sd.x;
                x1 += (double)sd.y;
                x2 = fmax(x2 + (double)sd.z, 0.5 * x2);
            }
            if constexpr (ARGMAX) argmax_group<G, NE>(z, v, om, sc.x, sc.y, true, yv, y0new);
            else project_group<G, NE>(z, v, om, sv.x, sc.x, sc.y, true, 0xffffffffu, S.max_newton, x0, x1, x2, yv,
                                      y0new, st);
#pragma unroll
            for (int tq = 0; tq < Q; ++tq) {
                const int32_t q = q0 + lane + G * tq;
                if (q < q1) st256(S.y + 4 * (int64_t)q, yv[4 * tq], yv[4 * tq + 1], yv[4 * tq + 2], yv[4 * tq + 3]);
            }
            if (lane == 0) {
                st256(reinterpret_cast<double *>(S.segv + i), y0new, x0, x1, x2);
                if (EX && t + 1 < SPFOM_EXTRAP_UNTIL)
                    S.segd[i] = make_float4((float)(x0 - sv.y), (float)(x1 - sv.z), (float)(x2 - sv.w), 0.f);
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) {                    // a5
                const int j = idx[e];
                double c = yv[e];
                if constexpr (SAMPLED) c -= yold[e];
                const int off = j < spread_n ? spread_rel + j : j;
                red_add_if(S.s + off, c, j < N);
            }
        }
        grid.sync();
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < S.N; j += (int64_t)gridDim.x * blockDim.x)
            dual_update(S, j, A.full_mode, 0);                // a7
        grid.sync();
    }
    if constexpr (!ARGMAX) {
        if (st.passes) {
            atomicAdd(S.counters + 1, st.passes);
            if (st.failures) atomicAdd(S.counters + 0, st.failures);
            if (st.restarts) atomicAdd(S.counters + 2, st.restarts);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *S.t += A.iters;
}

// ----------------------------------------------------------------- recovery
// SBLP -> CBLP policy recovery (P:L476-492 Lemma "recover", GAM reading
// SV App. A.1): per segment, the products sorted by u_j = y_j / v_j descending
// (ties: ascending original product id) and the probabilities of the
// nested assortments S_l = first l products, l = 0..k:
//   alpha_l = (u_(l) - u_(l+1)) D(S_l) / lambda,  u_(0) = U, u_(k+1) = 0,
//   D(S) = vt0 + sum_{j in S} (v_j - w_j).
// One warp per segment of the device-slot chunk [a, b); rank by counting
// (k <= KM, the capacity of the warp's shared-memory rows, chosen per chunk
// from its longest row so that short rows keep many warps per SM), warp-scan
// of the sorted vt for D.  Outputs for slot k start at 4 (qoff[k] - qoff[a])
// (order, original ids) and that + (k - a) (alpha).
constexpr int kRecoverMaxK = 1024;
template <int KM>
__host__ __device__ constexpr int recover_warps() { return KM > 256 ? 4 : 8; }
template <int KM>
struct RecoverSmem {
    static constexpr int W = recover_warps<KM>();
    double u[W][KM];      // row order
    double vt[W][KM];
    double su[W][KM];     // sorted order
    double svt[W][KM];
    int32_t oid[W][KM];
};

template <int KM>
__global__ void __launch_bounds__(32 * recover_warps<KM>()) k_recover(DevState S, int64_t a, int64_t b, int64_t t,
                                                                const int32_t *orig_of, int32_t *order_out,
                                                                double *alpha_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RecoverSmem<KM> &sm = *reinterpret_cast<RecoverSmem<KM> *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *u = sm.u[warp], *vt = sm.vt[warp], *su = sm.su[warp], *svt = sm.svt[warp];
    int32_t *oid = sm.oid[warp];
    const int64_t qa = S.qoff[a];
    constexpr int W = recover_warps<KM>();
    for (int64_t k = a + (int64_t)blockIdx.x * W + warp; k < b; k += (int64_t)gridDim.x * W) {
        const int64_t q0 = S.qoff[k], q1 = S.qoff[k + 1];
        const double2 sc = S.segc[t * S.m + k];                // (lambda, vt0)
        const double y0 = S.segv[t * S.m + k].x;
        const double *yrow = S.y + 4 * (t * S.nq + q0);
        const int32_t *ids = reinterpret_cast<const int32_t *>(S.pidx + q0);
        // the row's real entries come first (pads carry id N, the largest relabelled id)
        const int np = (int)(4 * (q1 - q0));
        int kk = 0;
        double swy = 0.0;
        for (int e = lane; e < np; e += 32) {
            const int32_t j = ids[e];
            const bool real = j < S.N;
            const double v = S.v[4 * q0 + e], om = S.om[4 * q0 + e], y = yrow[e];
            u[e] = real ? y / v : 0.0;
            vt[e] = real ? fma(-v, om, v) : 0.0;
            oid[e] = real ? orig_of[j] : INT32_MAX;
            swy += real ? om * y : 0.0;
            kk += real ? 1 : 0;
        }
        for (int o = 16; o >= 1; o >>= 1) {
            swy += __shfl_xor_sync(0xffffffffu, swy, o);
            kk += __shfl_xor_sync(0xffffffffu, kk, o);
        }
        __syncwarp();
        // rank by counting: u descending, ties by ascending original product id
        const int64_t ob = 4 * (q0 - qa), ab = ob + (k - a);
        // each lane ranks NR of the row's entries (lane, lane + 32, ..) in one pass over u
        constexpr int NR = KM <= 64 ? 2 : 1;
        for (int e0 = lane; e0 < kk; e0 += 32 * NR) {
            double ue[NR];
            int32_t ie[NR];
            int rank[NR];
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                const int e = e0 + 32 * c;
                ue[c] = e < kk ? u[e] : -1.0;          // u >= 0: an absent entry ranks last
                ie[c] = e < kk ? oid[e] : INT32_MAX;
                rank[c] = 0;
            }
#pragma unroll 8
            for (int f = 0; f < kk; ++f) {
                const double uf = u[f];
#pragma unroll
                for (int c = 0; c < NR; ++c) {
                    rank[c] += uf > ue[c] ? 1 : 0;
                    if (uf == ue[c]) rank[c] += oid[f] < ie[c] ? 1 : 0;   // ties (and f = e): rare, by id
                }
            }
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                const int e = e0 + 32 * c;
                if (e < kk) {
                    su[rank[c]] = ue[c];
                    svt[rank[c]] = vt[e];
                    order_out[ob + rank[c]] = ie[c];
                }
            }
        }
        __syncwarp();
        // D_l = vt0 + sum_{r < l} vt_(r): each lane scans one contiguous chunk of l
        const int per = (kk + 31) / 32;
        const int l0 = min(kk, lane * per), l1 = min(kk, l0 + per);
        double part = 0.0;
        for (int l = l0; l < l1; ++l) part += svt[l];
        double incl = part;
        for (int o = 1; o < 32; o <<= 1) {
            const double x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        double D = sc.y + (incl - part);
        const double U = (y0 + swy) / sc.y;
        for (int l = l0; l < l1; ++l) {
            const double prev = (l == 0) ? U : su[l - 1];
            alpha_out[ab + l] = (prev - su[l]) * D / sc.x;
            D += svt[l];
        }
        // alpha_k (the full prefix, u_(k+1) = 0): by the lane that ends the last chunk
        if (kk > 0 && l1 == kk && l0 < l1) alpha_out[ab + kk] = su[kk - 1] * D / sc.x;
        if (kk == 0 && lane == 0) alpha_out[ab] = U * sc.y / sc.x;
        __syncwarp();
    }
}

// a8 averaging of the primal (all rows, so that stale rows count in sampled mode)
__global__ void __launch_bounds__(kThreads) k_average(DevState S, int64_t nq) {
    const double inv = 1.0 / (double)(*S.t + 1);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        double a, b, c, d, ea, eb, ec, ed;
        ld256(S.y + 4 * q, a, b, c, d);
        ld256(S.ybar + 4 * q, ea, eb, ec, ed);
        st256(S.ybar + 4 * q, ea + (a - ea) * inv, eb + (b - eb) * inv, ec + (c - ec) * inv, ed + (d - ed) * inv);
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S.m * S.T; i += (int64_t)gridDim.x * blockDim.x)
        S.y0bar[i] += (S.segv[i].x - S.y0bar[i]) * inv;
}

// fresh usage: out[j] += sum_i y_ij (out zeroed by the caller); head products
// accumulate in a per-block shared histogram first (the Zipf head would
// serialise global atomics on a handful of addresses).
__global__ void __launch_bounds__(kThreads) k_usage(DevState S, int64_t nq, double *out, int32_t H) {
    __shared__ double hh[kHeadMax];
    for (int j = threadIdx.x; j < H; j += blockDim.x) hh[j] = 0.0;
    __syncthreads();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        const int4 id = S.pidx[q < S.nq ? q : q % S.nq];      // y is [T][nq]: the structure repeats
        double y[4];
        ld256(S.y + 4 * q, y[0], y[1], y[2], y[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = idx_of(id, e);
            if (j < H) atomicAdd(hh + j, y[e]);
            else if (j < S.N) atomicAdd(out + j, y[e]);
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < H; j += blockDim.x)
        if (hh[j] != 0.0) atomicAdd(out + j, hh[j]);
}

// ----------------------------------------------------------------- residuals
// Per segment: lambda_i z_i*(r - eta) (Dinkelbach on g = r - eta, the price
// vector k_dual maintains) and the balance / scale / negativity audits of the
// current iterate; per-block partials [4] = (sum D_seg, max bal, max scale, max neg).
// Multi-period: launched once per period t with (seg_off, quad_off) = (t m, t nq).
template <int G, int Q>
__global__ void __launch_bounds__(kThreads) k_resid_seg(DevState S, SegList L, double *partials, int64_t seg_off,
                                                        int64_t quad_off) {
    constexpr int NE = 4 * Q;
    __shared__ double red[kThreads / 32][4];
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int64_t groups_per_block = (int64_t)kThreads / G;
    const SegSpan span = seg_span(L, S);
    const int64_t total = span.count;
    const int64_t stride = (int64_t)gridDim.x * groups_per_block;
    const int64_t slot_end = ((total + stride - 1) / stride) * stride;
    double dsum = 0.0, bmax = 0.0, smax = 0.0, nmax = 0.0;
    for (int64_t slot = (int64_t)blockIdx.x * groups_per_block + threadIdx.x / G; slot < slot_end; slot += stride) {
        int64_t i = 0;
        const bool active = span_slot(span, slot, i);
        double lam = 1.0, vt0 = 1.0, y0 = 1.0;
        int32_t q0 = 0, q1 = 0;
        if (active) {
            lam = S.segc[seg_off + i].x; vt0 = S.segc[seg_off + i].y; y0 = S.segv[seg_off + i].x;
            q0 = S.qoff[i]; q1 = S.qoff[i + 1];
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
                y[4 * t + e] = ok ? S.y[4 * quad_off + p] : 0.0;
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
        // accumulate: one launch per period writes into the same (zeroed) partials
        partials[4 * blockIdx.x + 0] += a;
        partials[4 * blockIdx.x + 1] = fmax(partials[4 * blockIdx.x + 1], b);
        partials[4 * blockIdx.x + 2] = fmax(partials[4 * blockIdx.x + 2], c);
        partials[4 * blockIdx.x + 3] = fmax(partials[4 * blockIdx.x + 3], d);
    }
}

// Per product (j < n_present): partials[8] per block =
// (sum r s, sum c eta, max over, max over/max(1,c), sum over^2, sum c^2, sum eta |c - s|, max over/s)
__global__ void __launch_bounds__(kThreads) k_resid_prod(DevState S, const double *sfresh, int64_t n_present,
                                                         double *partials) {
    __shared__ double red[kThreads / 32][8];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_present; j += (int64_t)gridDim.x * blockDim.x) {
        const double s = sfresh[j];
        acc[0] += S.r[j] * s;
        if (S.L > 0) continue;                 // bundles: capacity rows are resources (k_resid_res)
        const double c = S.c[j], e = S.eta[j];
        const double over = fmax(0.0, s - c);
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
