// spfom_primal.cuh -- K1, the fused primal kernel of one SPFOM iteration.
//
//   a2 gather g_ij = r_j - eta_j (head of g staged in shared memory)
//   a3 gradient step z_ij = y_ij + theta g_ij, z_i0 = y_i0
//   a4 projection of (z_i0, z_i) onto Y_i (GAM polytope, reading c3/c5): semi-
//      smooth Newton on the 3-scalar KKT system in (nu, kappa, U), warm-started
//      from the segment's previous multipliers; theta = inf: exact inner argmax
//      by Dinkelbach (reading c6)
//   a5 usage scatter s_j += y_ij (sampled: y_new - y_old): the Zipf head
//      j < head goes to per-warp shared-memory histograms, flushed once per
//      persistent block; the tail uses global fp64 reductions.
//
// Thread mapping: a group of G lanes owns one segment; lane l holds quads
// l, l+G, .. (Q of them) of the padded row; a quad = 4 entries = one 128-bit
// id load + three 256-bit loads (v, omega, y).
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
// (sufficient-decrease test, backtracking on ||R||_inf).  Every pass also
// produces y at its point, so the terminating pass yields the output.
//
// Head scatter: the warp's segments share one histogram, so their updates of
// a hot product would collide.  Every lane stages its (id, contribution)
// pairs in shared memory; then, one segment at a time, all 32 lanes apply
// that segment's staged updates -- ids within a segment are distinct, so a
// round has no conflicts and needs no atomics.
#pragma once

#include "spfom_common.cuh"

namespace spfom {

// Solve J d = -R (3x3) by cofactors; false if singular / non-finite.
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
    d[0] = -(c00 * R[0] + c10 * R[1] + c20 * R[2]) * inv;   // J^{-1} = adj(J) / det
    d[1] = -(c01 * R[0] + c11 * R[1] + c21 * R[2]) * inv;
    d[2] = -(c02 * R[0] + c12 * R[1] + c22 * R[2]) * inv;
    return isfinite(d[0]) && isfinite(d[1]) && isfinite(d[2]);
}

struct PieceSums {
    double sfa, sfwa, rva, cv, cvw, cvv, fw, fww;
    int nf;
};

// FULL pass, one entry: classify at (x0, x1, x2) = (nu, kappa, U), accumulate
// the piece-constant sums, set the class bits, return y_j (branch-free; ptxas
// turns the selects into FSEL, which beats predicated fp64 here).
__device__ __forceinline__ double full_entry(double z, double v, double om, double x0, double x1, double x2,
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
    s.nf += isF ? 1 : 0;
    return isC ? cap : af;
}

// CHECK pass, one entry: class bits and y_j at (x0, x1, x2) only.
__device__ __forceinline__ double check_entry(double z, double v, double om, double x0, double x1, double x2,
                                              uint32_t bit, uint32_t &cm, uint32_t &fm) {
    const double a = fma(om, x1, z - x0);
    const double cap = v * x2;
    const bool isC = a >= cap;
    const bool isF = !isC && (a > 0.0);
    cm |= isC ? bit : 0u;
    fm |= isF ? bit : 0u;
    return isC ? cap : (isF ? a : 0.0);
}

template <int Q>
struct PrimalSmem {
    static constexpr int WARPS = kPrimalThreads / 32;
    static constexpr int NE = 4 * Q;
    double hist[WARPS][kHeadMax];          // per-warp usage of the head products
    double ghead[kHeadMax];                // price vector g on the head products
    double stage_val[WARPS][32 * NE];      // staged head contributions, [warp][e * 32 + lane]
    int stage_idx[WARPS][32 * NE];
};

// Resident blocks per SM the register budget targets: one quad per lane fits 4
// blocks (128 registers), wider lanes 3.
template <int Q>
constexpr int primal_min_blocks() { return kPrimalMinBlocks; }

template <int G, int Q, bool ARGMAX, bool SAMPLED>
__global__ void __launch_bounds__(kPrimalThreads, primal_min_blocks<Q>()) k_primal(DevState S, SegList L) {
    constexpr int NE = 4 * Q;               // entries per lane
    constexpr int GPW = 32 / G;             // segments per warp
    constexpr int WARPS = kPrimalThreads / 32;
    static_assert(NE <= 32, "class bitmasks hold at most 32 entries per lane");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    PrimalSmem<Q> &sm = *reinterpret_cast<PrimalSmem<Q> *>(smem_raw);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int gidx = lane / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gidx * G));
    const int H = L.head;

    for (int j = threadIdx.x; j < H; j += kPrimalThreads) {
        sm.ghead[j] = S.g[j];
#pragma unroll
        for (int w = 0; w < WARPS; ++w) sm.hist[w][j] = 0.0;
    }
    __syncthreads();
    double *hw = sm.hist[warp];
    double *stv = sm.stage_val[warp];
    int *sti = sm.stage_idx[warp];

    const int64_t groups_per_block = kPrimalThreads / G;
    const int64_t total = seg_count(L, S);
    const int64_t stride = (int64_t)gridDim.x * groups_per_block;
    const int64_t slot_end = ((total + stride - 1) / stride) * stride;   // warp-uniform trip count
    unsigned long long passes_acc = 0, fail_acc = 0, restart_acc = 0;

    for (int64_t slot = (int64_t)blockIdx.x * groups_per_block + threadIdx.x / G; slot < slot_end; slot += stride) {
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
                    idx[4 * t + e] = (int)S.N;
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

        double yv[NE];                          // y at the terminating point
        double y0new;
        if constexpr (ARGMAX) {
            // ---- exact inner argmax, Dinkelbach from z = 0 (reading c6)
            double zs = 0.0, den = 0.0, sv_in = 0.0;
            bool go = active;
            for (int it = 0; it < 64; ++it) {
                double num = 0.0, dd = 0.0, sv = 0.0;
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    const double gv = z[e] * v[e], vt = fma(-v[e], om[e], v[e]);
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
            for (int e = 0; e < NE; ++e) yv[e] = (z[e] * v[e] > zs * fma(-v[e], om[e], v[e])) ? v[e] * U : 0.0;
            y0new = lam - U * sv_in;
        } else {
            double sabs = 0.0;
#pragma unroll
            for (int e = 0; e < NE; ++e) sabs += fabs(z[e]);
            sabs = group_sum<G>(sabs);
            const double tol = 1e-13 * (lam + fabs(z0) + sabs) * fmax(1.0, vt0);

            const double4 wm = active ? S.warm[i] : make_double4(0.0, 0.0, 1.0, 0.0);
            double x0 = wm.x, x1 = wm.y, x2 = wm.z;             // trial point (nu, kappa, U)
            double a0 = x0, a1 = x1, a2 = x2;                   // last accepted point
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, step = 1.0, Ra = 0.0;
            uint32_t cA = 0, fA = 0;                            // class bitmasks at the accepted point
            bool go = active, full = true, first = true, failed = false, restarted = false;
            int passes = 0;
            const int restart_at = S.max_newton / 2;
            while (__any_sync(0xffffffffu, go)) {
                // safeguard: a segment still unconverged after half the budget restarts
                // from the cold point (nu, kappa, U) = ((z0 + sum z - lam)/(k+1), 0, lam/(vt0 + sum vt))
                if (__any_sync(0xffffffffu, go && passes == restart_at)) {
                    double sz = 0.0, svt = 0.0, nk = 0.0;
#pragma unroll
                    for (int e = 0; e < NE; ++e) {
                        sz += z[e];
                        svt += fma(-v[e], om[e], v[e]);
                        nk += v[e] > 0.0 ? 1.0 : 0.0;
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
                PieceSums ps = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0};
                if (need) {
#pragma unroll
                    for (int e = 0; e < NE; ++e) (void)full_entry(z[e], v[e], om[e], x0, x1, x2, 1u << e, ps, cm, fm);
                    ps.sfa = group_sum<G>(ps.sfa);   ps.sfwa = group_sum<G>(ps.sfwa);
                    ps.rva = group_sum<G>(ps.rva);   ps.cv = group_sum<G>(ps.cv);
                    ps.cvw = group_sum<G>(ps.cvw);   ps.cvv = group_sum<G>(ps.cvv);
                    ps.fw = group_sum<G>(ps.fw);     ps.fww = group_sum<G>(ps.fww);
#pragma unroll
                    for (int o = G / 2; o >= 1; o >>= 1) ps.nf += __shfl_xor_sync(0xffffffffu, ps.nf, o);
                } else {
#pragma unroll
                    for (int e = 0; e < NE; ++e) (void)check_entry(z[e], v[e], om[e], x0, x1, x2, 1u << e, cm, fm);
                }
                const bool changed = (__ballot_sync(0xffffffffu, (cm != cA) || (fm != fA)) & gmask) != 0u;
                if (go) {
                    ++passes;
                    if (!full) {
                        // CHECK pass after a full Newton step from the accepted point
                        if (!changed) go = false;     // same piece: R(x) = 0 exactly
                        else full = true;             // piece moved: evaluate R, J here
                    } else {
                        const double y0c = z0 - x0 + x1;
                        const double sy = fma(x2, ps.cv, ps.sfa);
                        const double swy = fma(x2, ps.cvw, ps.sfwa);
                        const double r1 = fma(-x2, ps.cvv, ps.rva);
                        const double R[3] = {r1 - vt0 * x1, y0c + swy - vt0 * x2, y0c + sy - lam};
                        const double nr = fmax(fabs(R[0]), fmax(fabs(R[1]), fabs(R[2])));
                        bool done = !(nr > tol);
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
                                    failed = true;
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
                            if (!done && passes >= S.max_newton) {
                                // budget spent: keep the last evaluated point
                                done = true;
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
            if (active && gl == 0) {
                passes_acc += (unsigned long long)passes;
                fail_acc += failed ? 1ull : 0ull;
                restart_acc += restarted ? 1ull : 0ull;
                S.warm[i] = make_double4(x0, x1, x2, 0.0);
            }
            uint32_t cm = 0, fm = 0;
#pragma unroll
            for (int e = 0; e < NE; ++e) yv[e] = check_entry(z[e], v[e], om[e], x0, x1, x2, 1u << e, cm, fm);
            y0new = z0 - x0 + x1;
        }

        // ---- write back, a5 usage scatter (tail: global RED; head: staged)
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int32_t q = q0 + gl + G * t;
            const bool ok = active && q < q1;
            if (ok) st256(S.y + 4 * (int64_t)q, yv[4 * t], yv[4 * t + 1], yv[4 * t + 2], yv[4 * t + 3]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 4 * t + e;
                const int j = ok ? idx[k] : (int)S.N;
                double c = yv[k];
                if constexpr (SAMPLED) c -= yold[k];
                if (j >= H && j < S.N) atomicAdd(S.s + j, c);
                stv[k * 32 + lane] = c;
                sti[k * 32 + lane] = j < H ? j : -1;
            }
        }
        if (active && gl == 0) S.y0[i] = y0new;
        if (H > 0) {
            __syncwarp();
            // one segment of the warp at a time; its G*NE staged updates hit distinct ids
#pragma unroll
            for (int gg = 0; gg < GPW; ++gg) {
#pragma unroll
                for (int u = lane; u < G * NE; u += 32) {
                    const int p = (u / G) * 32 + gg * G + (u % G);   // entry u / G of lane gg*G + u % G
                    const int j = sti[p];
                    if (j >= 0) hw[j] += stv[p];
                }
                __syncwarp();
            }
        }
    }
    if constexpr (!ARGMAX) {
        if (gl == 0 && passes_acc) {
            atomicAdd(S.counters + 1, passes_acc);
            if (fail_acc) atomicAdd(S.counters + 0, fail_acc);
            if (restart_acc) atomicAdd(S.counters + 2, restart_acc);
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < H; j += kPrimalThreads) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) sum += sm.hist[w][j];
        if (sum != 0.0) atomicAdd(S.s + j, sum);
    }
}

}  // namespace spfom
