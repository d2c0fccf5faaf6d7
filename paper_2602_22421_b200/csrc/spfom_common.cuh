// spfom_common.cuh -- device state, memory helpers and segment lists shared by
// the SPFOM kernels (sm_100a, fp64).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

#ifndef SPFOM_L2_HINTS
#define SPFOM_L2_HINTS 0   // measured: evict-first on the K1 streams costs ~1% on huge
#endif

namespace spfom {

constexpr int kThreads = 256;       // non-primal kernels
constexpr int kPrimalThreads = 128; // K1: 4 warps per block, 4 blocks per SM
#ifndef SPFOM_PRIMAL_MIN_BLOCKS
#define SPFOM_PRIMAL_MIN_BLOCKS 3
#endif
constexpr int kPrimalMinBlocks = SPFOM_PRIMAL_MIN_BLOCKS;
constexpr int kHeadMax = 1024;      // products privatised in shared memory (Zipf head)
#ifndef SPFOM_GHEAD_MAX
#define SPFOM_GHEAD_MAX 4096
#endif
constexpr int kGHeadStreamMax = SPFOM_GHEAD_MAX;   // K1 stream: head of g staged in shared memory

struct DevState {
    // per quad (4 padded entries), relabelled product ids, rows sorted by new id
    const int4 *pidx;     // [nq]
    const double *v;      // [4 nq]  attraction (0 on pads)
    const double *om;     // [4 nq]  omega = w / v (0 on pads)
    double *y;            // [4 nq]  sales iterate
    double *ybar;         // [4 nq]  average (averaging on) or null
    // per local segment (stored in bin order)
    const int32_t *qoff;  // [m+1] quad offsets
    const double2 *segc;  // [m]   (lambda, vt0 = v0 + sum w), read-only
    double4 *segv;        // [m]   (y0, nu, kappa, U): no-purchase iterate + warm start of the projection
    float4 *segd;         // [m]   last change of (nu, kappa, U) (full-sweep stream kernel: the warm
                          //       start is extrapolated along it; 0 elsewhere / after set_state)
    double *y0bar;        // [m]   or null
    // per product, N + 1 slots (slot N = dummy of the pads: g = 0)
    const double *r, *c, *tau;
    double *eta, *g, *s, *s_prev, *etabar;   // s: usage accumulator (N + 1 slots, then the spread copies)
    // usage-accumulator copies for the warm part of the Zipf head (stream K1):
    // products [hh, spread_n) reduce into spread[c * spread_n + j], c = warp % spread_c,
    // so that no single address takes every segment's update; folded into s
    // by K3 (world == 1) or k_fold before the allreduce
    // bundles / NRM (L > 0): eta, c, tau, etabar hold the L resources; bundle j
    // (relabelled) consumes bres[bptr[j] .. bptr[j+1]); resource l is used by
    // the bundles rbun[rptr[l] .. rptr[l+1]) (ascending original bundle id)
    int32_t L;
    const int32_t *bptr, *bres, *rptr, *rbun;
    double *stilde;                // [N + 1] extrapolated bundle usage of the iteration
    double *spread;                // = s + spread_off
    int32_t spread_n, spread_c, spread_off;
    int32_t fold_in_dual;
    // counters (device)
    unsigned long long *counters;  // [0] newton failures, [1] passes
    int64_t *t;                    // completed iterations
    int64_t m, N;              // local base segments, products
    int64_t nq;                // base quads; y, ybar are [T][nq] quads, segc / segv / y0bar [T][m]
    int32_t T;                 // periods sharing the structure (1 = single period)
    double theta, mu, omega_x;
    int32_t max_newton;
    int32_t sampled;               // 1 => scatter y_new - y_old into s (stale rows kept)
};

// ----------------------------------------------------------------- device checks
// SPFOM_DEVICE_CHECKS (debug build, tests/test_device_checks.py): index and
// size checks in the primal kernels; a failed check increments counters[5]
// (the next synchronising getter returns SPFOM_ENUMERIC) instead of trapping.
// compute-sanitizer is closed on this GPU pool; this is its stand-in.
#ifdef SPFOM_DEVICE_CHECKS
#define SPFOM_DCHECK(S, cond) do { if (!(cond)) atomicAdd((S).counters + 5, 1ull); } while (0)
#else
#define SPFOM_DCHECK(S, cond) do { } while (0)
#endif

// ----------------------------------------------------------------- memory helpers
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
// ----------------------------------------------------------------- TMA bulk copies + mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// TMA 1-D bulk copy global -> shared, completion counted on `bar` (16-B multiples/alignment)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// L2 evict-first policy for data streamed once per iteration (keeps g, the
// usage accumulators and the per-segment state resident in L2)
// TMA tile::gather4 (sm_100a): 4 rows of a 2-D tensor (box {cols, 1}) with
// arbitrary row coordinates, landing as 4 packed rows at dst
__device__ __forceinline__ void tma_gather4(uint32_t dst, const void *tmap, int32_t r0, int32_t r1, int32_t r2,
                                            int32_t r3, uint64_t *bar, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;"
                 ::"r"(dst), "l"(tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)), "l"(pol)
                 : "memory");
}
// 16-B global -> shared copy through L2 only (.cg: no L1 allocation), and
// the per-thread group commit / wait (sampled stream kernel's row gather)
__device__ __forceinline__ void cp16_g2s(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
#if SPFOM_L2_HINTS
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
#else
    (void)pol;
    bulk_g2s(dst, src, bytes, bar);
#endif
}
__device__ __forceinline__ void st256_stream(double *p, double a, double b, double c, double d) {
#if SPFOM_L2_HINTS
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
#else
    st256(p, a, b, c, d);
#endif
}

// shared-memory fp64 access through a 32-bit shared-window address (keeps
// ptxas from rebuilding the generic->shared conversion in predicated code)
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double x;
    asm("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a));
    return x;
}
// ordered variant for data this warp also writes (read-modify-write)
__device__ __forceinline__ double lds_f64_v(uint32_t a) {
    double x;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a) : "memory");
    return x;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double x) {
    asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(x) : "memory");
}
// Lane 0 claims the next work chunk (atomic add on a global counter); the
// result register is written by the predicated atomic itself and first read
// when the warp moves to that chunk, so nothing waits on the atomic's latency
// (a C-level `if (lane == 0) c = atomicAdd(..)` gets a merge right after it).
// The increment is written as lane + 1 (= 1 on lane 0): with a warp-uniform
// operand ptxas rewrites the atomic into its warp-aggregated form, whose
// shuffle of the result right after the atomic would wait for it.
__device__ __forceinline__ unsigned long long claim_chunk(unsigned long long *ctr, int lane) {
    unsigned long long c = 0;
    const unsigned long long inc = (unsigned long long)(lane + 1);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, 0;\n\t@p atom.global.add.u64 %0, [%2], %3;\n\t}"
                 : "+l"(c) : "r"(lane), "l"(ctr), "l"(inc) : "memory");
    return c;
}

// fp64 reduction into global memory under a predicate, without a branch
__device__ __forceinline__ void red_add_if(double *p, double v, bool pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p red.global.add.f64 [%0], %1;\n\t}"
                 :: "l"(p), "d"(v), "r"((int)pred) : "memory");
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

// ----------------------------------------------------------------- segment lists
// Segments processed by a launch: ids[first .. first+count) (local ids) or,
// ids == null, the contiguous range [first, first + count).  In sampled mode
// the list is the (iteration row, bin) slice of the block table, found from *t.
struct SegList {
    const int32_t *ids;
    int64_t first, count;
    const int32_t *row_off;      // sampled: [block_iters][nbins+1] offsets into ids
    int32_t bin, nbins;
    int64_t block_iters;
    int32_t head;                // K1: products [0, head) privatised in shared memory (0 = none)
};

// The launch's segment list resolved once: ids (null = contiguous from first) and count.
struct SegSpan {
    const int32_t *ids;
    int64_t first, count;
};
__device__ __forceinline__ SegSpan seg_span(const SegList &L, const DevState &S) {
    if (L.row_off) {
        const int64_t row = (*S.t) % L.block_iters;
        const int32_t *ro = L.row_off + row * (L.nbins + 1);
        const int64_t a = ro[L.bin], b = ro[L.bin + 1];
        return SegSpan{L.ids + a, 0, b - a};
    }
    return SegSpan{L.ids ? L.ids + L.first : nullptr, L.ids ? 0 : L.first, L.count};
}
__device__ __forceinline__ bool span_slot(const SegSpan &P, int64_t slot, int64_t &i) {
    if (slot >= P.count) return false;
    i = P.ids ? (int64_t)P.ids[slot] : P.first + slot;
    return true;
}
}  // namespace spfom
