// spfom.cu -- host side of the C ABI declared in include/spfom.h.
//
// create: validate (S:L34-36 + GAM rules) -> global column counts n_j (NCCL
// allreduce when world > 1) -> popularity relabelling of products (descending
// n_j) -> padded quad CSR (rows sorted by new id, padded to 4 entries with
// inert pads: v = omega = y = 0, id = N) -> length bins -> copy into the
// caller's workspace -> initial state (reading c10).
// step: CUDA-graph replay of one iteration (K1 per bin -> NCCL allreduce of
// the usage accumulator -> K3 [-> averaging] -> tick).
#include <cuda.h>            // CUtensorMap (encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <time.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <array>
#include <vector>

#include "spfom.h"
#include "spfom_kernels.cuh"

using namespace spfom;

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
typedef int nccl_res;                       // ncclResult_t
typedef struct { char internal[128]; } nccl_uid;
typedef void *nccl_comm;
enum { kNcclInt64 = 4, kNcclFloat64 = 8 };  // ncclDataType_t
enum { kNcclSum = 0, kNcclMax = 2 };        // ncclRedOp_t

struct NcclApi {
    bool ok = false;
    nccl_res (*GetUniqueId)(nccl_uid *) = nullptr;
    nccl_res (*CommInitRank)(nccl_comm *, int, nccl_uid, int) = nullptr;
    nccl_res (*AllReduce)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_res (*ReduceScatter)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_res (*AllGather)(const void *, void *, size_t, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_res (*CommDestroy)(nccl_comm) = nullptr;
    const char *(*GetErrorString)(nccl_res) = nullptr;
};
NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.GetUniqueId = (nccl_res(*)(nccl_uid *))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (nccl_res(*)(nccl_comm *, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
        api.AllReduce = (nccl_res(*)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
        api.CommDestroy = (nccl_res(*)(nccl_comm))dlsym(h, "ncclCommDestroy");
        api.ReduceScatter = (nccl_res(*)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclReduceScatter");
        api.AllGather = (nccl_res(*)(const void *, void *, size_t, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllGather");
        api.GetErrorString = (const char *(*)(nccl_res))dlsym(h, "ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy && api.ReduceScatter &&
                 api.AllGather;
    });
    return api;
}

thread_local std::string g_create_error;

// Large host arrays of create (pos_map, the per-segment state): uninitialised
// (every element is written by the layout loop; no serial zero-fill), freed
// with free().  (2 MiB-aligned transparent-huge-page advice was measured on the
// GPU hosts: no change in create or the getters, so none is given.)
struct FreeDel { void operator()(void *p) const { free(p); } };
template <class T>
static std::unique_ptr<T[], FreeDel> host_array(int64_t n) {
    return std::unique_ptr<T[], FreeDel>(static_cast<T *>(malloc((size_t)std::max<int64_t>(n, 1) * sizeof(T))));
}

// Pinned staging buffers (kPinQuads * 80 B, two per handle: create's H2D ring
// and the getters' D2H ring) come from a process-wide pool, so that a handle
// does not pay cudaMallocHost's page pinning when an earlier handle of the
// process already did.  A destroyed handle returns its buffers (after their
// last copy completed).  Pinned memory is portable across devices under
// unified addressing.  SPFOM_NO_PIN_POOL=1: a fresh allocation every time.
static std::mutex g_pin_mu;
static std::vector<void *> g_pin_free;
static cudaError_t pin_take(double **p, size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        if (!g_pin_free.empty() && !getenv("SPFOM_NO_PIN_POOL")) {
            *p = static_cast<double *>(g_pin_free.back());
            g_pin_free.pop_back();
            return cudaSuccess;
        }
    }
    return cudaMallocHost(reinterpret_cast<void **>(p), bytes);
}
static void pin_give(double *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(p);
}

// Bin = (G lanes per segment, Q quads per lane) -> capacity 4 G Q entries.
// E > 0: the full-sweep stream kernel maps E entries per lane on G lanes
// (rows of up to E G entries, StreamLayout); the other kernels use (G, Q).
#ifndef SPFOM_BIN_E
#define SPFOM_BIN_E 13   // G = 4: k = 49..52 entries exactly fill the lanes (the BASELINE k = 50 configs)
#endif
// Bins 2-4 are entry-mapped in the full-sweep stream kernel: E entries per lane
// on G = 4 / 8 / 16 lanes, rows of up to 52 / 104 / 208 entries (StreamLayout);
// every other kernel treats a bin as the quad mapping (G, Q).
#define SPFOM_BINS(X) X(0, 4, 1, 0) X(1, 4, 2, 0) X(2, 4, 4, SPFOM_BIN_E) X(3, 8, 4, SPFOM_BIN_E) \
    X(4, 16, 4, SPFOM_BIN_E) X(5, 32, 4, 0) X(6, 32, 8, 0)
struct BinCfg { int G, Q, E; };
#define SPFOM_BIN_INIT(B, G, Q, E) {G, Q, E},
constexpr BinCfg kBins[] = {SPFOM_BINS(SPFOM_BIN_INIT)};
#undef SPFOM_BIN_INIT
constexpr int kNumBins = sizeof(kBins) / sizeof(kBins[0]);
// Wide variant of a bin: the same quad capacity on G*Q lanes (<= 32) with one
// quad per lane -- shorter per-lane dependency chains for latency-bound launches.
constexpr int wide_g(int G, int Q) { return G * Q <= 32 ? G * Q : 32; }
constexpr int wide_q(int G, int Q) { return G * Q / wide_g(G, Q); }

#ifndef SPFOM_SAMP_G4
#define SPFOM_SAMP_G4 1   // sampled uniform bins: whole rows by TMA tile::gather4 (0: per-row bulk copies)
#endif
#ifndef SPFOM_SAMPLED_STREAM
#define SPFOM_SAMPLED_STREAM 1   // sampled blocks through the stream kernels (0: list kernels)
#endif
constexpr int64_t kMaxQuads = 4 * 32 * 8 / 4 * 1;  // 256 quads = 1024 entries

constexpr int64_t bin_cap(const BinCfg &c) { return c.E > 0 ? (int64_t)c.E * c.G / 4 : (int64_t)c.G * c.Q; }   // quads

int bin_of(int64_t nq) {
    for (int b = 0; b < kNumBins; ++b)
        if (nq <= bin_cap(kBins[b])) return b;
    return -1;
}

constexpr int kResidBlocks = 592;   // 4 x 148 SMs
#ifndef SPFOM_GRAPH_UNROLL
#define SPFOM_GRAPH_UNROLL 4
#endif
constexpr int kGraphUnroll = SPFOM_GRAPH_UNROLL;   // iterations per CUDA graph in spfom_step (k >= this)

// Per-device launch facts (opt-in shared memory set on the kernel, occupancy):
// cudaFuncSetAttribute applies to the current device's context only, so a
// process driving several GPUs needs one entry per device.
constexpr int kMaxDevices = 64;
struct PerDevice {
    int v[kMaxDevices];
    PerDevice() { for (int &x : v) x = -1; }
    // the slot of the current device (devices past kMaxDevices share a
    // sentinel that is never cached: the caller re-queries every time)
    int *slot() {
        static thread_local int scratch;
        int d = 0;
        cudaGetDevice(&d);
        if (d >= 0 && d < kMaxDevices) return &v[d];
        scratch = -1;
        return &scratch;
    }
};

// Makes the handle's device current for the duration of an entry point.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Plan {
    int64_t m = 0, N = 0, nq = 0, T = 1;   // m, nq: base segments / quads; T periods (shared structure)
    int64_t bin_count[kNumBins] = {0};
    double bin_work[kNumBins] = {0};   // sampled: mean over block rows of the bin's padded quads + rows
    int64_t block_entries = 0;      // total local sampled ids
    bool sampled = false;
    bool averaging = false;
    size_t off[40] = {0};
    size_t total = 0;
};

enum Slot {
    O_PIDX, O_V, O_OM, O_Y, O_YBAR, O_QOFF, O_SEGC, O_SEGV, O_Y0BAR, O_R, O_C, O_TAU, O_ETA, O_G,
    O_ACC, O_SCUR, O_ETABAR, O_TMP, O_BLKIDS, O_ROWOFF, O_RESSEG, O_RESPROD, O_COUNTERS, O_T,
    O_COUNTS, O_RECORD, O_RECALPHA, O_ORIG, O_BPTR, O_BRES, O_RPTR, O_RBUN, O_STILDE, O_RESRES, O_WORK, O_TMAPS, O_SEGD, O_NSLOTS
};

constexpr int kSpreadCopies = SPFOM_SPREAD_C;
#ifndef SPFOM_SPREAD_N
#define SPFOM_SPREAD_N 16384
#endif
int64_t spread_range(int64_t N) { return kSpreadCopies > 0 ? std::min<int64_t>(N, SPFOM_SPREAD_N) : 0; }
// Product vectors hold N + 1 slots (slot N: the pads' dummy product) plus
// kRankPad, so that with world P <= kRankPad the padded length round_up(N + 1,
// P) that ReduceScatter / AllGather split into P equal slices fits.
constexpr int64_t kRankPad = 64;
int64_t prod_slots(int64_t N) { return N + 1 + kRankPad; }
int64_t spread_off(int64_t N) { return (prod_slots(N) + 31) / 32 * 32; }   // first spread slot after the acc slots

// pinned staging ring of a handle: 2 buffers of kPinQuads quads x 80 B (ids +
// v + omega at create; the getters' D2H uses 32 B per quad of it)
constexpr int64_t kPinQuads = (int64_t)1 << 18;
static_assert(kPinQuads >= kMaxQuads, "a chunk holds at least one row");

int64_t recover_chunk(int64_t nq) { return std::min<int64_t>(std::max<int64_t>(4 * nq, 4096), (int64_t)1 << 22); }

void make_plan(const spfom_instance *in, const spfom_params *p, Plan &pl) {
    pl.m = in->num_segments;
    pl.N = in->num_products;
    pl.T = std::max<int64_t>(1, in->num_periods);
    pl.nq = 0;
    for (int64_t i = 0; i < pl.m; ++i) {
        int64_t k = in->seg_ptr[i + 1] - in->seg_ptr[i];
        int64_t q = (k + 3) / 4;
        pl.nq += q;
        int b = bin_of(q);
        if (b >= 0) pl.bin_count[b] += 1;
    }
    pl.sampled = p && p->blocks != nullptr;
    pl.averaging = p && p->averaging;
    pl.block_entries = pl.sampled ? p->block_iters * p->block_size : 0;
    const int64_t nq = std::max<int64_t>(pl.nq, 1), m = std::max<int64_t>(pl.m, 1), N1 = prod_slots(pl.N), T = pl.T;
    size_t sz[O_NSLOTS] = {0};
    sz[O_PIDX] = nq * 16;
    sz[O_V] = sz[O_OM] = nq * 32;
    sz[O_Y] = T * nq * 32;                    // [T][nq] quads
    sz[O_YBAR] = pl.averaging ? T * nq * 32 : 0;
    sz[O_QOFF] = (m + 1 + 64) * 4;           // + slack: K1's 16-B qoff windows may read past the end
    sz[O_SEGC] = T * m * 16;                  // [T][m]
    sz[O_SEGV] = T * m * 32;
    sz[O_SEGD] = T * m * 16;                  // float4 [T][m]
    sz[O_Y0BAR] = pl.averaging ? T * m * 8 : 0;
    const int64_t L = std::max<int64_t>(0, in->num_resources);
    const int64_t D1 = std::max<int64_t>(N1, L + 1);       // duals: products or resources
    sz[O_R] = sz[O_G] = sz[O_SCUR] = sz[O_TMP] = N1 * 8;
    sz[O_C] = sz[O_TAU] = sz[O_ETA] = D1 * 8;
    const int64_t nb = L > 0 ? in->bundle_ptr[pl.N] : 0;
    sz[O_BPTR] = L > 0 ? N1 * 4 + 4 : 4;
    sz[O_BRES] = sz[O_RBUN] = std::max<int64_t>(nb, 1) * 4;
    sz[O_RPTR] = (L + 2) * 4;
    sz[O_STILDE] = L > 0 ? N1 * 8 : 8;
    sz[O_RESRES] = (size_t)kResidBlocks * 8 * 8;
    sz[O_ACC] = (spread_off(pl.N) + (size_t)kSpreadCopies * spread_range(pl.N)) * 8;   // acc, then spread copies
    sz[O_ETABAR] = pl.averaging ? D1 * 8 : 0;

    sz[O_BLKIDS] = std::max<int64_t>(pl.block_entries, 1) * 4;
    sz[O_ROWOFF] = pl.sampled ? p->block_iters * (kNumBins + 1) * 4 : 4;
    sz[O_RESSEG] = (size_t)kNumBins * kResidBlocks * 4 * 8;
    sz[O_RESPROD] = (size_t)kResidBlocks * 8 * 8;
    sz[O_COUNTERS] = 8 * 8;
    sz[O_T] = 8;
    sz[O_WORK] = 16 * kNumBins;  // K1 stream: dynamic round-chunk counter + exited-block count, per bin
    sz[O_TMAPS] = pl.sampled ? (size_t)kNumBins * 6 * sizeof(CUtensorMap) : 0;   // sampled uniform bins: gather4 maps
    sz[O_COUNTS] = N1 * 8;
    // recovery scratch (spfom_recover works in chunks of at most recover_chunk() padded entries)
    sz[O_RECORD] = (size_t)recover_chunk(pl.nq) * 4;
    sz[O_RECALPHA] = (size_t)recover_chunk(pl.nq) * 2 * 8;
    sz[O_ORIG] = N1 * 4;
    size_t o = 0;
    for (int s = 0; s < O_NSLOTS; ++s) {
        pl.off[s] = o;
        o += align256(sz[s]);
    }
    pl.total = o;
}
}  // namespace

// ------------------------------------------------------------------ handle
struct spfom_handle {
    Plan pl;
    spfom_params params;
    int rank = 0, world = 1;
    nccl_comm comm = nullptr;
    cudaStream_t stream = nullptr;
    char *ws = nullptr;
    DevState S;
    int64_t nq = 0, m = 0, N = 0, nnz = 0, n_present = 0, T = 1;   // base quads / segments / entries; periods
    int64_t L = 0;                                                  // resources (bundles / NRM), 0 = none
    std::vector<int32_t> bptr_h, bres_h;                            // relabelled bundle CSR (set_state)
    std::vector<int32_t> new2old, old2new;     // products
    std::unique_ptr<int32_t[], FreeDel> pos_map;   // original entry -> padded entry [nnz] (no zero-fill; < 2^31 by validation)
    std::vector<int32_t> sorder;               // device segment slot -> local segment (bin order)
    std::vector<int64_t> seg_off;              // original CSR offsets (base rows) [m + 1]
    std::vector<int32_t> qoff_h;               // device-order quad offsets [m + 1] (host copy)
    bool bin_uniform[kNumBins] = {false};      // entry-mapped bin whose rows all have exactly E quads
    const void *bin_tmaps[kNumBins] = {nullptr};   // sampled uniform bins: 6 gather4 tensor maps (device)
    double *pin[2] = {nullptr, nullptr};       // pinned D2H staging ring (getters), allocated on first use
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    std::vector<int32_t> bin_first;            // [kNumBins+1] first device slot of each bin
    int64_t iter = 0;
    cudaGraphExec_t graph = nullptr, graph_refresh = nullptr;
    cudaGraphExec_t graph_u = nullptr;         // kGraphUnroll iterations in one graph (no refresh)
    cudaGraphExec_t graph_primal = nullptr, graph_rest = nullptr, graph_rest_refresh = nullptr;   // split form (refresh iterations of spfom_step_timed)
    // timed form: the iteration graph with an event-record node before and after
    // the primal kernels; spfom_step_timed points them at fresh events per launch
    // timed form: c iterations in one graph, event-record nodes before and after
    // the primal kernels of each and one after the last (events owned here);
    // built on first use per chunk size c, kept for the handle's lifetime
    struct TimedGraph {
        int64_t iters = 0;
        cudaGraphExec_t exec = nullptr;
        std::vector<cudaEvent_t> ev;   // [2 iters + 1]
    };
    std::vector<TimedGraph> timed;
    std::string err;
    int sm_count = 148;
    // world > 1 (plain products): ReduceScatter -> K3 on the slice -> AllGather
    // of g; the product vectors are split into world slices of `chunk`
    bool rs = false;
    int64_t chunk = 0, np = 0;
    int device = 0;                            // every entry point runs with this device current
    bool own_stream = false;
    // full sweep with several non-empty bins: one side stream per bin, SM share per bin
    int nbins_active = 0;
    int bin_sms[kNumBins] = {0};
    cudaStream_t side[kNumBins] = {nullptr};
    cudaEvent_t ev_fork = nullptr, ev_join[kNumBins] = {nullptr};
    // small regime: persistent cooperative kernel, whole iterations per launch
    bool small = false;
    int small_q = 1, small_blocks = 0;
};

namespace {
spfom_status fail(spfom_handle *h, spfom_status st, const std::string &msg) {
    if (h) h->err = msg; else g_create_error = msg;
    return st;
}
#define CUDA_TRY(h, expr)                                                                          \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(h, SPFOM_ECUDA, std::string(#expr ": ") + cudaGetErrorString(e_));          \
    } while (0)

template <typename T>
T *slot_ptr(spfom_handle *h, int s) { return reinterpret_cast<T *>(h->ws + h->pl.off[s]); }

spfom_status allreduce(spfom_handle *h, const void *src, void *dst, size_t n, int dtype, int op) {
    if (!h->comm) {
        if (src != dst) CUDA_TRY(h, cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToDevice, h->stream));
        return SPFOM_OK;
    }
    nccl_res r = nccl().AllReduce(src, dst, n, dtype, op, h->comm, h->stream);
    if (r != 0) return fail(h, SPFOM_ENCCL, std::string("ncclAllReduce: ") + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
    return SPFOM_OK;
}

// rs mode: make a sliced product vector (eta, s_prev, etabar) whole on every
// rank (collective; in place)
spfom_status gather_slices(spfom_handle *h, double *v) {
    if (!h->rs) return SPFOM_OK;
    nccl_res r = nccl().AllGather(v + h->rank * h->chunk, v, (size_t)h->chunk, kNcclFloat64, h->comm, h->stream);
    if (r != 0) return fail(h, SPFOM_ENCCL, std::string("ncclAllGather: ") + nccl().GetErrorString(r));
    return SPFOM_OK;
}

// Persistent grid: at most (resident blocks per SM) x SMs blocks, each looping
// over segments; the Zipf head is privatised only when a block sees enough
// segments to amortise its flush (H REDs per block).
template <int G, int Q, bool ARGMAX, bool SAMPLED>
void launch_primal(const DevState &S, SegList L, int64_t max_count, int sm_count, cudaStream_t st) {
    static PerDevice cache;
    int &resident = *cache.slot();
    constexpr size_t smem = sizeof(ListSmem<Q, G>);
    if (resident < 0) {
        cudaFuncSetAttribute(k_primal<G, Q, ARGMAX, SAMPLED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_primal<G, Q, ARGMAX, SAMPLED>, kPrimalThreads, smem);
        resident = std::max(resident, 1);
    }
    const int64_t groups_per_block = kPrimalThreads / G;
    int64_t blocks = (max_count + groups_per_block - 1) / groups_per_block;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count * resident));
    const int64_t segs_per_block = (max_count + blocks - 1) / blocks;
    L.head = (segs_per_block >= 64) ? (int32_t)std::min<int64_t>(kHeadMax, S.N) : 0;
    k_primal<G, Q, ARGMAX, SAMPLED><<<(unsigned)blocks, kPrimalThreads, smem, st>>>(S, L);
}

// Full sweep of a contiguous bin: one persistent 12-warp block per SM; the
// rest of the opt-in shared memory stages the head of g.
template <int G, int Q, bool ARGMAX, int EQ = 0, bool UNI = false, bool SAMP = false>
void launch_stream(const DevState &S, StreamList L, int sm_count, cudaStream_t st) {
    using LY = StreamLayout<G, Q, EQ, SAMP && UNI>;
    static PerDevice cache;
    int &hg_cap = *cache.slot();
    constexpr size_t fixed = stream_smem_fixed<G, Q, EQ, SAMP, UNI>();
    if (hg_cap < 0) {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        hg_cap = (int)std::min<int64_t>(kGHeadStreamMax, std::max<int64_t>(0, ((int64_t)optin - (int64_t)fixed) / 8 / 32 * 32));
        cudaFuncSetAttribute(k_primal_stream<G, Q, ARGMAX, EQ, UNI, SAMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(fixed + (size_t)hg_cap * 8));
    }
    L.ghead = (int32_t)std::min<int64_t>(hg_cap, S.N + 1);
    L.hh = (int32_t)std::min<int64_t>(LY::HH, S.N);
    const int64_t rounds = (L.count + LY::GPW - 1) / LY::GPW;
    constexpr int W = LY::WARPS;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(sm_count, (rounds + W - 1) / W));
    k_primal_stream<G, Q, ARGMAX, EQ, UNI, SAMP><<<(unsigned)blocks, 32 * W, fixed + (size_t)L.ghead * 8, st>>>(S, L);
}

// Multi-period shared structure: units = rounds x T over one persistent block per SM.
template <int G, int Q, bool ARGMAX, int EQ = 0>
void launch_mp(const DevState &S, StreamList L, int sm_count, cudaStream_t st) {
    using LY = MPLayout<G, Q, EQ>;
    static PerDevice cache;
    int &hg_cap = *cache.slot();
    constexpr size_t fixed = mp_smem_fixed<G, Q, EQ>();
    if (hg_cap < 0) {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        hg_cap = (int)std::min<int64_t>(kGHeadStreamMax, std::max<int64_t>(0, ((int64_t)optin - (int64_t)fixed) / 8 / 32 * 32));
        cudaFuncSetAttribute(k_primal_mp<G, Q, ARGMAX, EQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(fixed + (size_t)hg_cap * 8));
    }
    L.ghead = (int32_t)std::min<int64_t>(hg_cap, S.N + 1);
    L.hh = 0;
    constexpr int W = LY::WARPS;
    const int64_t rounds = (L.count + LY::GPW - 1) / LY::GPW;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(sm_count, (rounds + W - 1) / W));
    k_primal_mp<G, Q, ARGMAX, EQ><<<(unsigned)blocks, 32 * W, fixed + (size_t)L.ghead * 8, st>>>(S, L);
}

void mp_dispatch(int b, bool argmax, const DevState &S, const StreamList &L, int sms, cudaStream_t st) {
    switch (b) {
#define CASE(B, G, Q, E)                                                                   \
    case B:                                                                                \
        if constexpr (Q <= 4) {                                                            \
            constexpr int EM = G == 4 ? E : 0;   /* shared periods: entry mapping on 4 lanes only */ \
            if (argmax) launch_mp<G, Q, true, EM>(S, L, sms, st);                          \
            else launch_mp<G, Q, false, EM>(S, L, sms, st);                                \
        }                                                                                  \
        break;
        SPFOM_BINS(CASE)
#undef CASE
    }
}

// Throughput config unless the bin gives each warp fewer than two rounds.
template <int G, int Q>
bool prefer_wide(int64_t count, int sms) {
    const int64_t rounds = (count + StreamLayout<G, Q>::GPW - 1) / StreamLayout<G, Q>::GPW;
    return rounds < 2 * (int64_t)sms * StreamLayout<G, Q>::WARPS;
}

// SAMP: the same kernels over this iteration's block list (sampled blocks).
template <bool SAMP = false>
void stream_dispatch(int b, bool argmax, const DevState &S, const StreamList &L, int sms, cudaStream_t st) {
    switch (b) {
#define CASE(B, G, Q, E)                                                                   \
    case B:                                                                                \
        if constexpr (Q <= 4) {                                                            \
            constexpr int WG = wide_g(G, Q), WQ = wide_q(G, Q);                            \
            if (prefer_wide<G, Q>(L.count, sms) && (WG != G)) {                            \
                if (argmax) launch_stream<WG, WQ, true, 0, false, SAMP>(S, L, sms, st);    \
                else launch_stream<WG, WQ, false, 0, false, SAMP>(S, L, sms, st);          \
            } else if constexpr (E > 0 && G == 4) {                                        \
                if (L.uni) {                                                               \
                    if (argmax) launch_stream<G, Q, true, E, true, SAMP>(S, L, sms, st);   \
                    else launch_stream<G, Q, false, E, true, SAMP>(S, L, sms, st);         \
                } else if (argmax) launch_stream<G, Q, true, E, false, SAMP>(S, L, sms, st); \
                else launch_stream<G, Q, false, E, false, SAMP>(S, L, sms, st);           \
            } else if (argmax) launch_stream<G, Q, true, E, false, SAMP>(S, L, sms, st);   \
            else launch_stream<G, Q, false, E, false, SAMP>(S, L, sms, st);                \
        }                                                                                  \
        break;
        SPFOM_BINS(CASE)
#undef CASE
    }
}

// Segment lists (sampled blocks, rows > 512 entries): register-direct loads,
// latency-bound launches -> the wide mapping (one quad per lane up to 32 lanes).
void primal_dispatch(int b, bool argmax, bool sampled, const DevState &S, const SegList &L, int64_t cnt, int sms,
                     cudaStream_t st) {
    switch (b) {
#define CASE(B, G, Q, E)                                                                   \
    case B: {                                                                              \
        constexpr int WG = wide_g(G, Q), WQ = wide_q(G, Q);                                \
        if (argmax) {                                                                      \
            if (sampled) launch_primal<WG, WQ, true, true>(S, L, cnt, sms, st);            \
            else launch_primal<WG, WQ, true, false>(S, L, cnt, sms, st);                   \
        } else {                                                                           \
            if (sampled) launch_primal<WG, WQ, false, true>(S, L, cnt, sms, st);           \
            else launch_primal<WG, WQ, false, false>(S, L, cnt, sms, st);                  \
        }                                                                                  \
        break;                                                                             \
    }
        SPFOM_BINS(CASE)
#undef CASE
    }
}

void resid_dispatch(int b, const DevState &S, const SegList &L, double *part, int64_t seg_off, int64_t quad_off,
                    cudaStream_t st) {
    switch (b) {
#define CASE(B, G, Q, E) case B: k_resid_seg<G, Q><<<kResidBlocks, kThreads, 0, st>>>(S, L, part, seg_off, quad_off); break;
        SPFOM_BINS(CASE)
#undef CASE
    }
}

// Enqueue one iteration (used under stream capture).  refresh: sampled-mode
// fresh recompute of s = A y before the dual step.
// Sampled blocks on uniform bins (every row E quads): 2-D tensor maps over the
// bin's rows for TMA tile::gather4 -- ids / v / omega / y as [rows][4 E]
// (row pitch 16 E / 32 E bytes), segv [rows][4], segc [rows][2]; box {cols, 1}.
// Without the driver's encoder (or if it rejects a map) the bin keeps the
// per-row bulk copies.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
spfom_status encode_gather_maps(spfom_handle *h) {
    static EncodeTiledFn enc = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q{};
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            enc = reinterpret_cast<EncodeTiledFn>(fn);
    });
    if (!enc) return SPFOM_OK;
    const DevState &S = h->S;
    std::vector<CUtensorMap> maps((size_t)kNumBins * 6);
    bool any = false;
    for (int b = 0; b < kNumBins; ++b) {
        const int64_t rows = h->bin_first[b + 1] - h->bin_first[b];
        if (!h->bin_uniform[b] || rows == 0 || kBins[b].E == 0) continue;
        const int E = kBins[b].E;
        const int64_t first = h->bin_first[b], q0 = h->qoff_h[first];
        struct A { CUtensorMapDataType dt; void *base; cuuint64_t cols, pitch; };
        const A arr[6] = {{CU_TENSOR_MAP_DATA_TYPE_INT32, (void *)(S.pidx + q0), (cuuint64_t)4 * E, (cuuint64_t)16 * E},
                          {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (void *)(S.v + 4 * q0), (cuuint64_t)4 * E, (cuuint64_t)32 * E},
                          {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (void *)(S.om + 4 * q0), (cuuint64_t)4 * E, (cuuint64_t)32 * E},
                          {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (void *)(S.y + 4 * q0), (cuuint64_t)4 * E, (cuuint64_t)32 * E},
                          {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (void *)(S.segv + first), 4, 32},
                          {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (void *)(S.segc + first), 2, 16}};
        bool ok = true;
        for (int a = 0; a < 6 && ok; ++a) {
            const cuuint64_t dims[2] = {arr[a].cols, (cuuint64_t)rows};
            const cuuint64_t strides[1] = {arr[a].pitch};
            const cuuint32_t box[2] = {(cuuint32_t)arr[a].cols, 1}, es[2] = {1, 1};
            ok = enc(&maps[(size_t)b * 6 + a], arr[a].dt, 2, arr[a].base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        if (!ok) continue;
        h->bin_tmaps[b] = slot_ptr<unsigned char>(h, O_TMAPS) + (size_t)b * 6 * sizeof(CUtensorMap);
        any = true;
    }
    if (any) {
        CUDA_TRY(h, cudaMemcpyAsync(slot_ptr<unsigned char>(h, O_TMAPS), maps.data(), maps.size() * sizeof(CUtensorMap),
                                    cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    }
    return SPFOM_OK;
}

// a1-a5: the primal kernels, one launch per non-empty length bin
spfom_status enqueue_primal(spfom_handle *h, int64_t *launches) {
    const bool argmax = std::isinf(h->params.theta);
    DevState S = h->S;
    int64_t nl = 0;
    const bool fork = h->nbins_active > 1;
    if (fork) {
        CUDA_TRY(h, cudaEventRecord(h->ev_fork, h->stream));
        for (int b = 0; b < kNumBins; ++b)
            if (h->side[b]) CUDA_TRY(h, cudaStreamWaitEvent(h->side[b], h->ev_fork, 0));
    }
    for (int b = 0; b < kNumBins; ++b) {
        SegList L{};
        L.bin = b;
        L.nbins = kNumBins;
        int64_t maxc = 0;
        if (h->pl.sampled) {
            L.ids = slot_ptr<int32_t>(h, O_BLKIDS);
            L.row_off = slot_ptr<int32_t>(h, O_ROWOFF);
            L.block_iters = h->params.block_iters;
            maxc = h->pl.bin_count[b] > 0 ? std::min<int64_t>(h->pl.bin_count[b], h->params.block_size) : 0;
            if (SPFOM_SAMPLED_STREAM && maxc > 0 && kBins[b].Q <= 4 && h->T == 1) {
                // the block's rows of this bin gathered into the stream kernel's slots
                StreamList SL{};
                SL.first = h->bin_first[b];
                SL.count = maxc;
                SL.work = slot_ptr<unsigned long long>(h, O_WORK) + 2 * b;
                SL.uni = h->bin_uniform[b] ? 1 : 0;
                SL.qbase = h->qoff_h[h->bin_first[b]];
                SL.ids = L.ids;
                SL.row_off = L.row_off;
                SL.bin = b;
                SL.nbins = kNumBins;
                SL.block_iters = L.block_iters;
                SL.tm = h->bin_tmaps[b];
                const int sms = h->nbins_active > 1 ? h->bin_sms[b] : h->sm_count;
                stream_dispatch<true>(b, argmax, S, SL, sms, h->nbins_active > 1 ? h->side[b] : h->stream);
                ++nl;
                continue;
            }
        } else {
            // full sweep: the bin is the contiguous device range [bin_first[b], bin_first[b+1])
            const int64_t cnt = h->bin_first[b + 1] - h->bin_first[b];
            if (cnt == 0) continue;
            if (kBins[b].Q <= 4) {
                StreamList SL{};
                SL.first = h->bin_first[b];
                SL.count = cnt;
                SL.work = slot_ptr<unsigned long long>(h, O_WORK) + 2 * b;   // reset by the launch's last block
                SL.uni = h->bin_uniform[b] ? 1 : 0;
                SL.qbase = h->qoff_h[h->bin_first[b]];
                // several bins: concurrent persistent kernels on disjoint SM shares
                // (forked streams; inside a graph they become parallel branches)
                const int sms = h->nbins_active > 1 ? h->bin_sms[b] : h->sm_count;
                cudaStream_t st = h->nbins_active > 1 ? h->side[b] : h->stream;
                if (h->T > 1) mp_dispatch(b, argmax, S, SL, sms, st);
                else stream_dispatch(b, argmax, S, SL, sms, st);
                ++nl;
                continue;
            }
            L.ids = nullptr;
            L.first = h->bin_first[b];
            L.count = cnt;
            maxc = cnt;
        }
        if (maxc == 0) continue;
        primal_dispatch(b, argmax, h->pl.sampled, S, L, maxc, fork ? h->bin_sms[b] : h->sm_count,
                        fork ? h->side[b] : h->stream);
        ++nl;
    }
    if (fork) {
        for (int b = 0; b < kNumBins; ++b)
            if (h->side[b]) {
                CUDA_TRY(h, cudaEventRecord(h->ev_join[b], h->side[b]));
                CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_join[b], 0));
            }
    }
    CUDA_TRY(h, cudaGetLastError());
    if (launches) *launches = nl;
    return SPFOM_OK;
}

// a6-a8: allreduce of the usage accumulator, dual step, averaging, tick
spfom_status enqueue_rest(spfom_handle *h, bool refresh, int64_t *launches) {
    DevState S = h->S;
    int64_t nl = 0;
    double *acc = slot_ptr<double>(h, O_ACC);
    int full_mode = h->pl.sampled ? 0 : 1;
    if (refresh) {
        CUDA_TRY(h, cudaMemsetAsync(acc, 0, (h->N + 1) * 8, h->stream));
        if (S.spread_n > 0)
            CUDA_TRY(h, cudaMemsetAsync(S.spread, 0, (size_t)S.spread_c * S.spread_n * 8, h->stream));
        k_usage<<<h->sm_count * 4, kThreads, 0, h->stream>>>(S, h->T * h->nq, acc, (int32_t)std::min<int64_t>(kHeadMax, h->N));
        full_mode = 1;
        ++nl;
    }
#ifdef SPFOM_DIAG_SEP_USAGE
    // diagnostic: the usage of the iteration recomputed from y (K1's scatter off or discarded)
    CUDA_TRY(h, cudaMemsetAsync(acc, 0, (h->N + 1) * 8, h->stream));
    if (S.spread_n > 0) CUDA_TRY(h, cudaMemsetAsync(S.spread, 0, (size_t)S.spread_c * S.spread_n * 8, h->stream));
    k_usage<<<h->sm_count * 4, kThreads, 0, h->stream>>>(S, h->T * h->nq, acc, (int32_t)std::min<int64_t>(kHeadMax, h->N));
#endif
    if (h->comm && S.spread_n > 0) {
        // fold the spread copies into acc before the cross-rank sum
        k_fold<<<std::max<int64_t>(1, (S.spread_n + kThreads - 1) / kThreads), kThreads, 0, h->stream>>>(S);
        ++nl;
    }
    if (h->rs) {
        // a6 + a7 split over the ranks: sum only this rank's slice of the usage,
        // update its duals, share the prices
        const int64_t lo = h->rank * h->chunk;
        nccl_res r = nccl().ReduceScatter(acc, acc + lo, (size_t)h->chunk, kNcclFloat64, kNcclSum, h->comm, h->stream);
        if (r != 0) return fail(h, SPFOM_ENCCL, std::string("ncclReduceScatter: ") + nccl().GetErrorString(r));
        const unsigned gs = (unsigned)std::max<int64_t>(1, std::min<int64_t>((h->np + kThreads - 1) / kThreads, h->sm_count * 8));
        k_dual_slice<<<gs, kThreads, 0, h->stream>>>(S, full_mode, h->pl.averaging ? 0 : 1, lo, h->chunk, h->np);
        r = nccl().AllGather(S.g + lo, S.g, (size_t)h->chunk, kNcclFloat64, h->comm, h->stream);
        if (r != 0) return fail(h, SPFOM_ENCCL, std::string("ncclAllGather: ") + nccl().GetErrorString(r));
        if (h->pl.averaging) k_average<<<h->sm_count * 8, kThreads, 0, h->stream>>>(S, h->T * h->nq);
        if (h->pl.averaging) k_tick<<<1, 1, 0, h->stream>>>(S.t);
        nl += 1 + (h->pl.averaging ? 2 : 0);
        CUDA_TRY(h, cudaGetLastError());
        if (launches) *launches = nl;
        return SPFOM_OK;
    }
    spfom_status st = allreduce(h, acc, acc, (size_t)h->N, kNcclFloat64, kNcclSum);
    if (st != SPFOM_OK) return st;
    // K3: s_new = full ? acc : s_cur + acc
    const unsigned gN = (unsigned)std::max<int64_t>(1, std::min<int64_t>((h->N + kThreads - 1) / kThreads, h->sm_count * 8));
    if (h->L > 0) {
        // bundles: per-bundle usage -> per-resource dual step -> bundle prices (+ tick)
        const unsigned gL = (unsigned)std::max<int64_t>(1, std::min<int64_t>((h->L + kThreads - 1) / kThreads, h->sm_count * 8));
        k_bundle_usage<<<gN, kThreads, 0, h->stream>>>(S, full_mode);
        k_bundle_dual<<<gL, kThreads, 0, h->stream>>>(S, h->pl.averaging ? 1 : 0);
        k_bundle_prices<<<gN, kThreads, 0, h->stream>>>(S, h->pl.averaging ? 0 : 1);
        nl += 2;
    } else {
        k_dual<<<gN, kThreads, 0, h->stream>>>(S, full_mode, h->pl.averaging ? 0 : 1);
    }
    if (h->pl.averaging) k_average<<<h->sm_count * 8, kThreads, 0, h->stream>>>(S, h->T * h->nq);
    if (h->pl.averaging) k_tick<<<1, 1, 0, h->stream>>>(S.t);   // else k_dual ticks
    nl += 1 + (h->pl.averaging ? 2 : 0);
    CUDA_TRY(h, cudaGetLastError());
    if (launches) *launches = nl;
    return SPFOM_OK;
}

spfom_status enqueue_iteration(spfom_handle *h, bool refresh) {
    spfom_status st = enqueue_primal(h, nullptr);
    return st != SPFOM_OK ? st : enqueue_rest(h, refresh, nullptr);
}

// part: 0 = whole iteration, 1 = primal kernels only, 2 = the rest
spfom_status build_graph(spfom_handle *h, bool refresh, cudaGraphExec_t *out, int part = 0, int iters = 1) {
    cudaGraph_t g;
    CUDA_TRY(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    spfom_status st = SPFOM_OK;
    for (int it = 0; it < iters && st == SPFOM_OK; ++it)
        st = part == 0 ? enqueue_iteration(h, refresh)
           : part == 1 ? enqueue_primal(h, nullptr) : enqueue_rest(h, refresh, nullptr);
    cudaGraph_t gg;
    cudaError_t e = cudaStreamEndCapture(h->stream, &gg);
    if (st != SPFOM_OK) return st;
    if (e != cudaSuccess) return fail(h, SPFOM_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    g = gg;
    e = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, SPFOM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    return SPFOM_OK;
}

// The timed graph of c iterations: per iteration, event record -> primal
// kernels -> event record -> the rest (no refresh); a final event record.
// cudaEventRecordExternal makes the records event-record nodes (a plain
// record inside a capture only orders streams).  Its events are fixed, so a
// launch needs no graph update.
spfom_status timed_graph(spfom_handle *h, int64_t c, spfom_handle::TimedGraph **out) {
    for (auto &tg : h->timed)
        if (tg.iters == c) {
            *out = &tg;
            return SPFOM_OK;
        }
    spfom_handle::TimedGraph tg;
    tg.iters = c;
    tg.ev.assign(2 * c + 1, nullptr);
    auto cleanup = [&]() {
        for (cudaEvent_t e : tg.ev)
            if (e) cudaEventDestroy(e);
    };
    for (auto &e : tg.ev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            cleanup();
            return fail(h, SPFOM_ECUDA, "timed graph: event create");
        }
    if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cleanup();
        return fail(h, SPFOM_ECUDA, "timed graph: begin capture");
    }
    spfom_status st = SPFOM_OK;
    auto rec = [&](cudaEvent_t e) {
        if (st == SPFOM_OK && cudaEventRecordWithFlags(e, h->stream, cudaEventRecordExternal) != cudaSuccess)
            st = fail(h, SPFOM_ECUDA, "timed graph: event record");
    };
    for (int64_t it = 0; it < c && st == SPFOM_OK; ++it) {
        rec(tg.ev[2 * it]);
        if (st == SPFOM_OK) st = enqueue_primal(h, nullptr);
        rec(tg.ev[2 * it + 1]);
        if (st == SPFOM_OK) st = enqueue_rest(h, false, nullptr);
    }
    rec(tg.ev[2 * c]);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (st == SPFOM_OK && e != cudaSuccess) st = fail(h, SPFOM_ECUDA, std::string("timed graph capture: ") + cudaGetErrorString(e));
    if (st == SPFOM_OK && cudaGraphInstantiate(&tg.exec, g, 0) != cudaSuccess) st = fail(h, SPFOM_ECUDA, "timed graph: instantiate");
    if (g) cudaGraphDestroy(g);
    if (st != SPFOM_OK) {
        cleanup();
        return st;
    }
    h->timed.push_back(std::move(tg));
    *out = &h->timed.back();
    return SPFOM_OK;
}

void destroy_timed(spfom_handle *h) {
    for (auto &tg : h->timed) {
        if (tg.exec) cudaGraphExecDestroy(tg.exec);
        for (cudaEvent_t e : tg.ev)
            if (e) cudaEventDestroy(e);
    }
    h->timed.clear();
}

// ------------------------------------------------------------------ device-resident instances
// spfom_instance.on_device = 1: the arrays are device pointers (e.g. torch
// tensors); the layout build is a host pass, so they are staged to host
// memory first and the rest of create runs on the staged copy.
struct StagedInstance {
    spfom_instance in{};
    std::vector<int64_t> seg_ptr, bundle_ptr;
    std::vector<int32_t> prod_idx, bundle_res;
    std::vector<double> attract, shadow, no_purchase, arrival, price, capacity, resource_capacity;
};
template <typename T>
bool stage_array(std::vector<T> &dst, const T *src, int64_t n) {
    if (!src || n <= 0) return true;
    dst.resize((size_t)n);
    return cudaMemcpy(dst.data(), src, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost) == cudaSuccess;
}
// in points at caller device memory; on success out.in points at host copies
spfom_status stage_instance(const spfom_instance *in, StagedInstance &out) {
    out.in = *in;
    out.in.on_device = 0;
    const int64_t m = in->num_segments, N = in->num_products, T = std::max<int64_t>(1, in->num_periods);
    if (m < 0 || N < 1 || in->nnz < 0 || !in->seg_ptr) return fail(nullptr, SPFOM_EINVAL, "instance: missing array or bad size");
    bool ok = stage_array(out.seg_ptr, in->seg_ptr, m + 1) && stage_array(out.prod_idx, in->prod_idx, in->nnz) &&
              stage_array(out.attract, in->attract, in->nnz) && stage_array(out.shadow, in->shadow, in->nnz) &&
              stage_array(out.no_purchase, in->no_purchase, m) && stage_array(out.arrival, in->arrival, T * m) &&
              stage_array(out.price, in->price, N) && stage_array(out.capacity, in->capacity, N);
    if (ok && in->num_resources > 0 && in->bundle_ptr) {
        ok = stage_array(out.bundle_ptr, in->bundle_ptr, N + 1) &&
             stage_array(out.resource_capacity, in->resource_capacity, in->num_resources);
        if (ok && !out.bundle_ptr.empty()) ok = stage_array(out.bundle_res, in->bundle_res, out.bundle_ptr[N]);
    }
    if (!ok) return fail(nullptr, SPFOM_EINVAL, "instance: on_device arrays are not readable device memory");
    auto P = [](auto &v, auto *orig) { return orig ? v.data() : nullptr; };
    out.in.seg_ptr = P(out.seg_ptr, in->seg_ptr);
    out.in.prod_idx = P(out.prod_idx, in->prod_idx);
    out.in.attract = P(out.attract, in->attract);
    out.in.shadow = P(out.shadow, in->shadow);
    out.in.no_purchase = P(out.no_purchase, in->no_purchase);
    out.in.arrival = P(out.arrival, in->arrival);
    out.in.price = P(out.price, in->price);
    out.in.capacity = P(out.capacity, in->capacity);
    out.in.bundle_ptr = P(out.bundle_ptr, in->bundle_ptr);
    out.in.bundle_res = P(out.bundle_res, in->bundle_res);
    out.in.resource_capacity = P(out.resource_capacity, in->resource_capacity);
    return SPFOM_OK;
}
}  // namespace

// ------------------------------------------------------------------ API
// Layout helper: position of each entry of a row in ascending order of the
// (distinct, by validation) relabelled product ids.  Short rows: rank by
// counting (rank_q = #{x : key_x < key_q}; branch-free, vectorised -- an
// O(k^2) count beats a comparison sort's mispredicted branches up to ~128
// entries: huge's layout 2.5x faster on the host); longer rows: sort.
template <bool WIDE>
static void row_ranks_impl(const uint32_t *key, int64_t len, int32_t *rank, std::vector<uint64_t> &tmp) {
    if (len <= 128) {
        for (int64_t q = 0; q < len; ++q) {
            const uint32_t kq = key[q];
            int32_t r = 0;
            for (int64_t x = 0; x < len; ++x) r += key[x] < kq ? 1 : 0;
            rank[q] = r;
        }
        return;
    }
    tmp.resize(len);
    for (int64_t q = 0; q < len; ++q) tmp[q] = ((uint64_t)key[q] << 32) | (uint64_t)q;
    std::sort(tmp.begin(), tmp.end());
    for (int64_t r = 0; r < len; ++r) rank[(uint32_t)tmp[r]] = (int32_t)r;
}
__attribute__((target("avx2"))) static void row_ranks_avx2(const uint32_t *key, int64_t len, int32_t *rank,
                                                           std::vector<uint64_t> &tmp) {
    row_ranks_impl<true>(key, len, rank, tmp);
}
static void row_ranks_base(const uint32_t *key, int64_t len, int32_t *rank, std::vector<uint64_t> &tmp) {
    row_ranks_impl<false>(key, len, rank, tmp);
}
static void row_ranks(const uint32_t *key, int64_t len, int32_t *rank, std::vector<uint64_t> &tmp) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2) row_ranks_avx2(key, len, rank, tmp);
    else row_ranks_base(key, len, rank, tmp);
}

extern "C" {

void spfom_abi_sizes(size_t *out) {
    out[0] = sizeof(spfom_instance);
    out[1] = sizeof(spfom_params);
    out[2] = sizeof(spfom_info_t);
    out[3] = sizeof(spfom_residuals_t);
    out[4] = sizeof(spfom_dist);
}

const char *spfom_build_info(void) {
    return "spfom-b200 0.1 (sm_100a, fp64)";
}

spfom_status spfom_partition(const int64_t *seg_ptr, int64_t m, int32_t world, int64_t *bounds) {
    if (!seg_ptr || !bounds || world < 1 || m < 0) return SPFOM_EINVAL;
    const int64_t nnz = seg_ptr[m];
    bounds[0] = 0;
    for (int r = 1; r < world; ++r) {
        // first segment boundary at or after the ideal nnz split
        const int64_t target = (nnz * r + world - 1) / world;
        const int64_t *p = std::lower_bound(seg_ptr, seg_ptr + m + 1, target);
        int64_t b = (int64_t)(p - seg_ptr);
        // choose the closer of b-1 and b
        if (b > 0 && b <= m && (target - seg_ptr[b - 1]) < (seg_ptr[b] - target)) b -= 1;
        b = std::max(b, bounds[r - 1]);
        bounds[r] = std::min<int64_t>(b, m);
    }
    bounds[world] = m;
    return SPFOM_OK;
}

spfom_status spfom_nccl_unique_id(void *out128) {
    if (!out128) return SPFOM_EINVAL;
    if (!nccl().ok) { g_create_error = "libnccl.so.2 not found"; return SPFOM_ENCCL; }
    nccl_uid id;
    if (nccl().GetUniqueId(&id) != 0) { g_create_error = "ncclGetUniqueId failed"; return SPFOM_ENCCL; }
    memcpy(out128, &id, 128);
    return SPFOM_OK;
}

spfom_status spfom_workspace_bytes(const spfom_instance *inst, const spfom_params *params, size_t *bytes) {
    if (!inst || !bytes || !inst->seg_ptr || inst->num_segments < 0 || inst->num_products < 1)
        return fail(nullptr, SPFOM_EINVAL, "spfom_workspace_bytes: bad arguments");
    StagedInstance staged;
    if (inst->on_device) {
        spfom_status st = stage_instance(inst, staged);
        if (st != SPFOM_OK) return st;
        inst = &staged.in;
    }
    Plan pl;
    make_plan(inst, params, pl);
    *bytes = pl.total;
    return SPFOM_OK;
}

static spfom_status validate(const spfom_instance *in, const spfom_params *p) {
    char buf[256];
    const int64_t m = in->num_segments, N = in->num_products;
    if (m < 0 || N < 1 || in->nnz < 0 || !in->seg_ptr || (in->nnz > 0 && (!in->prod_idx || !in->attract)) ||
        (m > 0 && (!in->no_purchase || !in->arrival)) || !in->price || (in->num_resources <= 0 && !in->capacity))
        return fail(nullptr, SPFOM_EINVAL, "instance: missing array or bad size");
    if (in->seg_ptr[0] != 0 || in->seg_ptr[m] != in->nnz)
        return fail(nullptr, SPFOM_EDATA, "instance: seg_ptr[0] must be 0 and seg_ptr[m] == nnz");
    if (in->num_periods < 0) return fail(nullptr, SPFOM_EINVAL, "instance: num_periods must be >= 0");
    const int64_t T = std::max<int64_t>(1, in->num_periods);
    if (T > 1 && p && p->blocks) return fail(nullptr, SPFOM_EINVAL, "sampled blocks are not supported with num_periods > 1");
    if (N >= INT32_MAX) return fail(nullptr, SPFOM_EDATA, "instance: num_products too large");
    if (in->nnz + 3 * m >= INT32_MAX)   // padded entries index int32 device offsets
        return fail(nullptr, SPFOM_EDATA, "instance: too many entries for one GPU (shard it over more ranks)");
    // per-segment rules: a parallel scan finds the first offending segment, the
    // serial loop below (from there) reports it
    int64_t first_bad = m;
#pragma omp parallel for schedule(static, 4096) reduction(min : first_bad)
    for (int64_t i = 0; i < m; ++i) {
        const int64_t a = in->seg_ptr[i], b = in->seg_ptr[i + 1];
        bool ok = b >= a && !(T > 1 && (b - a + 3) / 4 > 128) && (b - a + 3) / 4 <= kMaxQuads &&
                  in->no_purchase[i] > 0.0 && std::isfinite(in->no_purchase[i]);
        for (int64_t t = 0; t < T && ok; ++t) ok = in->arrival[t * m + i] > 0.0 && std::isfinite(in->arrival[t * m + i]);
        for (int64_t e = a; e < b && ok; ++e) {
            const int32_t j = in->prod_idx[e];
            const double v = in->attract[e], w = in->shadow ? in->shadow[e] : 0.0;
            ok = j >= 0 && j < N && !(e > a && j <= in->prod_idx[e - 1]) && v > 0.0 && std::isfinite(v) && w >= 0.0 && w < v;
        }
        if (!ok && i < first_bad) first_bad = i;
    }
    for (int64_t i = first_bad; i < m; ++i) {
        const int64_t a = in->seg_ptr[i], b = in->seg_ptr[i + 1];
        if (b < a) { snprintf(buf, sizeof buf, "seg_ptr not monotone at segment %lld", (long long)i); return fail(nullptr, SPFOM_EDATA, buf); }
        if (T > 1 && (b - a + 3) / 4 > 128) {
            snprintf(buf, sizeof buf, "segment %lld: multi-period rows longer than 512 entries unsupported", (long long)i);
            return fail(nullptr, SPFOM_EDATA, buf);
        }
        if ((b - a + 3) / 4 > kMaxQuads) {
            snprintf(buf, sizeof buf, "segment %lld: consideration set of %lld > 1024 products unsupported", (long long)i, (long long)(b - a));
            return fail(nullptr, SPFOM_EDATA, buf);
        }
        if (!(in->no_purchase[i] > 0.0) || !std::isfinite(in->no_purchase[i])) { snprintf(buf, sizeof buf, "no_purchase[%lld] must be > 0", (long long)i); return fail(nullptr, SPFOM_EDATA, buf); }
        for (int64_t t = 0; t < T; ++t)
            if (!(in->arrival[t * m + i] > 0.0) || !std::isfinite(in->arrival[t * m + i])) { snprintf(buf, sizeof buf, "arrival[%lld] must be > 0", (long long)(t * m + i)); return fail(nullptr, SPFOM_EDATA, buf); }
        for (int64_t e = a; e < b; ++e) {
            const int32_t j = in->prod_idx[e];
            if (j < 0 || j >= N || (e > a && j <= in->prod_idx[e - 1])) {
                snprintf(buf, sizeof buf, "prod_idx[%lld] out of range or not strictly increasing in segment %lld", (long long)e, (long long)i);
                return fail(nullptr, SPFOM_EDATA, buf);
            }
            const double v = in->attract[e], w = in->shadow ? in->shadow[e] : 0.0;
            if (!(v > 0.0) || !std::isfinite(v) || !(w >= 0.0) || !(w < v)) {
                snprintf(buf, sizeof buf, "entry %lld: need v > 0 and 0 <= w < v", (long long)e);
                return fail(nullptr, SPFOM_EDATA, buf);
            }
        }
    }
    const int64_t L = in->num_resources;
    if (L < 0) return fail(nullptr, SPFOM_EINVAL, "instance: num_resources must be >= 0");
    for (int64_t j = 0; j < N; ++j) {
        if (!(in->price[j] >= 0.0) || !std::isfinite(in->price[j])) { snprintf(buf, sizeof buf, "price[%lld] must be >= 0", (long long)j); return fail(nullptr, SPFOM_EDATA, buf); }
        if (L == 0 && (!(in->capacity[j] >= 0.0) || !std::isfinite(in->capacity[j]))) { snprintf(buf, sizeof buf, "capacity[%lld] must be >= 0", (long long)j); return fail(nullptr, SPFOM_EDATA, buf); }
    }
    if (L > 0) {
        if (!in->bundle_ptr || !in->bundle_res || !in->resource_capacity)
            return fail(nullptr, SPFOM_EINVAL, "instance: bundles need bundle_ptr, bundle_res, resource_capacity");
        if (in->bundle_ptr[0] != 0) return fail(nullptr, SPFOM_EDATA, "bundle_ptr[0] must be 0");
        if (L >= INT32_MAX) return fail(nullptr, SPFOM_EDATA, "num_resources too large");
        for (int64_t j = 0; j < N; ++j) {
            const int64_t a = in->bundle_ptr[j], b = in->bundle_ptr[j + 1];
            if (b <= a) { snprintf(buf, sizeof buf, "bundle %lld consumes no resource", (long long)j); return fail(nullptr, SPFOM_EDATA, buf); }
            for (int64_t e = a; e < b; ++e)
                if (in->bundle_res[e] < 0 || in->bundle_res[e] >= L || (e > a && in->bundle_res[e] <= in->bundle_res[e - 1])) {
                    snprintf(buf, sizeof buf, "bundle_res of bundle %lld out of range or not strictly increasing", (long long)j);
                    return fail(nullptr, SPFOM_EDATA, buf);
                }
        }
        for (int64_t l = 0; l < L; ++l)
            if (!(in->resource_capacity[l] >= 0.0) || !std::isfinite(in->resource_capacity[l])) { snprintf(buf, sizeof buf, "resource_capacity[%lld] must be >= 0", (long long)l); return fail(nullptr, SPFOM_EDATA, buf); }
    }
    if (!p) return fail(nullptr, SPFOM_EINVAL, "params: NULL");
    if (!(p->theta > 0.0)) return fail(nullptr, SPFOM_EINVAL, "params: theta must be > 0 (INFINITY = exact argmax)");
    if (!(p->tau > 0.0) || !std::isfinite(p->tau)) return fail(nullptr, SPFOM_EINVAL, "params: tau must be > 0");
    if (!(p->mu >= 0.0) || !std::isfinite(p->mu)) return fail(nullptr, SPFOM_EINVAL, "params: mu must be >= 0");
    if (p->tau_mode == 0 && p->tau * p->mu > 1.0) return fail(nullptr, SPFOM_EINVAL, "params: tau * mu must be <= 1 (S:L296)");
    if (!(p->extrapolation >= 0.0 && p->extrapolation <= 1.0)) return fail(nullptr, SPFOM_EINVAL, "params: extrapolation in [0, 1]");
    if (p->tau_mode != 0 && p->tau_mode != 1) return fail(nullptr, SPFOM_EINVAL, "params: tau_mode must be 0 or 1");
    if (p->blocks) {
        if (p->block_size < 1 || p->block_iters < 1) return fail(nullptr, SPFOM_EINVAL, "params: block_size and block_iters must be >= 1");
        const int64_t M = in->num_segments_global > 0 ? in->num_segments_global : m;
        for (int64_t t = 0; t < p->block_iters; ++t) {
            const int32_t *row = p->blocks + t * p->block_size;
            for (int64_t b = 0; b < p->block_size; ++b)
                if (row[b] < 0 || row[b] >= M || (b > 0 && row[b] <= row[b - 1]))
                    return fail(nullptr, SPFOM_EINVAL, "params: block rows must hold strictly increasing global ids < m");
        }
    }
    return SPFOM_OK;
}

// SPFOM_TRACE_CREATE=1: host-side phase times of spfom_create on stderr
struct PhaseTimer {
    bool on = getenv("SPFOM_TRACE_CREATE") != nullptr;
    double t0 = now();
    static double now() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec + 1e-9 * ts.tv_nsec;
    }
    void mark(const char *what) {
        if (!on) return;
        const double t = now();
        fprintf(stderr, "[spfom_create] %-28s %8.1f ms\n", what, (t - t0) * 1e3);
        t0 = t;
    }
};

spfom_status spfom_create(const spfom_instance *in, const spfom_params *p, const spfom_dist *dist,
                          void *cuda_stream, void *workspace, size_t ws_bytes, spfom_handle **out) {
    if (!in || !out) return fail(nullptr, SPFOM_EINVAL, "spfom_create: NULL argument");
    *out = nullptr;
    PhaseTimer ptimer;
    StagedInstance staged;
    if (in->on_device) {
        spfom_status sst = stage_instance(in, staged);
        if (sst != SPFOM_OK) return sst;
        in = &staged.in;
        ptimer.mark("stage device instance");
    }
    spfom_status st = validate(in, p);
    ptimer.mark("validate");
    if (st != SPFOM_OK) return st;
    Plan pl;
    make_plan(in, p, pl);
    if (!workspace || ws_bytes < pl.total) return fail(nullptr, SPFOM_ENOMEM, "workspace smaller than spfom_workspace_bytes()");
    if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0) return fail(nullptr, SPFOM_EINVAL, "workspace must be 256-byte aligned");

    auto *h = new spfom_handle();
    h->pl = pl;
    h->params = *p;
    if (h->params.max_newton <= 0) h->params.max_newton = 200;
    h->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    if (h->stream == nullptr || h->stream == cudaStreamLegacy) {
        // the legacy default stream cannot be captured into a CUDA graph: use a private one
        if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
            g_create_error = "cudaStreamCreate failed";
            delete h;
            return SPFOM_ECUDA;
        }
        h->own_stream = true;
    }
    h->ws = reinterpret_cast<char *>(workspace);
    h->m = in->num_segments;
    h->N = in->num_products;
    h->nnz = in->nnz;
    h->nq = pl.nq;
    h->T = pl.T;
    int dev = 0;
    cudaGetDevice(&dev);
    h->device = dev;
    cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, dev);
    auto bail = [&](spfom_status s) {
        g_create_error = h->err;
        for (int b = 0; b < kNumBins; ++b) {
            if (h->side[b]) cudaStreamDestroy(h->side[b]);
            if (h->ev_join[b]) cudaEventDestroy(h->ev_join[b]);
        }
        if (h->ev_fork) cudaEventDestroy(h->ev_fork);
        for (cudaGraphExec_t g : {h->graph, h->graph_u, h->graph_refresh, h->graph_primal, h->graph_rest,
                                  h->graph_rest_refresh})
            if (g) cudaGraphExecDestroy(g);
        destroy_timed(h);
        for (int c = 0; c < 2; ++c) {
            if (h->pin_ev[c]) cudaEventSynchronize(h->pin_ev[c]);
            pin_give(h->pin[c]);
            if (h->pin_ev[c]) cudaEventDestroy(h->pin_ev[c]);
        }
        if (h->own_stream) cudaStreamDestroy(h->stream);
        delete h;
        return s;
    };

    // distributed mode: world > 1, or world == 1 with an NCCL id (the multi-rank
    // code path -- NCCL allreduce, k_fold -- on one GPU; tests use it)
    if (dist && (dist->world > 1 || dist->nccl_id)) {
        if (!nccl().ok) { h->err = "distributed mode but libnccl.so.2 not loadable"; return bail(SPFOM_ENCCL); }
        if (!dist->nccl_id || dist->rank < 0 || dist->rank >= dist->world) { h->err = "bad spfom_dist"; return bail(SPFOM_EINVAL); }
        h->rank = dist->rank;
        h->world = dist->world;
        nccl_uid id;
        memcpy(&id, dist->nccl_id, 128);
        if (nccl().CommInitRank(&h->comm, h->world, id, h->rank) != 0) { h->err = "ncclCommInitRank failed"; return bail(SPFOM_ENCCL); }
    }
    const int64_t m = h->m, N = h->N;

    ptimer.mark("plan+handle+streams");
    // ---- global column counts n_j
    std::vector<int64_t> counts(N + 1, 0);
#pragma omp parallel
    {
        std::vector<int64_t> loc(N + 1, 0);                    // per-thread histogram, merged below
#pragma omp for schedule(static) nowait
        for (int64_t e = 0; e < in->nnz; ++e) loc[in->prod_idx[e]] += h->T;   // stacked segments (T per base row)
#pragma omp critical
        for (int64_t j = 0; j <= N; ++j) counts[j] += loc[j];
    }
    if (h->comm) {
        int64_t *dcounts = slot_ptr<int64_t>(h, O_COUNTS);
        if (cudaMemcpyAsync(dcounts, counts.data(), N * 8, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) { h->err = "H2D counts"; return bail(SPFOM_ECUDA); }
        if (allreduce(h, dcounts, dcounts, N, kNcclInt64, kNcclSum) != SPFOM_OK) return bail(SPFOM_ENCCL);
        if (cudaMemcpyAsync(counts.data(), dcounts, N * 8, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
            cudaStreamSynchronize(h->stream) != cudaSuccess) { h->err = "D2H counts"; return bail(SPFOM_ECUDA); }
    }
    ptimer.mark("column counts");
    // ---- popularity relabelling: new id = rank by (-n_j, j)
    h->new2old.resize(N);
    std::iota(h->new2old.begin(), h->new2old.end(), 0);
    std::stable_sort(h->new2old.begin(), h->new2old.end(), [&](int32_t a, int32_t b) { return counts[a] > counts[b]; });
    h->old2new.resize(N);
    for (int64_t j = 0; j < N; ++j) h->old2new[h->new2old[j]] = (int32_t)j;
    h->n_present = 0;
    for (int64_t j = 0; j < N; ++j) h->n_present += counts[j] > 0;

    ptimer.mark("relabelling");
    // ---- per-product arrays (relabelled), slot N = dummy
    const int64_t L = in->num_resources;
    h->L = L;
    const int64_t D1 = std::max<int64_t>(N + 1, L + 1);
    std::vector<double> r(N + 1, 0.0), c(D1, 0.0), tau(D1, 0.0);
    for (int64_t jn = 0; jn < N; ++jn) {
        const int32_t jo = h->new2old[jn];
        r[jn] = in->price[jo];
        if (L > 0) continue;
        c[jn] = in->capacity[jo];
        tau[jn] = (p->tau_mode == 1 && counts[jo] > 0) ? p->tau / (double)counts[jo] : p->tau;
        if (p->tau_mode == 1 && tau[jn] * p->mu > 1.0) { h->err = "params: tau_j * mu must be <= 1"; return bail(SPFOM_EINVAL); }
    }
    // bundles (NRM): relabelled CSR by bundle, CSC by resource (ascending original bundle id,
    // the oracle's summation order), per-resource tau_l = tau / n_l, n_l = sum_{j uses l} n_j
    std::vector<int32_t> bptr_d(N + 2, 0), bres_d, rptr_d(L + 2, 0), rbun_d;
    if (L > 0) {
        const int64_t nbz = in->bundle_ptr[N];
        bres_d.resize(std::max<int64_t>(nbz, 1));
        rbun_d.resize(std::max<int64_t>(nbz, 1));
        for (int64_t jn = 0; jn < N; ++jn) {
            const int32_t jo = h->new2old[jn];
            bptr_d[jn + 1] = bptr_d[jn] + (int32_t)(in->bundle_ptr[jo + 1] - in->bundle_ptr[jo]);
            for (int64_t e = in->bundle_ptr[jo]; e < in->bundle_ptr[jo + 1]; ++e)
                bres_d[bptr_d[jn] + (e - in->bundle_ptr[jo])] = in->bundle_res[e];
        }
        std::vector<int64_t> nl(L, 0);
        for (int64_t e = 0; e < nbz; ++e) rptr_d[in->bundle_res[e] + 1] += 1;
        for (int64_t l = 0; l < L; ++l) rptr_d[l + 1] += rptr_d[l];
        std::vector<int32_t> fill(rptr_d.begin(), rptr_d.end() - 1);
        for (int64_t jo = 0; jo < N; ++jo)                       // ascending original bundle id
            for (int64_t e = in->bundle_ptr[jo]; e < in->bundle_ptr[jo + 1]; ++e) {
                const int32_t l = in->bundle_res[e];
                rbun_d[fill[l]++] = h->old2new[jo];
                nl[l] += counts[jo];
            }
        for (int64_t l = 0; l < L; ++l) {
            c[l] = in->resource_capacity[l];
            tau[l] = (p->tau_mode == 1 && nl[l] > 0) ? p->tau / (double)nl[l] : p->tau;
            if (p->tau_mode == 1 && tau[l] * p->mu > 1.0) { h->err = "params: tau_l * mu must be <= 1"; return bail(SPFOM_EINVAL); }
        }
    }

    ptimer.mark("product arrays + bundles");
    // ---- length bins; device segment order = (bin, local id), so that every
    // bin is one contiguous range
    std::vector<int> segbin(std::max<int64_t>(m, 1));
    std::vector<int32_t> snew(std::max<int64_t>(m, 1));       // local id -> device slot
    h->bin_first.assign(kNumBins + 1, 0);
    {
        std::vector<int64_t> cnt(kNumBins, 0);
        for (int64_t i = 0; i < m; ++i) {
            segbin[i] = bin_of((in->seg_ptr[i + 1] - in->seg_ptr[i] + 3) / 4);
            cnt[segbin[i]]++;
        }
        for (int b = 0; b < kNumBins; ++b) h->bin_first[b + 1] = (int32_t)(h->bin_first[b] + cnt[b]);
        std::vector<int64_t> fill(h->bin_first.begin(), h->bin_first.end() - 1);
        h->sorder.assign(std::max<int64_t>(m, 1), 0);
        for (int64_t i = 0; i < m; ++i) {
            const int64_t k = fill[segbin[i]]++;
            h->sorder[k] = (int32_t)i;
            snew[i] = (int32_t)k;
        }
    }

    ptimer.mark("bins + device order");
    // ---- padded quad CSR in device order
    std::vector<int32_t> qoff(m + 1, 0);
    for (int64_t k = 0; k < m; ++k) {
        const int64_t i = h->sorder[k];
        qoff[k + 1] = qoff[k] + (int32_t)((in->seg_ptr[i + 1] - in->seg_ptr[i] + 3) / 4);
    }
    const int64_t nq = qoff[m];
    const int64_t T = h->T;
    auto segc = host_array<double2>(T * m);   // every slot written below
    auto segv = host_array<double4>(T * m);
    h->pos_map = host_array<int32_t>(in->nnz);
    if (!segc || !segv || !h->pos_map) { h->err = "host allocation"; return bail(SPFOM_ENOMEM); }
    ptimer.mark("qoff + host arrays");
    double t_wait = 0.0, t_build = 0.0;
    h->seg_off.assign(in->seg_ptr, in->seg_ptr + m + 1);
    bool bad_numeric = false;
    // The padded arrays (ids, v, omega) are built chunk by chunk of device
    // slots straight into a pinned double buffer and copied to the workspace
    // asynchronously, so chunk c + 1 is built while chunk c is in flight (no
    // pageable staging of the whole instance, no serial H2D afterwards).  The
    // same pinned ring later stages the getters' D2H copies.
    for (int c = 0; c < 2; ++c) {
        if (pin_take(&h->pin[c], kPinQuads * 80) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->pin_ev[c], cudaEventDisableTiming) != cudaSuccess) {
            h->err = "pinned staging";
            return bail(SPFOM_ENOMEM);
        }
    }
    ptimer.mark("pinned staging ring");
    char *d_pidx = h->ws + h->pl.off[O_PIDX], *d_v = h->ws + h->pl.off[O_V], *d_om = h->ws + h->pl.off[O_OM];
    bool copy_ok = true;
    int64_t chunk_no = 0;
    for (int64_t k0 = 0; k0 < m;) {
        int64_t k1 = k0 + 1;
        while (k1 < m && (int64_t)qoff[k1 + 1] - qoff[k0] <= kPinQuads) ++k1;
        const int64_t q0 = qoff[k0], nqc = (int64_t)qoff[k1] - q0;   // <= kPinQuads (rows <= kMaxQuads)
        const int c = (int)(chunk_no & 1);
        const double tw0 = PhaseTimer::now();
        if (chunk_no >= 2 && cudaEventSynchronize(h->pin_ev[c]) != cudaSuccess) copy_ok = false;   // buffer free again
        const double tw1 = PhaseTimer::now();
        t_wait += tw1 - tw0;
        char *buf = reinterpret_cast<char *>(h->pin[c]);
        int32_t *pidx = reinterpret_cast<int32_t *>(buf);                 // [4 nqc]
        double *vv = reinterpret_cast<double *>(buf + 16 * nqc);           // [4 nqc]
        double *om = reinterpret_cast<double *>(buf + 48 * nqc);           // [4 nqc]
        const int64_t pbase = 4 * q0;
#pragma omp parallel
        {
        std::vector<uint32_t> key;                                       // per-thread row buffers
        std::vector<int32_t> rank;
        std::vector<double> wr;
        std::vector<uint64_t> tmp;
#pragma omp for schedule(dynamic, 1024)
        for (int64_t k = k0; k < k1; ++k) {
            const int64_t i = h->sorder[k];
            const int64_t a = in->seg_ptr[i], len = in->seg_ptr[i + 1] - a;
            key.resize(len);
            rank.resize(len);
            wr.resize(len);
            for (int64_t q = 0; q < len; ++q) key[q] = (uint32_t)h->old2new[in->prod_idx[a + q]];
            row_ranks(key.data(), len, rank.data(), tmp);
            const int64_t pend = 4 * (int64_t)qoff[k + 1] - pbase;
            for (int64_t p = 4 * (int64_t)qoff[k] - pbase + len; p < pend; ++p) {   // inert pads
                pidx[p] = (int32_t)N;
                vv[p] = 0.0;
                om[p] = 0.0;
            }
            const int64_t base = 4 * (int64_t)qoff[k];
            for (int64_t q = 0; q < len; ++q) {
                const int64_t e = a + q, o = base - pbase + rank[q];
                const double v = in->attract[e], w = in->shadow ? in->shadow[e] : 0.0;
                pidx[o] = (int32_t)key[q];
                vv[o] = v;
                om[o] = w / v;
                wr[rank[q]] = w;
                h->pos_map[e] = (int32_t)(base + rank[q]);
            }
            // vt0 and sum (v - w) in ascending new-id order (the summation order of the layout)
            double vt0 = in->no_purchase[i], svt = 0.0;
            for (int64_t q = 0; q < len; ++q) {
                vt0 += wr[q];
                svt += vv[base - pbase + q] - wr[q];
            }
            for (int64_t t = 0; t < T; ++t) {
                const double lam = in->arrival[t * m + i];
                segc[t * m + k] = make_double2(lam, vt0);
                // y0 = lambda and the initial projection multipliers (nu, kappa, U)
                segv[t * m + k] = make_double4(lam, 0.0, 0.0, lam / (vt0 + svt));
            }
            if (!std::isfinite(vt0)) bad_numeric = true;
        }
        }
        t_build += PhaseTimer::now() - tw1;
        if (nqc > 0) {
            copy_ok = copy_ok && cudaMemcpyAsync(d_pidx + 16 * q0, pidx, nqc * 16, cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
                      cudaMemcpyAsync(d_v + 32 * q0, vv, nqc * 32, cudaMemcpyHostToDevice, h->stream) == cudaSuccess &&
                      cudaMemcpyAsync(d_om + 32 * q0, om, nqc * 32, cudaMemcpyHostToDevice, h->stream) == cudaSuccess;
        }
        if (cudaEventRecord(h->pin_ev[c], h->stream) != cudaSuccess) copy_ok = false;
        ++chunk_no;
        k0 = k1;
    }
    if (!copy_ok) { h->err = "H2D copy of the padded CSR failed"; return bail(SPFOM_ECUDA); }
    if (bad_numeric) { h->err = "non-finite vt0"; return bail(SPFOM_EDATA); }

    h->qoff_h = qoff;
    for (int b = 0; b < kNumBins; ++b) {
        const int64_t k0 = h->bin_first[b], k1 = h->bin_first[b + 1];
        h->bin_uniform[b] = kBins[b].E > 0 && kBins[b].G == 4 && k1 > k0 &&
                            (int64_t)qoff[k1] - qoff[k0] == (k1 - k0) * kBins[b].E;
    }
    if (ptimer.on) fprintf(stderr, "[spfom_create]   (chunk builds %.1f ms, waits for the H2D ring %.1f ms)\n", t_build * 1e3, t_wait * 1e3);
    ptimer.mark("padded CSR (omp)");
    // ---- sampled block tables: per (iteration, bin) lists of device slots
    if (pl.sampled) {
        std::vector<int32_t> rowoff, blkids;
        const int64_t off = in->segment_offset;
        rowoff.assign(p->block_iters * (kNumBins + 1), 0);
        std::vector<std::vector<int32_t>> per(kNumBins);
        for (int64_t t = 0; t < p->block_iters; ++t) {
            for (auto &v : per) v.clear();
            const int32_t *row = p->blocks + t * p->block_size;
            for (int64_t b = 0; b < p->block_size; ++b) {
                const int64_t li = (int64_t)row[b] - off;
                if (li >= 0 && li < m) {
                    per[segbin[li]].push_back(snew[li]);
                    h->pl.bin_work[segbin[li]] += (double)(qoff[snew[li] + 1] - qoff[snew[li]] + 1) / (double)p->block_iters;
                }
            }
            int32_t *ro = rowoff.data() + t * (kNumBins + 1);
            ro[0] = (int32_t)blkids.size();
            for (int b = 0; b < kNumBins; ++b) {
                blkids.insert(blkids.end(), per[b].begin(), per[b].end());
                ro[b + 1] = (int32_t)blkids.size();
            }
        }
        // per-bin max count per row, for static grid sizes
        for (int b = 0; b < kNumBins; ++b) {
            int64_t mx = 0;
            for (int64_t t = 0; t < p->block_iters; ++t) {
                const int32_t *ro = rowoff.data() + t * (kNumBins + 1);
                mx = std::max<int64_t>(mx, ro[b + 1] - ro[b]);
            }
            h->pl.bin_count[b] = mx;
        }
        if (!blkids.empty() && cudaMemcpyAsync(slot_ptr<int32_t>(h, O_BLKIDS), blkids.data(), blkids.size() * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) { h->err = "H2D blocks"; return bail(SPFOM_ECUDA); }
        if (cudaMemcpyAsync(slot_ptr<int32_t>(h, O_ROWOFF), rowoff.data(), rowoff.size() * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) { h->err = "H2D rowoff"; return bail(SPFOM_ECUDA); }
        if (cudaStreamSynchronize(h->stream) != cudaSuccess) { h->err = "sync"; return bail(SPFOM_ECUDA); }
    }

    ptimer.mark("block tables");
    // ---- copies into the workspace
    auto H2D = [&](int slot, const void *src, size_t bytes) {
        return bytes == 0 || cudaMemcpyAsync(h->ws + h->pl.off[slot], src, bytes, cudaMemcpyHostToDevice, h->stream) == cudaSuccess;
    };
    std::vector<double> y0(std::max<int64_t>(T * m, 1));
    for (int64_t k = 0; k < T * m; ++k) y0[k] = segv[k].x;
    bool ok = H2D(O_QOFF, qoff.data(), (m + 1) * 4) && H2D(O_SEGC, segc.get(), T * m * 16) &&
              H2D(O_SEGV, segv.get(), T * m * 32) && H2D(O_R, r.data(), (N + 1) * 8) && H2D(O_C, c.data(), D1 * 8) &&
              H2D(O_TAU, tau.data(), D1 * 8) && H2D(O_G, r.data(), (N + 1) * 8) &&
              H2D(O_ORIG, h->new2old.data(), N * 4);
    h->bptr_h = bptr_d;
    h->bres_h = bres_d;
    if (L > 0)
        ok = ok && H2D(O_BPTR, bptr_d.data(), (N + 1) * 4) && H2D(O_BRES, bres_d.data(), bres_d.size() * 4) &&
             H2D(O_RPTR, rptr_d.data(), (L + 1) * 4) && H2D(O_RBUN, rbun_d.data(), rbun_d.size() * 4);
    if (pl.averaging) ok = ok && H2D(O_Y0BAR, y0.data(), T * m * 8);
    auto Z = [&](int slot, size_t bytes) { return bytes == 0 || cudaMemsetAsync(h->ws + h->pl.off[slot], 0, bytes, h->stream) == cudaSuccess; };
    ok = ok && Z(O_Y, T * nq * 32) && Z(O_ETA, std::max<int64_t>(D1, prod_slots(N)) * 8) && Z(O_ACC, (spread_off(N) + (size_t)kSpreadCopies * spread_range(N)) * 8) && Z(O_SCUR, prod_slots(N) * 8) &&
         Z(O_COUNTERS, 64) && Z(O_T, 8) && Z(O_WORK, 16 * kNumBins) && Z(O_SEGD, T * m * 16);
    if (pl.averaging) ok = ok && Z(O_YBAR, T * nq * 32) && Z(O_ETABAR, D1 * 8);
    if (!ok) { h->err = "H2D copy into workspace failed"; return bail(SPFOM_ECUDA); }
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) { h->err = "stream sync after create"; return bail(SPFOM_ECUDA); }

    DevState &S = h->S;
    S.pidx = slot_ptr<int4>(h, O_PIDX);
    S.v = slot_ptr<double>(h, O_V);
    S.om = slot_ptr<double>(h, O_OM);
    S.y = slot_ptr<double>(h, O_Y);
    S.ybar = pl.averaging ? slot_ptr<double>(h, O_YBAR) : nullptr;
    S.qoff = slot_ptr<int32_t>(h, O_QOFF);
    S.segc = slot_ptr<double2>(h, O_SEGC);
    S.segv = slot_ptr<double4>(h, O_SEGV);
    S.segd = slot_ptr<float4>(h, O_SEGD);
    S.y0bar = pl.averaging ? slot_ptr<double>(h, O_Y0BAR) : nullptr;
    S.r = slot_ptr<double>(h, O_R);
    S.c = slot_ptr<double>(h, O_C);
    S.tau = slot_ptr<double>(h, O_TAU);
    S.eta = slot_ptr<double>(h, O_ETA);
    S.g = slot_ptr<double>(h, O_G);
    S.s = slot_ptr<double>(h, O_ACC);
    S.L = (int32_t)L;
    S.bptr = slot_ptr<int32_t>(h, O_BPTR);
    S.bres = slot_ptr<int32_t>(h, O_BRES);
    S.rptr = slot_ptr<int32_t>(h, O_RPTR);
    S.rbun = slot_ptr<int32_t>(h, O_RBUN);
    S.stilde = slot_ptr<double>(h, O_STILDE);
    S.spread_off = (int32_t)spread_off(N);
    S.spread = S.s + S.spread_off;
    S.spread_n = (int32_t)spread_range(N);
    S.spread_c = kSpreadCopies;
    S.fold_in_dual = h->comm ? 0 : 1;
    // world > 1 with plain products: ReduceScatter -> K3 on the slice ->
    // AllGather (SPFOM_COLLECTIVE=allreduce keeps the allreduce + replicated K3)
    {
        const char *coll = getenv("SPFOM_COLLECTIVE");
        h->rs = h->comm && L == 0 && h->world <= kRankPad && !(coll && strcmp(coll, "allreduce") == 0);
        if (h->rs) {
            h->chunk = (N + 1 + h->world - 1) / h->world;
            h->np = h->chunk * h->world;
        }
    }
    S.s_prev = slot_ptr<double>(h, O_SCUR);
    S.etabar = pl.averaging ? slot_ptr<double>(h, O_ETABAR) : nullptr;
    S.counters = slot_ptr<unsigned long long>(h, O_COUNTERS);
    S.t = slot_ptr<int64_t>(h, O_T);
    S.m = m;
    S.N = N;
    S.nq = nq;
    S.T = (int32_t)T;
    S.theta = p->theta;
    S.mu = p->mu;
    S.omega_x = p->extrapolation;
    S.max_newton = h->params.max_newton;
    S.sampled = pl.sampled ? 1 : 0;

    // sampled uniform bins: TMA tensor maps for tile::gather4 of whole rows
    if (pl.sampled && T == 1 && SPFOM_SAMP_G4) {
        st = encode_gather_maps(h);
        if (st != SPFOM_OK) return bail(st);
    }
    // small regime (exec_mode 0 auto / 2 forced): whole iterations per cooperative launch
    {
        int64_t max_rq = 0;
        for (int64_t k = 0; k < m; ++k) max_rq = std::max<int64_t>(max_rq, qoff[k + 1] - qoff[k]);
        const int64_t per_iter = pl.sampled ? p->block_size : m;
        const bool eligible = !h->comm && T == 1 && h->L == 0 && !pl.averaging && !(pl.sampled && p->refresh_every > 0) &&
                              max_rq <= 256 && per_iter <= 4096;
        if (p->exec_mode == 2 && !eligible) {
            h->err = "exec_mode 2 needs world == 1, T == 1, no averaging/refresh, rows <= 1024 entries, <= 4096 segments per iteration";
            return bail(SPFOM_EINVAL);
        }
        if (eligible && p->exec_mode != 1) {
            h->small_q = max_rq <= 32 ? 1 : max_rq <= 64 ? 2 : max_rq <= 128 ? 4 : 8;
            int per_sm = 0;
            cudaError_t e = cudaSuccess;
            switch (h->small_q) {
#define OCC(Q) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small<Q, false, false>, kSmallThreads, 0); break;
                case 1: OCC(1)
                case 2: OCC(2)
                case 4: OCC(4)
                default: OCC(8)
#undef OCC
            }
            int coop = 0;
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
            if (e == cudaSuccess && per_sm >= 1 && coop) {
                h->small = true;
                h->small_blocks = h->sm_count;
            } else if (p->exec_mode == 2) {
                h->err = "exec_mode 2: cooperative launch unavailable";
                return bail(SPFOM_EINVAL);
            }
        }
    }
    // several active bins: concurrent launches on SM shares proportional to each bin's work
    // (padded entries x the bin's measured cost per entry; sampled: the mean over the
    // block rows of the bin's padded entries)
    if (!h->small) {
        int64_t wtot = 0, w[kNumBins] = {0};
        for (int b = 0; b < kNumBins; ++b) {
            const int64_t cnt = pl.sampled ? h->pl.bin_count[b] : (h->bin_first[b + 1] - h->bin_first[b]);
            // B200, medium config: an SM streams ~20 KB/us of a 4-lane bin, 16.0 of a
            // 16-lane and 13.6 of a 32-lane one (wider groups: more butterfly steps and
            // fewer segments per warp round), so wide bins get proportionally more SMs
            // (entry-mapped bins: 13 entries per lane; wider groups pay deeper butterflies)
            const double cost = kBins[b].E > 0 ? (kBins[b].G >= 16 ? 1.12 : kBins[b].G >= 8 ? 1.05 : 1.0)
                                               : (kBins[b].G >= 32 ? 1.5 : (kBins[b].G >= 16 ? 1.28 : 1.0));
            w[b] = pl.sampled ? (int64_t)(cost * h->pl.bin_work[b])
                              : (int64_t)(cost * (double)((int64_t)qoff[h->bin_first[b + 1]] - (int64_t)qoff[h->bin_first[b]] + cnt));
            if (cnt > 0) h->nbins_active += 1;
            wtot += w[b];
        }
        if (h->nbins_active > 1) {
            bool okc = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) == cudaSuccess;
            for (int b = 0; b < kNumBins && okc; ++b) {
                if (w[b] == 0) continue;
                h->bin_sms[b] = (int)std::max<int64_t>(1, (int64_t)((double)h->sm_count * (double)w[b] / (double)std::max<int64_t>(wtot, 1) + 0.5));
                okc = cudaStreamCreateWithFlags(&h->side[b], cudaStreamNonBlocking) == cudaSuccess &&
                      cudaEventCreateWithFlags(&h->ev_join[b], cudaEventDisableTiming) == cudaSuccess;
            }
            if (!okc) { h->err = "side stream creation failed"; return bail(SPFOM_ECUDA); }
#ifdef SPFOM_DIAG_BIN_SMS
            // diagnostic (exp/run_shares.sh): SM shares of the active bins from the environment, "a,b,c,.."
            if (const char *ov = getenv("SPFOM_BIN_SMS")) {
                for (int b = 0; b < kNumBins; ++b) {
                    if (w[b] == 0) continue;
                    h->bin_sms[b] = std::max(1, atoi(ov));
                    const char *c = strchr(ov, ',');
                    if (!c) break;
                    ov = c + 1;
                }
            }
            for (int b = 0; b < kNumBins; ++b)
                if (w[b]) fprintf(stderr, "[spfom] bin %d: w %lld sms %d\n", b, (long long)w[b], h->bin_sms[b]);
#endif
        }
    }
    ptimer.mark("H2D + state + modes");
    st = build_graph(h, false, &h->graph);
    if (st == SPFOM_OK && !(pl.sampled && p->refresh_every > 0)) st = build_graph(h, false, &h->graph_u, 0, kGraphUnroll);

    if (st != SPFOM_OK) return bail(st);
    if (pl.sampled && p->refresh_every > 0) {
        st = build_graph(h, true, &h->graph_refresh);
        if (st == SPFOM_OK) st = build_graph(h, false, &h->graph_primal, 1);
        if (st == SPFOM_OK) st = build_graph(h, false, &h->graph_rest, 2);
        if (st == SPFOM_OK) st = build_graph(h, true, &h->graph_rest_refresh, 2);
        if (st != SPFOM_OK) return bail(st);
    }
    ptimer.mark("graphs");
    *out = h;
    return SPFOM_OK;
}

}  // extern "C"

template <int Q, bool ARGMAX, bool SAMPLED>
static cudaError_t launch_small(spfom_handle *h, SmallArgs A) {
    void *args[] = {(void *)&h->S, (void *)&A};
    return cudaLaunchCooperativeKernel((const void *)k_small<Q, ARGMAX, SAMPLED>, dim3(h->small_blocks),
                                       dim3(kSmallThreads), args, 0, h->stream);
}

template <int Q>
static cudaError_t small_dispatch_q(spfom_handle *h, const SmallArgs &A) {
    const bool argmax = std::isinf(h->params.theta);
    if (h->pl.sampled) return argmax ? launch_small<Q, true, true>(h, A) : launch_small<Q, false, true>(h, A);
    return argmax ? launch_small<Q, true, false>(h, A) : launch_small<Q, false, false>(h, A);
}

static spfom_status step_small(spfom_handle *h, int64_t k) {
    constexpr int64_t kChunk = 1024;                 // iterations per cooperative launch
    while (k > 0) {
        SmallArgs A{};
        if (h->pl.sampled) {
            A.ids = slot_ptr<int32_t>(h, O_BLKIDS);
            A.row_off = slot_ptr<int32_t>(h, O_ROWOFF);
            A.block_iters = h->params.block_iters;
        }
        A.nbins = kNumBins;
        A.full_mode = h->pl.sampled ? 0 : 1;
        A.t0 = h->iter;
        A.iters = std::min(k, kChunk);
        cudaError_t e = cudaSuccess;
        switch (h->small_q) {
            case 1: e = small_dispatch_q<1>(h, A); break;
            case 2: e = small_dispatch_q<2>(h, A); break;
            case 4: e = small_dispatch_q<4>(h, A); break;
            default: e = small_dispatch_q<8>(h, A); break;
        }
        if (e != cudaSuccess) return fail(h, SPFOM_ECUDA, std::string("k_small launch: ") + cudaGetErrorString(e));
        h->iter += A.iters;
        k -= A.iters;
    }
    return SPFOM_OK;
}

extern "C" {

spfom_status spfom_step(spfom_handle *h, int64_t k) {
    if (!h || k < 0) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    if (h->small) return step_small(h, k);
    for (int64_t it = 0; it < k;) {
        if (h->graph_u && k - it >= kGraphUnroll) {
            // kGraphUnroll iterations per launch: their kernels follow each other
            // inside one graph (no graph-to-graph gap)
            CUDA_TRY(h, cudaGraphLaunch(h->graph_u, h->stream));
            h->iter += kGraphUnroll;
            it += kGraphUnroll;
            continue;
        }
        const bool refresh = h->graph_refresh && ((h->iter + 1) % h->params.refresh_every == 0);
        CUDA_TRY(h, cudaGraphLaunch(refresh ? h->graph_refresh : h->graph, h->stream));
        h->iter += 1;
        ++it;
    }
    return SPFOM_OK;
}

static spfom_status check_counters(spfom_handle *h) {
    unsigned long long cnt[6];
    CUDA_TRY(h, cudaMemcpyAsync(cnt, h->S.counters, sizeof cnt, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if (cnt[5] != 0) {   // SPFOM_DEVICE_CHECKS builds only
        char buf[128];
        snprintf(buf, sizeof buf, "device index / size checks failed %llu times", cnt[5]);
        h->err = buf;
        return SPFOM_ENUMERIC;
    }
    if (cnt[0] != 0) {
        char buf[128];
        snprintf(buf, sizeof buf, "projection hit max_newton on %llu segment-iterations", cnt[0]);
        h->err = buf;
        return SPFOM_ENUMERIC;
    }
    return SPFOM_OK;
}

// duals in caller order: products (original ids) or, with bundles, resources (not relabelled)
static spfom_status fetch_duals(spfom_handle *h, const double *src, double *eta) {
    if (h->L > 0) {
        CUDA_TRY(h, cudaMemcpyAsync(eta, src, h->L * 8, cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
        return SPFOM_OK;
    }
    std::vector<double> tmp(h->N);
    CUDA_TRY(h, cudaMemcpyAsync(tmp.data(), src, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    for (int64_t jn = 0; jn < h->N; ++jn) eta[h->new2old[jn]] = tmp[jn];
    return SPFOM_OK;
}

spfom_status spfom_duals(spfom_handle *h, double *eta) {
    if (!h || !eta) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    if (spfom_status gs = gather_slices(h, h->S.eta); gs != SPFOM_OK) return gs;
    spfom_status st = fetch_duals(h, h->S.eta, eta);
    return st != SPFOM_OK ? st : check_counters(h);
}

spfom_status spfom_usage(spfom_handle *h, double *s) {
    if (!h || !s) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    if (spfom_status gs = gather_slices(h, h->S.s_prev); gs != SPFOM_OK) return gs;
    std::vector<double> tmp(h->N);
    CUDA_TRY(h, cudaMemcpyAsync(tmp.data(), h->S.s_prev, h->N * 8, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    for (int64_t jn = 0; jn < h->N; ++jn) s[h->new2old[jn]] = tmp[jn];
    return SPFOM_OK;
}

// y0 in device order is either a plain array (pitch 8) or the x field of segv (pitch 32)
// y: device [T][nq] quads -> [T][nnz] stacked entry order.  The quads come
// down in chunks of device slots through a pinned double buffer: chunk c + 1
// copies (full PCIe rate) while the host un-permutes chunk c into y (rows of
// the slots' original segments; pos_map gives each entry's padded position).
static spfom_status fetch_primal(spfom_handle *h, const double *dy, const double *dy0, size_t pitch0, double *y,
                                 double *y0) {
    const int64_t T = h->T, m = h->m;
    std::vector<double> t0(std::max<int64_t>(T * m, 1));
    if (y0 && m)
        CUDA_TRY(h, cudaMemcpy2DAsync(t0.data(), 8, dy0, pitch0, 8, T * m, cudaMemcpyDeviceToHost, h->stream));
    if (y && h->nq) {
        for (int c = 0; c < 2; ++c) {
            if (!h->pin[c]) CUDA_TRY(h, pin_take(&h->pin[c], kPinQuads * 80));
            if (!h->pin_ev[c]) CUDA_TRY(h, cudaEventCreateWithFlags(&h->pin_ev[c], cudaEventDisableTiming));
        }
        // chunks: (period t, device slots [k0, k1)) with at most kPinQuads quads
        struct Chunk { int64_t t, k0, k1; };
        std::vector<Chunk> chunks;
        const int32_t *qo = h->qoff_h.data();
        for (int64_t t = 0; t < T; ++t) {
            int64_t k0 = 0;
            while (k0 < m) {
                int64_t k1 = k0 + 1;
                while (k1 < m && (int64_t)qo[k1 + 1] - qo[k0] <= kPinQuads) ++k1;
                chunks.push_back({t, k0, k1});
                k0 = k1;
            }
        }
        const int32_t *pm = h->pos_map.get();
        const double *pin_of[2] = {h->pin[0], h->pin[1]};
        auto issue = [&](size_t c) -> spfom_status {
            const Chunk &ch = chunks[c];
            const int64_t q0 = qo[ch.k0], nqc = (int64_t)qo[ch.k1] - q0;   // <= kPinQuads
            CUDA_TRY(h, cudaMemcpyAsync(h->pin[c & 1], dy + 4 * (ch.t * h->nq + q0), nqc * 32, cudaMemcpyDeviceToHost,
                                        h->stream));
            CUDA_TRY(h, cudaEventRecord(h->pin_ev[c & 1], h->stream));
            return SPFOM_OK;
        };
        spfom_status st = chunks.empty() ? SPFOM_OK : issue(0);
        for (size_t c = 0; c < chunks.size() && st == SPFOM_OK; ++c) {
            const Chunk &ch = chunks[c];
            const int64_t q0 = qo[ch.k0];
            CUDA_TRY(h, cudaEventSynchronize(h->pin_ev[c & 1]));
            const double *src = pin_of[c & 1];
            if (c + 1 < chunks.size()) st = issue(c + 1);   // next chunk copies while this one is placed
            double *dst = y + ch.t * h->nnz;
            const int64_t base = 4 * q0;
#pragma omp parallel for schedule(dynamic, 1024)
            for (int64_t k = ch.k0; k < ch.k1; ++k) {
                const int64_t i = h->sorder[k];
                for (int64_t e = h->seg_off[i]; e < h->seg_off[i + 1]; ++e) dst[e] = src[pm[e] - base];
            }
        }
        if (st != SPFOM_OK) return st;
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if (y0)
        for (int64_t t = 0; t < T; ++t)
            for (int64_t k = 0; k < m; ++k) y0[t * m + h->sorder[k]] = t0[t * m + k];
    return SPFOM_OK;
}

spfom_status spfom_primal(spfom_handle *h, double *y, double *y0) {
    if (!h) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    spfom_status st = fetch_primal(h, h->S.y, reinterpret_cast<const double *>(h->S.segv), 32, y, y0);
    return st != SPFOM_OK ? st : check_counters(h);
}

spfom_status spfom_averages(spfom_handle *h, double *ybar, double *y0bar, double *etabar) {
    if (!h) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    if (!h->pl.averaging) return fail(h, SPFOM_EINVAL, "averaging is off");
    if (spfom_status gs = gather_slices(h, h->S.etabar); gs != SPFOM_OK) return gs;
    spfom_status st = fetch_primal(h, h->S.ybar, h->S.y0bar, 8, ybar, y0bar);
    if (st != SPFOM_OK) return st;
    if (etabar) return fetch_duals(h, h->S.etabar, etabar);
    return SPFOM_OK;
}

spfom_status spfom_residuals(spfom_handle *h, spfom_residuals_t *out) {
    if (!h || !out) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    if (spfom_status gs = gather_slices(h, h->S.eta); gs != SPFOM_OK) return gs;
    DevState S = h->S;
    double *sf = slot_ptr<double>(h, O_TMP);
    CUDA_TRY(h, cudaMemsetAsync(sf, 0, (h->N + 1) * 8, h->stream));
    k_usage<<<h->sm_count * 4, kThreads, 0, h->stream>>>(S, h->T * h->nq, sf, (int32_t)std::min<int64_t>(kHeadMax, h->N));
    spfom_status st = allreduce(h, sf, sf, (size_t)h->N, kNcclFloat64, kNcclSum);
    if (st != SPFOM_OK) return st;
    double *pseg = slot_ptr<double>(h, O_RESSEG);
    CUDA_TRY(h, cudaMemsetAsync(pseg, 0, (size_t)kNumBins * kResidBlocks * 4 * 8, h->stream));
    for (int b = 0; b < kNumBins; ++b) {
        const int64_t cnt = h->bin_first[b + 1] - h->bin_first[b];
        if (cnt == 0) continue;
        SegList L{};
        L.ids = nullptr;
        L.first = h->bin_first[b];
        L.count = cnt;
        for (int64_t t = 0; t < h->T; ++t)   // partials accumulate over periods (sum / max), see the kernel
            resid_dispatch(b, S, L, pseg + (size_t)b * kResidBlocks * 4, t * h->m, t * h->nq, h->stream);
    }
    double *pprod = slot_ptr<double>(h, O_RESPROD);
    k_resid_prod<<<kResidBlocks, kThreads, 0, h->stream>>>(S, sf, h->n_present, pprod);
    double *pres = slot_ptr<double>(h, O_RESRES);
    if (h->L > 0) k_resid_res<<<kResidBlocks, kThreads, 0, h->stream>>>(S, sf, pres);   // resource rows
    CUDA_TRY(h, cudaGetLastError());
    // cross-rank: sum of D_seg, max of the audits (local segment quantities)
    double *red = slot_ptr<double>(h, O_COUNTS);   // reuse the counts slot as scratch (>= 4 doubles)
    std::vector<double> hs((size_t)kNumBins * kResidBlocks * 4), hp((size_t)kResidBlocks * 8);
    CUDA_TRY(h, cudaMemcpyAsync(hs.data(), pseg, hs.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaMemcpyAsync(hp.data(), pprod, hp.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    std::vector<double> hr(h->L > 0 ? hp.size() : 0);
    if (h->L > 0) CUDA_TRY(h, cudaMemcpyAsync(hr.data(), pres, hr.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    unsigned long long cnt[3];
    CUDA_TRY(h, cudaMemcpyAsync(cnt, h->S.counters, sizeof cnt, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    double dseg = 0.0, agg[3] = {0, 0, 0};
    for (size_t bb = 0; bb < (size_t)kNumBins * kResidBlocks; ++bb) {
        dseg += hs[4 * bb];
        for (int k = 0; k < 3; ++k) agg[k] = std::max(agg[k], hs[4 * bb + 1 + k]);
    }
    double pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = 0; b < kResidBlocks; ++b)
        for (int k = 0; k < 8; ++k)
            pr[k] = (k == 2 || k == 3 || k == 7) ? std::max(pr[k], hp[8 * b + k]) : pr[k] + hp[8 * b + k];
    for (size_t b = 0; b < hr.size() / 8; ++b)      // bundles: the capacity rows are resources
        for (int k = 0; k < 8; ++k)
            pr[k] = (k == 2 || k == 3 || k == 7) ? std::max(pr[k], hr[8 * b + k]) : pr[k] + hr[8 * b + k];
    if (h->comm) {
        double buf[4] = {dseg, agg[0], agg[1], agg[2]};
        CUDA_TRY(h, cudaMemcpyAsync(red, buf, 32, cudaMemcpyHostToDevice, h->stream));
        if ((st = allreduce(h, red, red, 1, kNcclFloat64, kNcclSum)) != SPFOM_OK) return st;
        if ((st = allreduce(h, red + 1, red + 1, 3, kNcclFloat64, kNcclMax)) != SPFOM_OK) return st;
        CUDA_TRY(h, cudaMemcpyAsync(buf, red, 32, cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
        dseg = buf[0];
        agg[0] = buf[1]; agg[1] = buf[2]; agg[2] = buf[3];
    }
    const double P = pr[0], D = pr[1] + dseg;
    out->iteration = h->iter;
    out->primal_obj = P;
    out->dual_obj = D;
    out->rel_gap = (D - P) / (1.0 + std::fabs(P) + std::fabs(D));
    out->infeas_abs = pr[2];
    out->infeas_rel = pr[3];
    out->infeas_rel_l2 = std::sqrt(pr[4]) / (1.0 + std::sqrt(pr[5]));
    out->balance_rel_max = agg[0];
    out->scale_rel_max = agg[1];
    out->neg_max = agg[2];
    out->compl_slack = pr[6] / (1.0 + std::fabs(P));
    out->alpha = pr[7];
    out->cert_lower = (1.0 - pr[7]) * P;
    out->cert_upper = D;
    out->newton_failures = (int64_t)cnt[0];
    out->newton_passes = (int64_t)cnt[1];
    out->newton_restarts = (int64_t)cnt[2];
    return SPFOM_OK;
}

spfom_status spfom_objective(spfom_handle *h, double *obj) {
    if (!h || !obj) return SPFOM_EINVAL;
    spfom_residuals_t r;
    spfom_status st = spfom_residuals(h, &r);
    if (st == SPFOM_OK) *obj = r.primal_obj;
    return st;
}

spfom_status spfom_set_state(spfom_handle *h, const double *y, const double *y0, const double *eta, const double *s_prev) {
    if (!h) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    const int64_t T = h->T;
    if ((y || y0) && h->m)   // a new iterate: no history to extrapolate the warm starts along
        CUDA_TRY(h, cudaMemsetAsync(h->S.segd, 0, (size_t)T * h->m * 16, h->stream));
    if (y) {
        std::vector<double> tmp(4 * std::max<int64_t>(T * h->nq, 1), 0.0);
        for (int64_t t = 0; t < T; ++t)
            for (int64_t e = 0; e < h->nnz; ++e) tmp[4 * t * h->nq + h->pos_map[e]] = y[t * h->nnz + e];
        CUDA_TRY(h, cudaMemcpyAsync(h->S.y, tmp.data(), T * h->nq * 32, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    }
    if (y0 && h->m) {
        std::vector<double> t0(T * h->m);
        for (int64_t t = 0; t < T; ++t)
            for (int64_t k = 0; k < h->m; ++k) t0[t * h->m + k] = y0[t * h->m + h->sorder[k]];
        CUDA_TRY(h, cudaMemcpy2DAsync(reinterpret_cast<double *>(h->S.segv), 32, t0.data(), 8, 8, T * h->m,
                                      cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    }
    std::vector<double> t1(std::max<int64_t>(h->N, h->L) + 1, 0.0), t2(h->N + 1, 0.0);
    if (eta) {
        std::vector<double> r(h->N + 1, 0.0);
        CUDA_TRY(h, cudaMemcpyAsync(r.data(), h->S.r, (h->N + 1) * 8, cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
        if (h->L > 0) {
            // resource duals as given; bundle prices g_j = r_j - sum_{l in B_j} eta_l
            for (int64_t l = 0; l < h->L; ++l) t1[l] = eta[l];
            for (int64_t jn = 0; jn < h->N; ++jn) {
                double b = 0.0;
                for (int32_t e = h->bptr_h[jn]; e < h->bptr_h[jn + 1]; ++e) b += eta[h->bres_h[e]];
                t2[jn] = r[jn] - b;
            }
        } else {
            for (int64_t jn = 0; jn < h->N; ++jn) { t1[jn] = eta[h->new2old[jn]]; t2[jn] = r[jn] - t1[jn]; }
        }
        CUDA_TRY(h, cudaMemcpyAsync(h->S.eta, t1.data(), t1.size() * 8, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(h, cudaMemcpyAsync(h->S.g, t2.data(), (h->N + 1) * 8, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    }
    if (s_prev) {
        std::vector<double> t3(h->N + 1, 0.0);
        for (int64_t jn = 0; jn < h->N; ++jn) t3[jn] = s_prev[h->new2old[jn]];
        CUDA_TRY(h, cudaMemcpyAsync(h->S.s_prev, t3.data(), (h->N + 1) * 8, cudaMemcpyHostToDevice, h->stream));
    } else if (y) {
        // s_prev is A y of the current iterate (sampled mode: the running
        // stale-inclusive usage, K3 adds this iteration's delta to it): a
        // restored y without its usage gets a fresh A y (+ the cross-rank sum)
        double *sf = slot_ptr<double>(h, O_TMP);
        CUDA_TRY(h, cudaMemsetAsync(sf, 0, (h->N + 1) * 8, h->stream));
        k_usage<<<h->sm_count * 4, kThreads, 0, h->stream>>>(h->S, T * h->nq, sf, (int32_t)std::min<int64_t>(kHeadMax, h->N));
        CUDA_TRY(h, cudaGetLastError());
        spfom_status st = allreduce(h, sf, sf, (size_t)h->N, kNcclFloat64, kNcclSum);
        if (st != SPFOM_OK) return st;
        CUDA_TRY(h, cudaMemcpyAsync(h->S.s_prev, sf, h->N * 8, cudaMemcpyDeviceToDevice, h->stream));
    }
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return SPFOM_OK;
}

spfom_status spfom_info(const spfom_handle *h_, spfom_info_t *out) {
    if (!h_ || !out) return SPFOM_EINVAL;
    spfom_handle *h = const_cast<spfom_handle *>(h_);
    memset(out, 0, sizeof *out);
    out->num_segments = h->m;
    out->num_periods = h->T;
    out->persistent = h->small ? 1 : 0;
    out->num_products = h->N;
    out->nnz = h->nnz;
    out->nnz_padded = 4 * h->nq;
    out->n_present = h->n_present;
    out->workspace_bytes = (int64_t)h->pl.total;
    out->num_bins = kNumBins;
    out->world = h->world;
    int64_t np = 0;
    for (int b = 0; b < kNumBins; ++b) {
        out->bin_G[b] = kBins[b].G;
        out->bin_Q[b] = kBins[b].Q;
        out->bin_segments[b] = h->pl.sampled ? h->pl.bin_count[b] : (h->bin_first[b + 1] - h->bin_first[b]);
        np += out->bin_segments[b] > 0;
    }
    out->primal_launches_per_iteration = np;
    // primal launches + K3 (+ k_average + k_tick with averaging) (+ k_fold when world > 1)
    out->launches_per_iteration = np + 1 + (h->pl.averaging ? 2 : 0) + (h->comm && h->S.spread_n > 0 ? 1 : 0) +
                                  (h->L > 0 ? 2 : 0);
    return SPFOM_OK;
}

spfom_status spfom_time_kernels(spfom_handle *h, int64_t iters, double *ms) {
    if (!h || !ms || iters < 1) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    cudaEvent_t ev[3];
    for (auto &e : ev) CUDA_TRY(h, cudaEventCreate(&e));
    double acc0 = 0.0, acc1 = 0.0;
    for (int64_t it = 0; it < iters; ++it) {
        const bool refresh = h->graph_refresh && ((h->iter + 1) % h->params.refresh_every == 0);
        CUDA_TRY(h, cudaEventRecord(ev[0], h->stream));
        spfom_status st = enqueue_primal(h, nullptr);
        if (st != SPFOM_OK) return st;
        CUDA_TRY(h, cudaEventRecord(ev[1], h->stream));
        st = enqueue_rest(h, refresh, nullptr);
        if (st != SPFOM_OK) return st;
        CUDA_TRY(h, cudaEventRecord(ev[2], h->stream));
        CUDA_TRY(h, cudaEventSynchronize(ev[2]));
        float a = 0.f, b = 0.f;
        CUDA_TRY(h, cudaEventElapsedTime(&a, ev[0], ev[1]));
        CUDA_TRY(h, cudaEventElapsedTime(&b, ev[1], ev[2]));
        acc0 += a;
        acc1 += b;
        h->iter += 1;
    }
    for (auto &e : ev) cudaEventDestroy(e);
    ms[0] = acc0;
    ms[1] = acc1;
    return SPFOM_OK;
}

spfom_status spfom_step_timed(spfom_handle *h, int64_t k, double *ms) {
    if (!h || !ms || k < 1) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    if (h->small) {
        // the persistent small-regime kernel runs whole iterations: one event pair
        // around all of them; the primal share is not separable (ms[0] = ms[1])
        cudaEvent_t e0, e1;
        CUDA_TRY(h, cudaEventCreate(&e0));
        CUDA_TRY(h, cudaEventCreate(&e1));
        CUDA_TRY(h, cudaEventRecord(e0, h->stream));
        spfom_status st = step_small(h, k);
        if (st == SPFOM_OK) {
            CUDA_TRY(h, cudaEventRecord(e1, h->stream));
            CUDA_TRY(h, cudaEventSynchronize(e1));
            float t = 0.f;
            CUDA_TRY(h, cudaEventElapsedTime(&t, e0, e1));
            ms[0] = ms[1] = t;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return st;
    }
    double primal = 0.0, total = 0.0;
    if (h->graph_refresh) {
        // sampled mode with periodic refreshes: iteration by iteration, events
        // between the primal graph and the rest (plain or refresh) graph
        std::vector<cudaEvent_t> ev(2 * k + 1, nullptr);
        spfom_status st = SPFOM_OK;
        for (auto &e : ev)
            if (st == SPFOM_OK && cudaEventCreate(&e) != cudaSuccess) st = fail(h, SPFOM_ECUDA, "event create");
        for (int64_t it = 0; it < k && st == SPFOM_OK; ++it) {
            const bool refresh = (h->iter + 1) % h->params.refresh_every == 0;
            cudaError_t e = cudaEventRecord(ev[2 * it], h->stream);
            if (e == cudaSuccess) e = cudaGraphLaunch(h->graph_primal, h->stream);
            if (e == cudaSuccess) e = cudaEventRecord(ev[2 * it + 1], h->stream);
            if (e == cudaSuccess) e = cudaGraphLaunch(refresh ? h->graph_rest_refresh : h->graph_rest, h->stream);
            if (e != cudaSuccess) st = fail(h, SPFOM_ECUDA, std::string("spfom_step_timed: ") + cudaGetErrorString(e));
            h->iter += 1;
        }
        if (st == SPFOM_OK && cudaEventRecord(ev[2 * k], h->stream) != cudaSuccess) st = fail(h, SPFOM_ECUDA, "final event");
        if (st == SPFOM_OK) {
            cudaError_t e = cudaEventSynchronize(ev[2 * k]);
            for (int64_t it = 0; it < k && e == cudaSuccess; ++it) {
                float a = 0.f;
                e = cudaEventElapsedTime(&a, ev[2 * it], ev[2 * it + 1]);
                primal += a;
            }
            float tt = 0.f;
            if (e == cudaSuccess) e = cudaEventElapsedTime(&tt, ev[0], ev[2 * k]);
            total = tt;
            if (e != cudaSuccess) st = fail(h, SPFOM_ECUDA, std::string("spfom_step_timed events: ") + cudaGetErrorString(e));
        }
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        ms[0] = primal;
        ms[1] = total;
        return st;
    }
    // chunks of up to kTimedChunk iterations, each one launch of a cached timed
    // graph; the device times of the chunks add up (between chunks the host
    // reads the events: a gap that is not counted)
    constexpr int64_t kTimedChunk = 256;
    for (int64_t done = 0; done < k;) {
        const int64_t c = std::min(k - done, kTimedChunk);
        spfom_handle::TimedGraph *tg = nullptr;
        spfom_status st = timed_graph(h, c, &tg);
        if (st != SPFOM_OK) return st;
        CUDA_TRY(h, cudaGraphLaunch(tg->exec, h->stream));
        CUDA_TRY(h, cudaEventSynchronize(tg->ev[2 * c]));
        for (int64_t it = 0; it < c; ++it) {
            float a = 0.f;
            CUDA_TRY(h, cudaEventElapsedTime(&a, tg->ev[2 * it], tg->ev[2 * it + 1]));
            primal += a;
        }
        float tt = 0.f;
        CUDA_TRY(h, cudaEventElapsedTime(&tt, tg->ev[0], tg->ev[2 * c]));
        total += tt;
        h->iter += c;
        done += c;
    }
    ms[0] = primal;
    ms[1] = total;
    return SPFOM_OK;
}

}   // extern "C" (templates below)

// k_recover over device slots [a, b) of period t, with the row capacity of the
// chunk's longest row (kmax entries)
template <int KM>
void launch_recover_km(spfom_handle *h, int64_t a, int64_t b, int64_t t) {
    constexpr int W = recover_warps<KM>();
    static PerDevice cache;
    int &attr = *cache.slot();
    if (attr < 0) {
        cudaFuncSetAttribute(k_recover<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RecoverSmem<KM>));
        attr = 1;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_recover<KM>, 32 * W, sizeof(RecoverSmem<KM>));
    const int64_t blocks = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)h->sm_count * std::max(1, per_sm), (b - a + W - 1) / W));
    k_recover<KM><<<(unsigned)blocks, 32 * W, sizeof(RecoverSmem<KM>), h->stream>>>(
        h->S, a, b, t, slot_ptr<int32_t>(h, O_ORIG), slot_ptr<int32_t>(h, O_RECORD), slot_ptr<double>(h, O_RECALPHA));
}
void launch_recover(spfom_handle *h, int64_t a, int64_t b, int64_t t, int64_t kmax) {
    if (kmax <= 64) launch_recover_km<64>(h, a, b, t);
    else if (kmax <= 256) launch_recover_km<256>(h, a, b, t);
    else launch_recover_km<kRecoverMaxK>(h, a, b, t);
}
// chunks of device slots whose outputs fit the workspace scratch (CH entries),
// with the longest row of each
std::vector<std::array<int64_t, 3>> recover_chunks(const std::vector<int32_t> &qoff, int64_t m, int64_t CH) {
    std::vector<std::array<int64_t, 3>> out;
    for (int64_t a = 0; a < m;) {
        int64_t b = a + 1, kmax = 4 * (int64_t)(qoff[a + 1] - qoff[a]);
        while (b < m && 4 * (int64_t)(qoff[b + 1] - qoff[a]) <= CH && (b + 1 - a) <= CH) {
            kmax = std::max<int64_t>(kmax, 4 * (int64_t)(qoff[b + 1] - qoff[b]));
            ++b;
        }
        out.push_back({a, b, kmax});
        a = b;
    }
    return out;
}

extern "C" {

spfom_status spfom_recover(spfom_handle *h, int32_t *order, double *alpha) {
    if (!h || !order || !alpha) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    const int64_t CH = recover_chunk(h->nq), m = h->m;
    std::vector<int32_t> qoff(m + 1);
    CUDA_TRY(h, cudaMemcpyAsync(qoff.data(), h->S.qoff, (m + 1) * 4, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    int32_t *dord = slot_ptr<int32_t>(h, O_RECORD);
    double *dal = slot_ptr<double>(h, O_RECALPHA);
    std::vector<int32_t> hord(CH);
    std::vector<double> hal(2 * CH);
    const auto chunks = recover_chunks(qoff, m, CH);
    for (int64_t t = 0; t < h->T; ++t) {
        for (const auto &c : chunks) {
            const int64_t a = c[0], b = c[1];
            launch_recover(h, a, b, t, c[2]);
            CUDA_TRY(h, cudaGetLastError());
            const int64_t ne = 4 * (int64_t)(qoff[b] - qoff[a]);
            if (ne) CUDA_TRY(h, cudaMemcpyAsync(hord.data(), dord, ne * 4, cudaMemcpyDeviceToHost, h->stream));
            CUDA_TRY(h, cudaMemcpyAsync(hal.data(), dal, (ne + (b - a)) * 8, cudaMemcpyDeviceToHost, h->stream));
            CUDA_TRY(h, cudaStreamSynchronize(h->stream));
            for (int64_t k = a; k < b; ++k) {
                const int64_t i = h->sorder[k];                          // original local segment
                const int64_t e0 = h->seg_off[i], len = h->seg_off[i + 1] - e0;
                const int64_t ob = 4 * (int64_t)(qoff[k] - qoff[a]), ab = ob + (k - a);
                int32_t *o = order + t * h->nnz + e0;
                double *al = alpha + t * (h->nnz + m) + e0 + i;
                for (int64_t r = 0; r < len; ++r) o[r] = hord[ob + r];
                for (int64_t l = 0; l <= len; ++l) al[l] = hal[ab + l];
            }
        }
    }
    return check_counters(h);
}

spfom_status spfom_recover_timed(spfom_handle *h, double *ms) {
    if (!h || !ms) return SPFOM_EINVAL;
    DeviceGuard dg_(h->device);
    const int64_t CH = recover_chunk(h->nq), m = h->m;
    std::vector<int32_t> qoff(m + 1);
    CUDA_TRY(h, cudaMemcpyAsync(qoff.data(), h->S.qoff, (m + 1) * 4, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    const auto chunks = recover_chunks(qoff, m, CH);   // the same launches as spfom_recover
    cudaEvent_t e0, e1;
    CUDA_TRY(h, cudaEventCreate(&e0));
    CUDA_TRY(h, cudaEventCreate(&e1));
    CUDA_TRY(h, cudaEventRecord(e0, h->stream));
    for (int64_t t = 0; t < h->T; ++t)
        for (const auto &c : chunks) launch_recover(h, c[0], c[1], t, c[2]);
    CUDA_TRY(h, cudaGetLastError());
    CUDA_TRY(h, cudaEventRecord(e1, h->stream));
    CUDA_TRY(h, cudaEventSynchronize(e1));
    float f = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&f, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ms[0] = f;
    ms[1] = (double)(chunks.size() * h->T);
    return SPFOM_OK;
}

int64_t spfom_iteration(const spfom_handle *h) { return h ? h->iter : -1; }

const char *spfom_last_error(const spfom_handle *h) { return h ? h->err.c_str() : g_create_error.c_str(); }

void spfom_destroy(spfom_handle *h) {
    if (!h) return;
    DeviceGuard dg_(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->graph) cudaGraphExecDestroy(h->graph);
    if (h->graph_refresh) cudaGraphExecDestroy(h->graph_refresh);
    for (cudaGraphExec_t g : {h->graph_u, h->graph_primal, h->graph_rest, h->graph_rest_refresh})
        if (g) cudaGraphExecDestroy(g);
    destroy_timed(h);
    if (h->comm && nccl().ok) nccl().CommDestroy(h->comm);
    for (int b = 0; b < kNumBins; ++b) {
        if (h->side[b]) cudaStreamDestroy(h->side[b]);
        if (h->ev_join[b]) cudaEventDestroy(h->ev_join[b]);
    }
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    for (int c = 0; c < 2; ++c) {
        if (h->pin_ev[c]) cudaEventSynchronize(h->pin_ev[c]);   // last copy through the buffer done
        pin_give(h->pin[c]);
        if (h->pin_ev[c]) cudaEventDestroy(h->pin_ev[c]);
    }
    if (h->own_stream) cudaStreamDestroy(h->stream);
    delete h;
}

}  // extern "C"

#ifdef SPFOM_DIAG_SPAN
extern "C" int spfom_diag_span(unsigned long long *out, int reset) {
    int e = (int)cudaMemcpyFromSymbol(out, spfom::g_diag_span, 4 * 160 * sizeof(unsigned long long));
    if (!e) e = (int)cudaMemcpyFromSymbol(out + 4 * 160, spfom::g_diag_key, 160 * sizeof(unsigned int));
    if (reset) {
        static unsigned long long z[4 * 160] = {0};
        cudaMemcpyToSymbol(spfom::g_diag_span, z, sizeof z);
    }
    return e;
}
#endif
#ifdef SPFOM_DIAG_PHASE
extern "C" int spfom_diag_phase(unsigned long long *out, int reset) {
    int e = (int)cudaMemcpyFromSymbol(out, spfom::g_diag_phase, 10 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(spfom::g_diag_phase, z, sizeof z);
    }
    return e;
}
#endif
#ifdef SPFOM_DIAG_TIME
extern "C" int spfom_diag_time(uint64_t *out, int n) {
    return (int)cudaMemcpyFromSymbol(out, spfom::g_diag_time, sizeof(uint64_t) * (size_t)n);
}
extern "C" int spfom_diag_loops(uint32_t *out, int n) {
    return (int)cudaMemcpyFromSymbol(out, spfom::g_diag_loops, sizeof(uint32_t) * (size_t)n);
}
#endif
