/*
 * spfom.h -- C ABI of the B200-native SPFOM iteration for the GAM sales-based
 * LP (arXiv 2602.22421, "Huge-Scale Assortment Optimization with Customer
 * Choice: A Parallel Primal-Dual Approach").
 *
 * One iteration (PAPER.md = P):
 *   a1  block selection I_t (full sweep, or a pre-generated sampled block,
 *       P:L353 "Randomly generate a subset of customers ... with size B")
 *   a2  price gather g_ij = r_j - eta_j
 *   a3  gradient step z_ij = y_ij + theta g_ij, z_i0 = y_i0
 *   a4  projection of (z_i0, z_i) onto the segment polytope Y_i
 *       (Eqs. 8-10, GAM reading); theta = INFINITY
 *       replaces a3+a4 by the exact inner argmax z_i (Alg. 2)
 *   a5  usage s_j = sum_i y_ij = (A y)_j
 *   a6  cross-rank sum of s (NCCL allreduce, Alg. 3)
 *   a7  eta_j <- max{0, (1 - tau_j mu) eta_j - tau_j (c_j - st_j)},
 *       st = s + omega_x (s - s_prev)    (Eq. 17; omega_x and
 *       per-product tau_j are NOT in the paper: DESIGN.md readings c8)
 *   a8  optional uniform averaging of (y, y0, eta)   (NOT in the paper, c9)
 *
 * Naming (BASELINE.json): m segments i (the paper's n customers), N products j
 * (the paper's m), v_ij attraction (the paper's w_ij), w_ij GAM shadow
 * attraction (the paper's v_ij), lambda_i arrival rate, r_j price, c_j
 * capacity, eta_j capacity dual (bid price).
 *
 * All reals are IEEE binary64.  Ids are 0-based.  Every entry point returns an
 * spfom_status; the message of the last failure is spfom_last_error().
 *
 * Memory and ownership: the caller owns every input array (host memory; the
 * library copies what it needs during spfom_create and never keeps a caller
 * pointer, except `params.blocks`, which is copied too).  Device memory is a
 * single caller-allocated workspace (PyTorch allocates it) of at least
 * spfom_workspace_bytes() bytes, owned by the caller and used exclusively by
 * the handle until spfom_destroy.  The library allocates no device memory of
 * its own except what CUDA graphs and NCCL allocate internally.
 * All device work is enqueued on the caller's CUDA stream.
 *
 * Threading: a handle is not reentrant; distinct handles are independent.
 * With world > 1 every call except spfom_iteration / spfom_last_error /
 * spfom_destroy is collective over the ranks of the handle's communicator.
 */
#ifndef SPFOM_H_
#define SPFOM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (exit-code semantics of S:L658). */
typedef enum {
    SPFOM_OK = 0,
    SPFOM_EINVAL = 1,   /* bad argument or parameter                          */
    SPFOM_EDATA = 2,    /* invalid instance (message names the first offender)*/
    SPFOM_ENUMERIC = 3, /* projection did not converge / non-finite value     */
    SPFOM_ECUDA = 4,    /* CUDA runtime error                                  */
    SPFOM_ENCCL = 5,    /* NCCL error (world > 1)                              */
    SPFOM_ENOMEM = 6    /* workspace too small                                 */
} spfom_status;

/*
 * Instance (host arrays), this rank's contiguous shard of segments.
 *   seg_ptr      [num_segments+1] int64 CSR offsets, seg_ptr[0] = 0, nondecreasing
 *   prod_idx     [nnz] int32, strictly increasing within a row, in [0, num_products)
 *   attract      [nnz] v_ij > 0
 *   shadow       [nnz] 0 <= w_ij < v_ij, or NULL for MNL (w = 0)
 *   no_purchase  [num_segments] v_i0 > 0
 *   arrival      [num_segments] lambda_i > 0
 *   price        [num_products] r_j >= 0 (replicated on every rank)
 *   capacity     [num_products] c_j >= 0 (replicated on every rank)
 *   segment_offset  global id of local segment 0 (sampled blocks use global ids)
 *   num_segments_global  total m over all ranks
 *   num_periods  T; 0 or 1 = single period.  T > 1: multi-period SBLP with a
 *                shared structure (reading c15, SPEC stack_periods):
 *                the CSR arrays, attract, shadow and no_purchase describe the
 *                num_segments BASE segments once; arrival is [T][num_segments]
 *                (period-major); segment (t, i) of the stacked SBLP has
 *                consideration set C_i, weights v_i., w_i., v_i0 and arrival
 *                arrival[t * num_segments + i], and every period shares one
 *                inventory c_j.  The device stores the structure once and y as
 *                [T][entries]; getters return stacked (period-major) order:
 *                y [T][nnz], y0 [T][num_segments].  n_j (tau_j = tau / n_j)
 *                counts stacked segments (T x base count).  Sampled blocks are
 *                not supported with T > 1 (SPFOM_EINVAL); rows must have <= 512
 *                entries (SPFOM_EDATA).
 *   num_resources  L; 0 = every product is its own capacity row (capacity[j]).
 *                L > 0: bundles / NRM (Eq. 33): product j
 *                is a bundle consuming the base resources bundle_res[bundle_ptr[j]
 *                .. bundle_ptr[j+1]) (strictly increasing, >= 1 per bundle, < L);
 *                the capacity rows are sum_i sum_j Bt_lj y_ij <= resource_capacity[l];
 *                `capacity` is ignored; the duals eta (spfom_duals, set_state,
 *                averages) are per resource (length L); prices g_j = r_j -
 *                sum_{l in B_j} eta_l; tau_l = tau / n_l with n_l = sum_{j : l in B_j}
 *                n_j (tau_mode 1, reading c17).
 *   on_device    0: every array above is host memory.  1: every array is device
 *                memory readable from the current device (e.g. torch tensors):
 *                spfom_workspace_bytes / spfom_create stage them to host memory
 *                first (the layout build is a host pass) and keep no pointer;
 *                unreadable pointers => SPFOM_EINVAL.  (SPEC S:L31-37 data model;
 *                SURVEY §8(b) `on_device`.)
 * Violations are reported as SPFOM_EDATA.
 */
typedef struct {
    int64_t num_segments;
    int64_t num_products;
    int64_t nnz;
    int64_t segment_offset;
    int64_t num_segments_global;
    const int64_t *seg_ptr;
    const int32_t *prod_idx;
    const double *attract;
    const double *shadow;
    const double *no_purchase;
    const double *arrival;
    const double *price;
    const double *capacity;
    int64_t num_periods;
    int64_t num_resources;
    const int64_t *bundle_ptr;
    const int32_t *bundle_res;
    const double *resource_capacity;
    int64_t on_device;
} spfom_instance;

/*
 * Parameters (SURVEY §8(c) c8 presets):
 *   paper:    theta = INFINITY, tau_mode = 0, tau = 0.1, mu >= 0,
 *             extrapolation = 0, sampled blocks, averaging = 0
 *   converge: theta = 1, tau_mode = 1, tau = 0.9, mu = 0, extrapolation = 1,
 *             full sweep, averaging = 0
 *   theta          primal step > 0; INFINITY => exact inner argmax
 *   tau, tau_mode  tau_j = tau (mode 0) or tau / n_j (mode 1; n_j = global
 *                  number of segments considering j; tau when n_j = 0)
 *   mu             Eq. 17 penalty >= 0 with tau_j mu <= 1
 *   extrapolation  omega_x in [0, 1]
 *   averaging      0 / 1
 *   blocks         NULL => full sweep; else [block_iters][block_size] int32
 *                  global segment ids, each row strictly increasing; iteration
 *                  t uses row t mod block_iters.  Copied at create.
 *   refresh_every  sampled mode: recompute s = A y from scratch every K
 *                  iterations (0 = never)
 *   exec_mode      0 = auto; 1 = one CUDA-graph replay per iteration (primal
 *                  kernels, K3); 2 = persistent cooperative kernel running
 *                  whole iterations per launch (grid-wide barriers between the
 *                  primal and dual phases) -- the small regime: world == 1,
 *                  T == 1, no averaging / refresh, rows <= 1024 entries and at
 *                  most 4096 segments per iteration (SPFOM_EINVAL otherwise).
 *                  Auto picks 2 when eligible.  Results are identical up to
 *                  summation order.
 *   max_newton     cap on projection passes per segment (0 => 200); a segment
 *                  still unconverged after half of it restarts from the cold
 *                  point; one that exhausts it is counted as a failure and
 *                  makes the next synchronising getter return SPFOM_ENUMERIC
 */
typedef struct {
    double theta;
    double tau;
    double mu;
    double extrapolation;
    int32_t tau_mode;
    int32_t averaging;
    int32_t max_newton;
    int32_t exec_mode;
    int64_t block_size;
    int64_t block_iters;
    const int32_t *blocks;
    int64_t refresh_every;
} spfom_params;

/* Distribution: nccl_id points at the 128-byte
 * ncclUniqueId produced on rank 0 by spfom_nccl_unique_id() and broadcast by
 * the caller (torch.distributed).  world > 1 needs it.  world == 1 with
 * nccl_id == NULL (or no spfom_dist at all) => single GPU; world == 1 with an
 * id runs the multi-rank code path (NCCL allreduce of the usage, k_fold) on
 * one GPU with identical results -- a way to exercise it without peers. */
/* Per iteration with world > 1 (products, no bundles), inside the CUDA graph:
 * K1's usage partials -> ncclReduceScatter (rank r gets the summed usage of
 * products [r c, (r + 1) c), c = ceil((N + 1) / world)) -> the Eq. 17 dual step
 * on that slice only -> ncclAllGather of the prices g = r - eta.  eta and the
 * usage stay sliced between iterations; spfom_duals / spfom_usage /
 * spfom_averages / spfom_residuals gather them first (they are collective).
 * Bundles (num_resources > 0), or the environment variable
 * SPFOM_COLLECTIVE=allreduce at create, use ncclAllReduce of the usage and the
 * dual step on every rank instead.  world <= 64. */
typedef struct {
    int32_t rank;
    int32_t world;
    const void *nccl_id;
} spfom_dist;

/* Residuals and certificate (reading c11).  With world > 1 they are global. */
typedef struct {
    int64_t iteration;
    double primal_obj;      /* P = sum_j r_j s_j, s = fresh A y            */
    double dual_obj;        /* D = c^T eta + sum_i lambda_i z_i*(r - eta)  */
    double rel_gap;         /* (D - P) / (1 + |P| + |D|)                   */
    double infeas_abs;      /* max_j (s_j - c_j)^+                         */
    double infeas_rel;      /* max_j (s_j - c_j)^+ / max(1, c_j)  (gate)   */
    double infeas_rel_l2;   /* ||(s - c)^+||_2 / (1 + ||c||_2)             */
    double balance_rel_max; /* max_i |y_i0 + sum_j y_ij - lambda_i| / lambda_i */
    double scale_rel_max;   /* max_ij (y_ij - v_ij U_i)^+ / lambda_i       */
    double neg_max;         /* max (-y)^+                                   */
    double compl_slack;     /* sum_j eta_j |c_j - s_j| / (1 + |P|)          */
    double cert_lower;      /* (1 - alpha) P, alpha = max_j (s_j - c_j)^+ / s_j */
    double cert_upper;      /* D                                            */
    double alpha;
    int64_t newton_failures;/* segments whose projection hit max_newton     */
    int64_t newton_passes;  /* total projection passes since create         */
    int64_t newton_restarts;/* segment-iterations that used the cold restart */
} spfom_residuals_t;

typedef struct spfom_handle spfom_handle;

/* Bytes of device workspace the instance needs (reads seg_ptr / sizes only). */
spfom_status spfom_workspace_bytes(const spfom_instance *inst, const spfom_params *params,
                                   size_t *bytes);

/* Validate, lay out (product relabelling by popularity, padded 128-bit CSR,
 * length bins), copy to the workspace, initialise y = 0, y0 = lambda,
 * eta = 0, s = 0 (reading c10).  cuda_stream: cudaStream_t; NULL (or the
 * legacy default stream, which cannot be graph-captured) => the handle creates
 * and owns a private non-blocking stream.  workspace: 256-byte aligned device
 * pointer of >= spfom_workspace_bytes() bytes.  The handle also holds a 40 MB
 * pinned host staging ring (two cudaMallocHost buffers): the padded CSR is
 * built into it chunk by chunk and uploaded while the next chunk is built, and
 * the getters stage their device->host copies through it.  The buffers come
 * from a process-wide pool: spfom_destroy returns them (after their last copy
 * completed) for the next handle, and the pool is not released before the
 * process exits (SPFOM_NO_PIN_POOL=1: always allocate fresh).  SPFOM_ENOMEM if
 * the ring cannot be allocated. */
spfom_status spfom_create(const spfom_instance *inst, const spfom_params *params,
                          const spfom_dist *dist, void *cuda_stream, void *workspace,
                          size_t workspace_bytes, spfom_handle **out);

/* Enqueue k iterations on the stream (asynchronous; CUDA-graph replay). */
spfom_status spfom_step(spfom_handle *h, int64_t k);

/* Synchronising getters, results in ORIGINAL product / entry order. */
spfom_status spfom_duals(spfom_handle *h, double *eta /* [N] */);
spfom_status spfom_primal(spfom_handle *h, double *y /* [nnz] local */, double *y0 /* [m] local */);
spfom_status spfom_usage(spfom_handle *h, double *s /* [N] = A y of the last iteration */);
spfom_status spfom_averages(spfom_handle *h, double *ybar, double *y0bar, double *etabar);
spfom_status spfom_objective(spfom_handle *h, double *obj);       /* r^T (A y), fresh */
spfom_status spfom_residuals(spfom_handle *h, spfom_residuals_t *out);

/* Overwrite the iterate (checkpoint / resume): original orders, like the getters.
 * Any argument may be NULL (that part of the state is kept).  s_prev is the
 * usage A y of the iterate (sampled mode: the running stale-inclusive usage the
 * next dual step adds its delta to): when y is given without s_prev, the
 * library recomputes s_prev = A y on the device (cross-rank sum when world > 1),
 * so the next dual step is consistent with the restored y.  The projection's
 * warm-start multipliers are kept (they only change the Newton starting point,
 * not the result), and so are the iteration counter and, with averaging, the
 * running averages (set_state restores the iterate, not the averages). */
spfom_status spfom_set_state(spfom_handle *h, const double *y, const double *y0, const double *eta,
                             const double *s_prev);

/* Layout and launch facts of a handle (for the roofline and launch counts). */
typedef struct {
    int64_t num_segments, num_products, nnz, nnz_padded, n_present;
    int64_t launches_per_iteration;   /* library kernels per iteration (NCCL excluded) */
    int64_t primal_launches_per_iteration;
    int64_t workspace_bytes;
    int64_t bin_segments[8];          /* segments per length bin (G, Q) */
    int32_t bin_G[8], bin_Q[8];
    int32_t num_bins, world;
    int64_t num_periods;              /* T (1 = single period) */
    int64_t persistent;               /* 1: spfom_step runs the small-regime persistent kernel */
} spfom_info_t;
spfom_status spfom_info(const spfom_handle *h, spfom_info_t *out);

/* Measurement helper: run `iters` iterations WITHOUT the graph, recording CUDA
 * events on the handle's stream around (a) the primal kernels K1 and (b) the
 * rest of the iteration (allreduce + K3 + tick); synchronises and writes the
 * summed milliseconds to ms[0] (K1) and ms[1] (rest).  Advances the iterate. */
spfom_status spfom_time_kernels(spfom_handle *h, int64_t iters, double *ms);

/* SBLP -> CBLP policy recovery of the current iterate (P:L473-492 Lemma
 * "recover"; GAM reading SV App. A.1), computed on the
 * device (one warp per segment, in chunks through a workspace scratch area).
 * For row i (original order; stacked period blocks when num_periods > 1):
 *   order[seg_ptr[i] .. seg_ptr[i+1])      int32 original product ids sorted by
 *                                          u_ij = y_ij / v_ij descending, ties by
 *                                          ascending product id;
 *   alpha[seg_ptr[i] + i .. seg_ptr[i+1] + i]  probabilities of the nested
 *                                          assortments S_0 (no product) .. S_k,
 *                                          S_l = the first l products of order:
 *   alpha_l = (u_(l) - u_(l+1)) * D(S_l) / lambda_i, u_(0) = U_i =
 *   (y_i0 + sum_j w_ij / v_ij y_ij) / vt_i0, u_(k+1) = 0,
 *   D(S) = v_i0 + sum_{j in S} v_ij + sum_{j in C_i \ S} w_ij.
 * Sizes: order [T][nnz], alpha [T][nnz + num_segments] (caller-owned host
 * arrays).  Synchronous; SPFOM_ENUMERIC if projection failures were counted. */
spfom_status spfom_recover(spfom_handle *h, int32_t *order, double *alpha);

/* Measurement helper for the recovery kernel (bench.py --mode features): run
 * the device part of spfom_recover -- every chunk of every period, the same
 * launches -- into the workspace only (no host copies, results discarded),
 * with CUDA events on the handle's stream around all launches; synchronises
 * and writes ms[0] = elapsed milliseconds, ms[1] = number of launches. */
spfom_status spfom_recover_timed(spfom_handle *h, double *ms);

/* Timed stepping (bench.py's timed region): enqueue k iterations exactly like
 * spfom_step -- one replay of the iteration's CUDA graph each, whose two
 * event-record nodes (before and after the primal kernels a1-a5) are pointed at
 * that iteration's pair of CUDA events before the launch (sampled refresh
 * iterations use two graphs with the events between them) -- then synchronise
 * and write ms[0] = summed event time of the primal kernels over the k
 * iterations, ms[1] = event time from the first to the last event (all k
 * iterations).  In the small regime (spfom_info.persistent) the iterations run
 * inside the persistent kernel: ms[0] = ms[1] = their event time.
 * Collective when world > 1.  Advances the iterate by k. */
spfom_status spfom_step_timed(spfom_handle *h, int64_t k, double *ms);

int64_t spfom_iteration(const spfom_handle *h);
const char *spfom_last_error(const spfom_handle *h); /* NULL handle => thread's last create error */
/* Frees the handle (graphs, streams, events, the NCCL communicator); the
 * pinned staging ring goes back to the process-wide pool (spfom_create).  The
 * caller's workspace is not touched. */
void spfom_destroy(spfom_handle *h);

/* --- host-side helpers (no GPU needed) ------------------------------------- */

/* Contiguous segment ranges balanced by nnz: bounds[r] .. bounds[r+1] for rank
 * r (bounds has world+1 entries); each rank's nnz is within one segment of
 * nnz / world.  Pure host function. */
spfom_status spfom_partition(const int64_t *seg_ptr, int64_t num_segments, int32_t world,
                             int64_t *bounds);

/* 128-byte ncclUniqueId for a new communicator (rank 0 only). */
spfom_status spfom_nccl_unique_id(void *out128);

/* sizeof of the ABI structs, for bindings to check their mirrors (host only):
 * out[0] spfom_instance, out[1] spfom_params, out[2] spfom_info_t,
 * out[3] spfom_residuals_t, out[4] spfom_dist. */
void spfom_abi_sizes(size_t *out);

/* Build information string (arch, version). */
const char *spfom_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SPFOM_H_ */
