/* ===========================================================================
 * fleet_plan.h -- C ABI of the B200 fleet-sizing sweep
 * (token-budget pool routing, arxiv 2604.08075).
 *
 * The library evaluates the paper's two-pool provisioning method over a whole
 * request trace on the GPU:
 *   route_batch      -- Alg. 1 applied to every request
 *                       of a trace for ONE (B_short, C_S, C_L) split;
 *   sweep_thresholds -- one HBM pass that routes every request against EVERY
 *                       candidate split at once (empirical CDF), then
 *                       sizes every (model, GPU, C_L, C_S, B) candidate with
 *                       Eq. (1)-(2), the Sec. 3 pool sizing
 *                       G = ceil(lambda/mu), Eq. `savings`
 *                        and annual cost;
 *   best_split       -- the per-model cheapest feasible candidate.
 * Readings of points where the paper is silent are DESIGN.md R1..R20.
 *
 * Conventions (all entry points):
 *   - Plain C types only. Device pointers (d_*) are CUDA device addresses on
 *     the plan's device; host pointers (h_*) are CPU addresses.
 *   - Return codes only: no exceptions cross the ABI, nothing aborts. The
 *     per-plan message of the last failure is fp_last_error(plan).
 *   - Calls are stream-ordered and asynchronous on `stream` (a cudaStream_t
 *     passed as void*, NULL = legacy default stream), EXCEPT: a non-NULL host
 *     output pointer makes the call synchronize `stream` before returning,
 *     and best_split always synchronizes.
 *   - The caller owns every buffer it passes and must not modify d_len /
 *     d_decision until the stream has passed the call. The plan owns its
 *     scratch memory, NCCL communicator and streams; fleet_plan_destroy frees
 *     them.
 *   - A plan is not thread-safe; distinct plans are independent.
 *   - Multi-GPU (world > 1): every rank must issue the same sequence of
 *     route_batch / sweep_thresholds / best_split calls with the same
 *     descriptor (NCCL collective semantics).
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     call fails with FP_ERR_CUDA.
 *   - Kernels that follow another kernel of the same call are issued as
 *     programmatic dependent launches (they wait on the device for their
 *     predecessor's results); environment FP_NO_PDL=1 issues plain launches.
 *     Either way the results are identical and the calls stay stream-ordered
 *     with respect to the caller's other work on `stream`.
 *   - Other environment knobs select measured alternatives with identical
 *     results: FP_SPEC_STRIPES (speculative sample stripes, 4),
 *     FP_SPEC_MIN_WIDE_LOG2 (u16-LUT speculation threshold, 28),
 *     FP_CALIB_STREAM=1 (calibrate_replay's single-pass streaming kernel,
 *     slower on a B200), FP_CALIB_PROFILE=1 (its phase stamps), FP_K3_PHASES=1
 *     (K3 phase stamps), FP_K4_BLOCK / FP_K4_BLOCKS_PER_SM (routing launch).
 * ======================================================================== */
#ifndef FLEET_PLAN_H
#define FLEET_PLAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP_ABI_VERSION 2u
#define FP_NAME_LEN 32

typedef enum fp_status {
  FP_OK = 0,
  FP_ERR_INVALID_ARG = 1, /* NULL where not allowed, invalid split, bad sizes      */
  FP_ERR_CONFIG = 2,      /* descriptor violates a documented constraint           */
  FP_ERR_EMPTY_TRACE = 3, /* sweep over zero requests (alpha undefined)     */
  FP_ERR_ALIGNMENT = 4,   /* reserved (misaligned d_len is handled, not rejected)  */
  FP_ERR_OOM = 5,         /* device or pinned-host allocation failed               */
  FP_ERR_CUDA = 6,        /* CUDA runtime/launch error, or no device               */
  FP_ERR_NCCL = 7,        /* NCCL unavailable or a collective failed               */
  FP_ERR_STATE = 8        /* call out of order (e.g. best_split before a sweep)    */
} fp_status;

/* ---- descriptor ----------------------------------------------------------- */

/* Model: the symbols of Eq. (1) `eq:kv-per-seq`. */
typedef struct fp_model {
  char name[FP_NAME_LEN];
  uint32_t n_layers;      /* n_l                                             */
  uint32_t n_kv_heads;    /* n_h (KV heads)                                  */
  uint32_t head_dim;      /* d_h                                             */
  uint32_t kv_elem_bytes; /* b_dtype (1, 2 or 4)                             */
} fp_model;

/* GPU: the symbols of Eq. (2) `eq:max-seqs` plus the activation
 * reserve of the Sec. 4.7 budget and a price. */
typedef struct fp_gpu {
  char name[FP_NAME_LEN];
  uint64_t hbm_bytes;                /* M_gpu                               */
  uint32_t util_num, util_den;       /* u = util_num / util_den, 0 < u <= 1 */
  uint64_t activation_reserve_bytes; /* subtracted from M_gpu * u           */
  double price_per_gpu_hour;         /* $ per GPU-hour, >= 0                */
} fp_gpu;

/* Deployment of model m on GPU g (row-major [n_models][n_gpus]). */
typedef struct fp_deploy {
  uint32_t tp_degree;            /* KV is split over tp GPUs: per-GPU M_seq = M_seq / tp */
  uint32_t gpus_per_instance;    /* GPUs counted per instance (DESIGN R6), >= 1          */
  uint64_t weight_bytes_per_gpu; /* M_model                                              */
} fp_deploy;

/* Candidate grid. Flat candidate index order (m, g, C_L, C_S, B), B fastest:
 *   index = (((m * n_gpus + g) * n_cl + l) * n_cs' + s) * n_b + k,
 *   n_cs' = max(n_cs, 1). n_cs == 0 ties C_S = B (Fig. 6 convention, R16).
 * A candidate is valid iff B <= C_S <= C_L. Every value >= 1.  */
typedef struct fp_grid {
  const uint32_t *b_short; uint32_t n_b;  /* thresholds B_short (tokens)      */
  const uint32_t *c_short; uint32_t n_cs; /* short-pool windows C_S, or none  */
  const uint32_t *c_long;  uint32_t n_cl; /* long-pool windows C_L (= C_H)    */
} fp_grid;

#define FP_FLAG_NO_MASS 0x1u         /* skip token-mass sums (occupancy = 0)          */
#define FP_FLAG_REPLICATED_GRID 0x2u /* world > 1: every rank evaluates all candidates */
#define FP_FLAG_KERNEL_TIMING 0x4u   /* record CUDA events around every kernel launch   */
#define FP_FLAG_CHECK_ORDER 0x8u     /* sweep_peak_windows: verify arrival order (8 B/req) */
#define FP_FLAG_TIME_TRACE 0x20u     /* record CUDA events around the trace-pass kernel
                                        only (each event pair costs a few us of stream
                                        time; timing K3/K4 too adds ~16 us per step)    */
#define FP_FLAG_P2P 0x40u            /* world > 1 (or FP_FLAG_COLLECTIVES): the sweep's
                                        histogram exchange goes through peer memory --
                                        each rank folds its K1 accumulators into one
                                        histogram and publishes it; every rank's K3
                                        reads all of them over NVLink (CUDA IPC), no
                                        all-reduce; implies FP_FLAG_REPLICATED_GRID.
                                        K3's wait for a peer is bounded (env
                                        FP_P2P_TIMEOUT_MS, default 10000): on timeout
                                        the sweep's results are invalid and the next
                                        synchronising call (best_split,
                                        sweep_histogram, a sweep with h_results)
                                        returns FP_ERR_NCCL.
                                        Needs fp_p2p_export / fp_p2p_import before the
                                        first sweep; NCCL or the hooks still serve
                                        route_batch, calibrate_replay, peak windows.
                                        Every rank must issue the same sequence of
                                        sweeps: a rank's K3 waits on the device for
                                        every peer's K1 of the same step. world <= 64 */
#define FP_FLAG_SPECULATE 0x80u      /* sweep_and_route, device trace, and a u8 LUT with
                                        |E| < 127 and >= 2^26 requests on this rank, or a
                                        u16 LUT (|E| >= 256) and >= 2^28 requests
                                        (FP_SPEC_MIN_WIDE_LOG2): speculative routing. A
                                        sample pass (every ~4th grid-wide stripe of this
                                        rank's trace, ~2%) and its K3 (the whole grid,
                                        rank-local) pick a split; the full trace pass
                                        then writes Alg. 1's decision bytes for that split
                                        directly into d_decision (no bin round trip:
                                        5 B/request instead of 6.5); the full K3 picks the
                                        true split and a verify kernel re-routes every
                                        request from L_total when the two differ. Results
                                        are identical to the non-speculative call; only
                                        the time depends on the sample. Difference: when
                                        route_model has no feasible split, d_decision's
                                        contents are unspecified (not left untouched),
                                        and `len` must stay unchanged until the call's
                                        work on `stream` has completed (the verify
                                        kernel may read it)                            */
#define FP_FLAG_COLLECTIVES 0x10u    /* run the cross-rank steps even when world == 1
                                        (a one-rank NCCL communicator or the hooks): the
                                        multi-rank code path on a single GPU, for tests  */

typedef struct fp_plan_desc {
  uint32_t abi_version;           /* FP_ABI_VERSION                                 */
  uint32_t flags;                 /* FP_FLAG_*                                      */
  const fp_model *models; uint32_t n_models;
  const fp_gpu *gpus;     uint32_t n_gpus;
  const fp_deploy *deploy;        /* [n_models][n_gpus]                             */
  fp_grid grid;
  const uint32_t *windows; uint32_t n_windows; /* strictly increasing list of every
                                     pool window a candidate uses (each C_S, C_L,
                                     and each B when n_cs == 0)                      */
  const double *mu_table;         /* [n_models][n_gpus][n_windows] profiled
                                     throughput mu, requests/s per instance (R5);
                                     finite, >= 0                                   */
  double hours_per_year;          /* cost horizon (R7), > 0                          */
  int32_t device;                 /* CUDA device ordinal for this rank               */
  int32_t rank, world;            /* 0 <= rank < world                               */
  const void *nccl_unique_id;     /* 128-byte ncclUniqueId, same on all ranks; used
                                     iff (world > 1 or FP_FLAG_COLLECTIVES) and
                                     collectives == NULL                             */
  const struct fp_collectives *collectives; /* optional host-side collectives that
                                     replace NCCL when world > 1 (NULL = NCCL)        */
} fp_plan_desc;

/* Host-side collective hooks (e.g. MPI or a CPU process group). When given,
 * the library synchronizes the stream, copies the operand to host
 * memory, calls the hook, and copies the result back; NCCL is not used.
 * Every rank must call the hooks in the same order (collective semantics).
 * Each returns 0 on success; anything else fails the call with FP_ERR_NCCL.
 * The struct is copied at fleet_plan_create; `user` must outlive the plan. */
typedef struct fp_collectives {
  /* in place: hbuf[i] = sum over ranks of hbuf[i], i < count */
  int (*allreduce_sum_u64)(uint64_t *hbuf, uint64_t count, void *user);
  /* hrecv[r * bytes .. (r + 1) * bytes) = rank r's hsend[0 .. bytes) */
  int (*allgather_bytes)(const void *hsend, void *hrecv, uint64_t bytes, void *user);
  void *user;
} fp_collectives;

/* ---- outputs -------------------------------------------------------------- */

typedef struct fp_route_counts {
  uint64_t n_short, n_long, n_reject; /* requests per outcome (sum = N)       */
  uint64_t mass_short, mass_long;     /* sum of L_total per served pool       */
} fp_route_counts;

#define FP_CAND_VALID 1u         /* B <= C_S <= C_L                                     */
#define FP_CAND_FEASIBLE 2u      /* both pools buildable (R13); only these enter argmin */
#define FP_CAND_HOMO_FEASIBLE 4u /* the homogeneous C_H = C_L fleet is buildable        */

/* One evaluated candidate (192 bytes). Invalid candidates carry zeros and
 * infinite costs; infeasible pools carry zero instances and infinite cost. */
typedef struct fp_candidate {
  uint32_t index, model, gpu;          /* flat index and (m, g)                   */
  uint32_t b_short, c_short, c_long;   /* the split                               */
  uint32_t flags, _pad;                /* FP_CAND_*                               */
  uint64_t nseq_short, nseq_long;      /* Eq. (2) N_seq at C_S and C_L            */
  uint64_t n_short, n_long, n_reject;  /* routed requests (global)                */
  uint64_t mass_short, mass_long;      /* token mass per pool                     */
  uint64_t inst_short, inst_long, inst_homo; /* ceil(lambda_p / mu_p)            */
  uint64_t gpus_dual, gpus_homo;       /* gpus_per_instance x instances           */
  double alpha;                        /* n_short / N                     */
  double rho;                          /* mu(C_S) / mu(C_L)               */
  double predicted_savings;            /* alpha (1 - 1/rho), Eq. `savings`        */
  double savings;                      /* (G_homo - G_dual) / G_homo              */
  double cost_dual, cost_homo;         /* GPUs x price x hours_per_year           */
  double occupancy_short, occupancy_long; /* mass / (n x C) (R20)     */
} fp_candidate;

typedef struct fp_plan_info {
  uint64_t n_candidates;        /* whole grid                                     */
  uint64_t cand_first, cand_count; /* this rank's slice of the grid             */
  uint32_t n_edges;             /* |E|, E = sortuniq(B u C_L)                     */
  uint32_t lut_shift;           /* s: every edge is a multiple of 2^s             */
  uint32_t lut_cells;           /* cells in the bin LUT (0 = binary-search mode)  */
  uint32_t n_windows;
  int32_t device, rank, world;
  uint32_t sm_count;
  uint32_t k1_grid, k1_block;   /* trace-pass launch configuration                */
  int32_t nccl_comm_size;       /* ranks in the plan's NCCL communicator (0: none) */
  uint32_t k3_shape;            /* K3 launch shape of the sweep: 0 cluster (paper-size
                                   grids), 1 factored (large grids), 2 grid-stride */
  uint32_t k3_blocks_per_model; /* K3 blocks per model (the cluster size for shape 0) */
  uint32_t spec_calls;          /* FP_FLAG_SPECULATE: speculative sweep_and_route calls */
  uint32_t spec_misses;         /* ... whose sampled split was not the final one (the
                                   verify kernel re-routed every request); reading it
                                   synchronizes the plan's last stream             */
} fp_plan_info;

typedef struct fp_plan fp_plan; /* opaque */

/* ---- entry points ----------------------------------------------------------- */

/* Validate `desc`, build the edge set and bin LUT, allocate device scratch on
 * desc->device, and (world > 1) initialise the NCCL communicator from
 * desc->nccl_unique_id. The descriptor's arrays are copied; the caller may
 * free them afterwards. On failure *out = NULL and a status is returned.
 * Errors: FP_ERR_INVALID_ARG (NULL), FP_ERR_CONFIG (constraint violated),
 * FP_ERR_CUDA, FP_ERR_OOM, FP_ERR_NCCL. */
fp_status fleet_plan_create(const fp_plan_desc *desc, fp_plan **out);

/* Alg. 1 for one split over this rank's n_local requests
 * d_len[0..n_local) (u32 L_total, any alignment). Per request writes
 * d_decision[i] = pool | stage << 2 (pool 0 short, 1 long, 2 rejected; stage 0
 * budget step, 1 feasibility step, 2 safety check, 3 rejection) when
 * d_decision != NULL. If h_counts != NULL, writes the GLOBAL counts (summed
 * over ranks) and synchronizes. Requires 1 <= B <= C_S <= C_L
 * (else FP_ERR_INVALID_ARG). n_local == 0 is a valid no-op.
 * d_len may also be a HOST pointer (pinned or pageable): it is then streamed
 * to the device in chunks inside the call; d_decision must be device memory. */
fp_status route_batch(fp_plan *plan, const uint32_t *d_len, uint64_t n_local, uint32_t b_short,
                      uint32_t c_short, uint32_t c_long, uint8_t *d_decision,
                      fp_route_counts *h_counts, void *stream);

/* The fleet-sizing sweep over this rank's shard d_len[0..n_local) at arrival
 * rate rate_rps (lambda, > 0, R17). Enqueues: trace pass + histogram,
 * (world > 1) NCCL all-reduce of the histogram, prefix scan + candidate
 * evaluation + per-model argmin over this rank's candidate slice, and
 * (world > 1, not replicated) an all-gather of the per-rank best records.
 * d_len may be a device pointer or a HOST pointer (streamed in chunks, as in
 * route_batch). If h_results != NULL it receives this rank's candidate slice
 * (fp_plan_info.cand_count records, in index order) and the call synchronizes.
 * Errors: FP_ERR_INVALID_ARG, FP_ERR_EMPTY_TRACE (world == 1 and n_local == 0;
 * with world > 1 an empty global trace is reported by best_split). */
fp_status sweep_thresholds(fp_plan *plan, const uint32_t *d_len, uint64_t n_local,
                           double rate_rps, fp_candidate *h_results, void *stream);

/* Per-model best split of the last sweep: h_best[m] for m < n_models (index =
 * UINT32_MAX and flags = 0 when model m has no feasible candidate).
 * Synchronizes the stream of the last sweep. Deterministic for any world size.
 * Errors: FP_ERR_STATE (no sweep yet), FP_ERR_EMPTY_TRACE (global N == 0). */
fp_status best_split(fp_plan *plan, fp_candidate *h_best);

/* The paper's whole workflow over one trace in one call: sweep_thresholds,
 * best_split (into h_best[n_models] if non-NULL), then route_batch with the
 * best split of model `route_model` (decisions into d_decision if non-NULL,
 * global counts into h_counts if non-NULL). A HOST trace crosses PCIe once:
 * it is copied into a plan-owned device buffer chunk by chunk while the trace
 * pass consumes each chunk, and the routing pass reads the device copy.
 * With |E| < 256 (u8 LUT) the trace pass also writes each request's 1-B bin
 * and the split is picked and applied on the device (no host round trip).
 * With a fine-cell LUT and |E| >= 256 (u16 LUT) and a DEVICE trace the same
 * holds with clamped bins (min(bin, 255)): the routing pass reads `len` back
 * for requests whose byte is 255 when the split has an edge index >= 255, so
 * `len` must stay unchanged until the call's work has completed on `stream`.
 * With FP_FLAG_SPECULATE (see the flag) the speculative form runs instead
 * where its preconditions hold: the same outputs from one full trace pass.
 * Synchronizes -- except in that bin mode with a device trace when h_best and
 * h_counts are both NULL: then the call is stream-ordered and asynchronous,
 * the records stay on the device for a later best_split, and a model without
 * a feasible split leaves d_decision untouched (best_split shows it).
 * Errors: as the three calls; FP_ERR_STATE if route_model has no feasible
 * split (h_best is still written). */
fp_status sweep_and_route(fp_plan *plan, const uint32_t *len, uint64_t n_local, double rate_rps,
                          uint32_t route_model, uint8_t *d_decision, fp_candidate *h_best,
                          fp_route_counts *h_counts, void *stream);

/* The step of sweep_and_route in its asynchronous form (device trace, bin
 * mode, h_best = h_counts = NULL) as a CUDA graph owned by the plan: the first
 * call with a given (len, n_local, rate_rps, route_model, d_decision) runs the
 * step once eagerly, then captures it -- once per accumulator parity (each
 * step's K3 clears the other parity's histogram copies for the next step), on
 * a plan-owned stream -- and every call launches the parity's graph on
 * `stream` (any stream, including the legacy default): one cudaGraphLaunch
 * instead of 3-5 kernel launches (the small traces' steps are launch-bound,
 * the plan owns the captured graph). Results are those of
 * sweep_and_route; read them with best_split / sweep_histogram. Same
 * contract on len and d_decision as the asynchronous call (caller-owned,
 * unchanged until the stream passes the call). Another argument tuple, or a
 * scratch reallocation by another call, recaptures. One rank only (world ==
 * 1, no FP_FLAG_COLLECTIVES / FP_FLAG_P2P) and no FP_FLAG_KERNEL_TIMING /
 * FP_FLAG_TIME_TRACE (FP_ERR_CONFIG otherwise); FP_ERR_INVALID_ARG for a
 * host trace, a NULL d_decision or n_local == 0; a step that the
 * asynchronous form cannot run (host outputs needed: |E| >= 256 with a host
 * trace, binary-search bins) gives FP_ERR_CONFIG. */
fp_status sweep_and_route_graph(fp_plan *plan, const uint32_t *len, uint64_t n_local, double rate_rps,
                                uint32_t route_model, uint8_t *d_decision, void *stream);

/* ---- token-budget estimation (NEXT-1) ----------------------------------------
 * Routing key from raw request columns (Eq. `budget`, with the
 * conservative ratio of Eq. `conservative`, Alg. 1):
 *   c*_k    = max(c_hat_k - gamma * sigma_hat_k, c_floor)     (R22)
 *   L_total = min(ceil(|r| / c*_k) + max_output_tokens, 2^32 - 1)
 * in IEEE binary64 (one division and a ceil per request), category
 * k >= n_cats counted as the last category ("mixed/other", R23). */
typedef struct fp_category_calibration {
  double c_hat;      /* calibrated bytes per token of the category (Eq. `ema`)   */
  double sigma_hat;  /* its EMA deviation, >= 0                                   */
} fp_category_calibration;

typedef struct fp_estimator {
  const fp_category_calibration *cats; /* frozen snapshot, indexed by category  */
  uint32_t n_cats;                     /* 1..256                                 */
  double gamma;                        /* conservatism weight, >= 0 (1.0) */
  double c_floor;                      /* lower bound of c*, > 0                 */
} fp_estimator;

/* Raw request columns (all device memory, n_local entries each). */
typedef struct fp_raw_trace {
  const uint32_t *body_bytes;          /* |r|                                     */
  const uint32_t *max_output_tokens;   /* r.max_output_tokens (L_out)             */
  const uint8_t *category;             /* k                                       */
  const uint32_t *true_prompt_tokens;  /* usage.prompt_tokens, nullable (only
                                          route_batch_raw reads it)               */
} fp_raw_trace;

/* sweep_thresholds on L_total estimated in the trace pass itself (9 B per
 * request read; no L_total column is materialised). Same outputs, errors
 * and collective semantics as sweep_thresholds; columns must be device
 * memory (else FP_ERR_INVALID_ARG). */
fp_status sweep_thresholds_raw(fp_plan *plan, const fp_raw_trace *trace, uint64_t n_local,
                               const fp_estimator *est, double rate_rps, fp_candidate *h_results,
                               void *stream);

/* route_batch on the estimated L_total. Optionally writes the estimates
 * (d_l_total, device) and, when true_prompt_tokens is given, Table 5's
 * mis-route counts into h_misroute[2]: requests routed to the
 * short (long) pool whose TRUE total true_prompt_tokens + max_output_tokens
 * exceeds C_S (C_L). Global over ranks; synchronizes if h_counts or
 * h_misroute is non-NULL. */
fp_status route_batch_raw(fp_plan *plan, const fp_raw_trace *trace, uint64_t n_local,
                          const fp_estimator *est, uint32_t b_short, uint32_t c_short, uint32_t c_long,
                          uint8_t *d_decision, uint32_t *d_l_total, fp_route_counts *h_counts,
                          uint64_t *h_misroute, void *stream);

/* The whole workflow on raw columns: sweep_thresholds_raw, best_split (into
 * h_best if non-NULL), then route_batch_raw's decisions for model
 * route_model's best split into d_decision (device; no L_total output, no
 * mis-route counts), the split's global counts into h_counts. With
 * FP_FLAG_SPECULATE and the columns in one 16-B phase (category 4-B aligned
 * at the first vector element), d_decision in that element's 4-B phase, a u8
 * LUT with |E| < 127 and >= 2^26 requests on the rank: the speculative form
 * (sample pass, decision bytes written by the full raw trace pass, verify /
 * re-route from the estimated L_total) -- 9 B read + 1 B written per request
 * instead of sweep_thresholds_raw's 9 B plus route_batch_raw's 13 B + 1 B;
 * stream-ordered and asynchronous when h_best and h_counts are NULL. Otherwise
 * the three calls in sequence (synchronising). Same results either way.
 * Errors: as the three calls; FP_ERR_STATE if route_model has no feasible
 * split (the non-speculative form; the speculative one leaves d_decision
 * unspecified then, like sweep_and_route). */
fp_status sweep_and_route_raw(fp_plan *plan, const fp_raw_trace *trace, uint64_t n_local,
                              const fp_estimator *est, double rate_rps, uint32_t route_model,
                              uint8_t *d_decision, fp_candidate *h_best, fp_route_counts *h_counts,
                              void *stream);

/* ---- NEXT-2: three pools ---------------------------------------
 * Pools 1, 2, 3 with windows C1 = B1 < C2 = B2 <= C3 = C_L from the B and C_L
 * grids (pairs i < j of B-grid indices). A request goes to the first pool
 * whose threshold it meets (L <= B1, else L <= B2, else L <= C_L), otherwise
 * it is rejected (R3); each pool is sized with the Sec. 3 formulas. Flat
 * index ((m * n_gpus + g) * n_cl + l) * n_pairs + p, pairs in lexicographic
 * (i, j) order, n_pairs = n_b (n_b - 1) / 2. 160 bytes. */
typedef struct fp_pool3_candidate {
  uint32_t index, model, gpu, b1, b2, c_long, flags, _pad;
  uint64_t n1, n2, n3, n_reject;           /* routed requests per pool (global)    */
  uint64_t nseq1, nseq2, nseq3;            /* Eq. (2) N_seq at C1, C2, C3           */
  uint64_t inst1, inst2, inst3, inst_homo; /* ceil(lambda_i / mu(C_i))              */
  uint64_t gpus, gpus_homo;
  double cost, cost_homo, savings;         /* savings vs homogeneous C_H = C_L      */
} fp_pool3_candidate;

/* Evaluate every three-pool candidate over the histogram of the LAST
 * sweep_thresholds / sweep_and_route call (global over ranks; every rank
 * evaluates the whole three-pool grid, no further collective). h_results
 * (nullable) receives all candidates; h_best[n_models] the per-model cheapest
 * feasible one (index UINT32_MAX if none). Synchronizes. Every B must be in
 * desc->windows and 2 <= n_b <= 4096 (else FP_ERR_CONFIG); FP_ERR_STATE
 * before a sweep. */
fp_status sweep_three_pools(fp_plan *plan, double rate_rps, fp_pool3_candidate *h_results,
                            fp_pool3_candidate *h_best, void *stream);

/* ---- NEXT-3: calibration replay (Alg. 1 OnResponse) ---------------
 * Replays a feedback stream in arrival order (device columns: body bytes
 * |r|, usage.prompt_tokens, category) through the per-category EMA of Eq.
 * `ema`: c_obs = |r| / prompt_tokens; c_hat <- beta c_hat +
 * (1 - beta) c_obs; sigma_hat <- beta sigma_hat + (1 - beta) |c_obs -
 * c_hat(before)| (R26). prompt_tokens == 0 is discarded; category >=
 * n_cats counts as the last (R23). Starting from init[k], writes the final
 * state h_final[k], the number of observations h_n_obs[k], and (nullable)
 * the state right after the snap_at-th observation of each category into
 * h_snap[k] (NaN if the category has fewer). Computed as a parallel scan of
 * affine maps: equal to the sequential replay up to fp64 reassociation.
 * world > 1: the stream is sharded in order (rank r holds the r-th piece,
 * n may be 0); ranks all-gather their composed maps (three small exchanges)
 * and every rank returns the state of the WHOLE stream. 1 <= n_cats <= 16,
 * 0 < beta < 1.
 * Synchronizes. The result is the fp_category_calibration snapshot that
 * sweep_thresholds_raw / route_batch_raw consume. */
fp_status calibrate_replay(fp_plan *plan, const uint32_t *d_body_bytes, const uint32_t *d_prompt_tokens,
                           const uint8_t *d_category, uint64_t n, uint32_t n_cats, double beta,
                           const fp_category_calibration *init, uint64_t snap_at,
                           fp_category_calibration *h_final, uint64_t *h_n_obs,
                           fp_category_calibration *h_snap, void *stream);

/* ---- NEXT-4: peak-window provisioning -----------------
 * Requests carry arrival times (ns, non-decreasing, device u64[n]). The trace
 * is cut into windows w = floor(arrival / window_ns); for every candidate of
 * the plan's grid each pool is sized for its busiest window instead of the
 * mean rate: lambda_p = max_w n_p(w) * (1e9 / window_ns) requests/s, then
 * I_p = ceil(lambda_p / mu_p) as in Sec. 3 (R27). Same flat index as
 * fp_candidate. 144 bytes. */
typedef struct fp_peak_candidate {
  uint32_t index, model, gpu, b_short, c_short, c_long, flags, _pad;
  uint64_t peak_short, peak_long, peak_homo;         /* requests in the busiest window */
  uint64_t inst_short, inst_long, inst_homo, gpus_dual, gpus_homo;
  double lambda_short, lambda_long, lambda_homo;     /* peak rates, requests/s          */
  double cost_dual, cost_homo, savings;
} fp_peak_candidate;

/* Peak-window sweep over d_len / d_arrival_ns (device, n_local each; the
 * whole trace < 2^32 requests). world > 1: each rank holds a shard (any
 * split, n_local may be 0); ranks agree on the window range (all-gather) and
 * sum their window x bin histograms (all-reduce), then every rank evaluates
 * the whole grid. Precondition: arrivals non-decreasing (a trace is in
 * arrival order) -- the requests of a window are then one contiguous
 * index range, which the kernels exploit; the first/last arrivals are always
 * checked, the whole column only with FP_FLAG_CHECK_ORDER (otherwise an
 * unsorted column gives unspecified, but memory-safe, results). h_results
 * (nullable) receives every candidate, h_best[n_models] the per-model
 * cheapest feasible one. Synchronizes. Errors: FP_ERR_EMPTY_TRACE
 * (n_local == 0), FP_ERR_INVALID_ARG (window_ns == 0, host or misaligned
 * pointers, n_local >= 2^32, more than 2^26 windows, arrivals found out of
 * order), FP_ERR_CONFIG (grid too large for shared memory), FP_ERR_OOM. */
fp_status sweep_peak_windows(fp_plan *plan, const uint32_t *d_len, const uint64_t *d_arrival_ns,
                             uint64_t n_local, uint64_t window_ns, fp_peak_candidate *h_results,
                             fp_peak_candidate *h_best, void *stream);

/* Global per-bin histogram of the last sweep (K1 output after the cross-rank
 * sum; synchronizes). With E = sortuniq(B u C_L) ascending (|E| = n_edges of
 * fleet_plan_info): h_edges[j] = e_j for j < |E|; bin j < |E| holds the
 * requests with e_{j-1} < L <= e_j (e_{-1} = -inf) and bin |E| those above
 * every edge. h_bin_cnt[j] = requests in bin j; h_bin_mass[j] = sum of their
 * L (0 for bin |E|, whose mass no candidate uses; also 0 with
 * FP_FLAG_NO_MASS). Any pointer may be NULL. */
fp_status sweep_histogram(fp_plan *plan, uint32_t *h_edges, uint64_t *h_bin_cnt, uint64_t *h_bin_mass);

/* Writes a fresh 128-byte ncclUniqueId (for rank 0 to broadcast before
 * fleet_plan_create with world > 1). FP_ERR_NCCL if NCCL cannot be loaded. */
fp_status fp_nccl_get_unique_id(void *out128);

/* FP_FLAG_P2P: the 64-byte CUDA IPC handle of this rank's exchange buffer
 * (K1 accumulators, two step parities, and the rank's arrival flag).
 * Every rank all-gathers the handles (any host transport) and passes the
 * [world][64] array, in rank order, to fp_p2p_import, which opens the peers'
 * buffers (cudaIpcOpenMemHandle; NVLink peer access on an 8-GPU box; also
 * works for processes sharing one device). FP_ERR_STATE without FP_P2P or on
 * a second import; FP_ERR_CUDA if a handle cannot be opened. A sweep on a
 * FP_P2P plan before the import fails with FP_ERR_STATE. */
#define FP_P2P_HANDLE_BYTES 64
fp_status fp_p2p_export(fp_plan *plan, void *handle_out);
fp_status fp_p2p_import(fp_plan *plan, const void *handles);
/* Teardown of a FP_P2P plan: a peer's K3 may still be reading this rank's
 * exchange buffer after this rank's last sweep returns. All ranks must
 * synchronise (e.g. a barrier after best_split) before any of them calls
 * fleet_plan_destroy, which frees the exported buffer. */

fp_status fleet_plan_info(const fp_plan *plan, fp_plan_info *out);

/* Number of kernels this library launched on the plan since creation. */
uint64_t fp_kernel_launches(const fp_plan *plan);

/* Kernel kinds for fp_kernel_time. */
#define FP_KERNEL_TRACE 0 /* K1: sweep trace pass (one launch per chunk)   */
#define FP_KERNEL_EVAL 1  /* K3: scan + candidate evaluation + argmin      */
#define FP_KERNEL_ROUTE 2 /* K4: route_batch                               */

/* With FP_FLAG_KERNEL_TIMING (every kind) or FP_FLAG_TIME_TRACE (FP_KERNEL_TRACE
 * only): total device time (ms, CUDA events recorded on the launch stream
 * around each launch) and launch count of kernel `kind` since the last
 * fp_kernel_time_reset (or creation). Synchronizes those events. The plan
 * keeps at most 256 event pairs per kind: older launches are folded into the
 * running total as new ones are recorded (bounded memory in long-running
 * processes). FP_ERR_STATE when the kind is not timed by the plan's flags. */
fp_status fp_kernel_time(fp_plan *plan, int32_t kind, double *total_ms, uint64_t *launches);
fp_status fp_kernel_time_reset(fp_plan *plan);

void fleet_plan_destroy(fp_plan *plan);

const char *fp_status_string(fp_status s);
const char *fp_last_error(const fp_plan *plan);

/* ---- host-side partition helpers (no device work; used by the library and
 * by multi-rank tests) -------------------------------------------------------- */

/* Contiguous shard of a global trace for `rank`: [*first, *first + *count),
 * boundaries rounded to 32 requests (128 B). */
void fp_shard_range(uint64_t n_total, int32_t rank, int32_t world, uint64_t *first,
                    uint64_t *count);

/* Contiguous slice of the candidate grid for `rank` (same rule, unrounded). */
void fp_candidate_range(uint64_t n_candidates, int32_t rank, int32_t world, uint64_t *first,
                        uint64_t *count);

/* Deterministic merge of per-rank bests: recs[r * n_models + m] is rank r's
 * best for model m; writes out[m] = the record with the smallest cost_dual
 * among feasible ones, ties to the lowest index. */
void fp_merge_best(const fp_candidate *recs, int32_t world, uint32_t n_models, fp_candidate *out);

#ifdef __cplusplus
}
#endif
#endif /* FLEET_PLAN_H */
