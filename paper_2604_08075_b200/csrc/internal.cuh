// Internal declarations shared by the library's translation units (not part of
// the ABI). See include/fleet_plan.h for the public contract and DESIGN.md §5
// for the kernels.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include "fleet_plan.h"

namespace fp {

// programmatic dependent launch: the kernel may start while the previous
// kernel in the stream drains; it must execute griddepcontrol.wait before
// touching that kernel's outputs. FP_NO_PDL=1 falls back to plain launches.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("FP_NO_PDL");
    return !(v && v[0] == '1');
  }();
  return on;
}

template <typename... Params, typename... Args>
cudaError_t launch_pdl(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int kMaxEdges = 4096;          // |E| limit (K3 scans |E|+1 bins in smem)
constexpr int kLutMaxCells = 16384;      // above this: binary search over E

// ---- K1: trace pass (route every request against every edge + histogram) ----
struct TraceArgs {
  const uint32_t *len;      // device, this chunk
  uint64_t n;               // elements in this chunk
  const void *lut;          // device: u8 or u16 [lut_cells] bin of each fine cell
  const uint32_t *edges;    // device: E ascending [n_edges] (binary-search mode)
  uint32_t lut_cells;       // 0 => binary search mode
  uint32_t lut_u8;          // LUT element width
  uint32_t shift;           // s
  uint32_t n_edges;         // |E|
  uint32_t max_edge;        // e_max (mass is accumulated only for L <= e_max)
  uint32_t flush_iters;     // lane-slot mass flush period (iterations), >= 1
  uint32_t want_mass;
  unsigned long long *g_cnt;   // copy 0 of the global accumulators: [copies][2][n_edges + 1] (cnt, mass)
  unsigned long long *g_mass;  // = g_cnt + n_edges + 1
  uint32_t hist_copies = 1;    // block b adds into copy b % hist_copies (spreads same-address atomics)
  // raw columns (NEXT-1; body != nullptr selects them instead of len)
  const uint32_t *body = nullptr;   // |r| bytes
  const uint32_t *maxout = nullptr; // max_output_tokens
  const uint8_t *cat = nullptr;     // category
  const double *calib = nullptr;    // device [n_cats][2] (c_hat, sigma_hat)
  uint32_t n_cats = 0;
  uint32_t raw_vec = 0;             // set by launch_trace
  double gamma = 1.0, c_floor = 0.5;
  // per-request bin output (sweep_and_route's bin pass), nullable
  uint8_t *bins_out = nullptr;
  // bins_pack: |E| + 1 <= 64 bins fit 6 bits. Packed per (step k, thread t)
  // of the trace pass -- its 4 uint4 j = 4 k S + u S + t (u < 4, S = grid x
  // block threads) = 16 requests -- into chunk c = k S + t: a u64 of low
  // nibbles in bins_out (bin 4u + e at bits 16u + 4e) and a u32 of high 2-bit
  // parts in bins_hi (at bits 8u + 2e). One 8-B and one 4-B coalesced store
  // per 16 requests. The < 4 head / < 4 tail elements' bins go to
  // bins_side[0..3) / [4..7) as bytes. Device traces of one launch only.
  uint32_t bins_pack = 0;
  uint8_t *bins_hi = nullptr;
  uint8_t *bins_side = nullptr;
  // speculative routing (FP_FLAG_SPECULATE, sweep_and_route):
  //  step_stride > 1: a SAMPLE pass -- only the grid steps k = 0, stride, 2 stride, ...
  //    (whole grid-wide stripes spread over the trace), no head / tail elements
  //  dec_route != NULL (byte bin variant): bins_out receives DECISION bytes
  //    (SWAR on the bins for a u8 LUT, |E| < 127; for a u16 LUT from L_total
  //    and the split's edge values) for the split {iB, iCS, iCL, ok} at dec_route (read after
  //    griddepcontrol.wait; ok == 0: nothing is written), pdl: launch as a
  //    programmatic dependent of the previous kernel
  uint32_t step_stride = 1;
  const uint32_t *dec_route = nullptr;
  uint32_t pdl = 0;
};
cudaError_t launch_trace(const TraceArgs &a, int grid, int block, size_t smem, cudaStream_t s);
// the grid launch_trace uses for `a` (the bin/raw variants are clamped to the resident grid)
int trace_grid(const TraceArgs &a, int grid, int block);
size_t trace_smem_bytes(const TraceArgs &a, int block);
cudaError_t trace_occupancy(const TraceArgs &a, int block, size_t smem, int *per_sm);

// ---- K4: route_batch --------------------------------------------------------
struct RouteArgs {
  const uint32_t *len;
  uint8_t *decision;          // nullable
  uint64_t n;
  uint32_t b, cs, cl;
  unsigned long long *g_counts;  // [5]
};
cudaError_t launch_route(const RouteArgs &a, int grid, int block, cudaStream_t s);

// K4r: route_batch_raw (NEXT-1): Alg. 1 on estimated L_total + mis-route counts
struct RouteRawArgs {
  const uint32_t *body, *maxout;
  const uint8_t *cat;
  const uint32_t *true_prompt;      // nullable
  const double *calib;              // device [n_cats][2]
  uint32_t n_cats;
  double gamma, c_floor;
  uint8_t *decision;                // nullable
  uint32_t *l_total;                // nullable: estimated L_total out
  uint64_t n;
  uint32_t b, cs, cl;
  unsigned long long *g_counts;     // [5]
  unsigned long long *g_mis;        // [2] short, long
};
cudaError_t launch_route_raw(const RouteRawArgs &a, int grid, int block, cudaStream_t s);

// K4b: decisions from per-request bins (sweep_and_route): with iB, iCS, iCL
// the indices in E of B, C_S, C_L, L <= e_j <=> bin <= j. With n_edges >= 255
// the bins are clamped bytes and len (the device trace, element i = bin i) is
// read back for byte 255 when the split has an edge index >= 255.
cudaError_t launch_route_bins(const uint8_t *bins, uint8_t *decision, uint64_t n, const fp_candidate *recs,
                              int ranks, uint32_t n_models, uint32_t model, const uint32_t *edges, uint32_t n_edges,
                              uint32_t *route, int grid, int block, cudaStream_t s, const uint32_t *len);
// K4p: the same from K1's 6-bit packed bins (TraceArgs::bins_pack), launched
// with the trace pass's grid x block (k1_grid x k1_block) so thread t reads
// the chunks it wrote
cudaError_t launch_route_packed(const uint8_t *lo, const uint8_t *hi, const uint8_t *side, uint32_t head,
                                uint8_t *decision, uint64_t n, const fp_candidate *recs, int ranks, uint32_t n_models,
                                uint32_t model, const uint32_t *edges, uint32_t n_edges, uint32_t *route, int k1_grid,
                                int k1_block, cudaStream_t s);
cudaError_t route_occupancy(int block, int *per_sm);
// FP_FLAG_SPECULATE: after the full K3 -- if the final split (route) differs
// from the speculated one (spec), every decision byte is recomputed from
// L_total (device trace len, decision[i] <-> len[i]) with the final split.
// the same for raw columns (sweep_and_route_raw): a.decision, a.n, the columns
// and the estimator fields of `a` are used
cudaError_t launch_route_verify_raw(const RouteRawArgs &a, const uint32_t *spec, const uint32_t *route,
                                    const uint32_t *edges, unsigned int *misses, int grid, int block, cudaStream_t s);
// the routed split {iB, iCS, iCL, ok} from the ranks' gathered best records (sliced grid)
cudaError_t launch_pick_route(const fp_candidate *recs, int ranks, uint32_t n_models, uint32_t model,
                              const uint32_t *edges, uint32_t n_edges, uint32_t *route, cudaStream_t s);
cudaError_t launch_route_verify(const uint32_t *len, uint8_t *decision, uint64_t n, const uint32_t *spec,
                                const uint32_t *route, const uint32_t *edges, unsigned int *misses, int grid,
                                int block, cudaStream_t s);

// ---- K3: candidate evaluation + argmin ---------------------------------------
struct BlockBest { double cost; uint32_t index; uint32_t valid; };

struct EvalArgs {
  const unsigned long long *hist_cnt;   // [copies][2][nbins] per-bin counts (global, all ranks), copy 0
  const unsigned long long *hist_mass;  // = hist_cnt + nbins
  uint32_t hist_copies = 1;             // K3 sums the copies (K1's spread atomics)
  // FP_FLAG_P2P: the histogram is the sum over ranks r of peer_hist[r] + p2p_off
  // (each rank's K1 copies, this step's parity), read once every peer_flag[r]
  // has reached p2p_epoch (no all-reduce)
  const unsigned long long *const *peer_hist = nullptr;
  const unsigned int *const *peer_flag = nullptr;
  uint32_t p2p_world = 0, p2p_epoch = 0;
  uint64_t p2p_off = 0;                 // u64 elements: parity * copies * 2 * nbins
  unsigned long long *hist_out = nullptr;  // [2][nbins] the summed histogram (written by one block)
  uint32_t nbins;                       // |E| + 1
  const uint32_t *b, *cs, *cl;          // grid values
  const uint16_t *b_edge, *cl_edge;     // index in E of each B / C_L
  const uint16_t *cs_edge = nullptr;    // index in E of each C_S
  const uint16_t *b_win, *cs_win, *cl_win;  // index in windows of each B / C_S / C_L
  uint32_t n_b, n_cs, n_cl, n_cs_eff;
  uint32_t fac_lc = 16;                 // k3_factored: C_L values per block (<= 64)
  // exact 32-bit division by n_b, n_cs_eff, n_cl, n_gpus: q = umul64hi(x, mul) (mul = ceil(2^64 / d), 0 for d = 1)
  unsigned long long div_b = 0, div_cs = 0, div_cl = 0, div_g = 0;
  uint32_t n_models, n_gpus, n_windows;
  const uint32_t *model_arch;           // [m][4] n_l, n_h, d_h, b
  const unsigned long long *gpu_u64;    // [g][4] hbm, u_num, u_den, act
  const double *price;                  // [g]
  const unsigned long long *deploy;     // [m][g][3] tp, gpus_per_instance, weights
  const uint32_t *windows;              // [n_windows]
  const double *mu;                     // [m][g][w]
  const unsigned long long *cap_nseq = nullptr;  // [m][g][w] N_seq (Eq. 2), computed once per plan
  const double *rmu = nullptr;          // [m][g][w] RN(1/mu) (0 outside mdiv's range), once per plan
  unsigned int *err_word = nullptr;     // device error word (P2P wait timed out: 1 | peer << 8)
  unsigned long long p2p_timeout_ns = 10000000000ull;
  unsigned long long *phase_ts = nullptr;  // diagnostic (env FP_K3_PHASES): %globaltimer at K3's phases
  double rate, hours;
  uint64_t per_model;                   // candidates per model
  uint64_t cand_first, cand_count;      // this rank's slice
  fp_candidate *results;                // nullable [cand_count]
  fp_candidate *best_out;               // [n_models] (this rank's)
  BlockBest *block_best;                // [n_models][grid_x]
  unsigned int *done;                   // [n_models] last-block-done counters (self-resetting)
  // non-null: the other parity's accumulator copies [copies][2][nbins], zeroed
  // by one block for the next sweep (its last reader, the previous sweep's K3
  // or fold kernel, completed before this sweep's plain-launched trace pass)
  unsigned long long *zero_copies = nullptr;
  size_t zero_elems = 0;                // u64 elements of zero_copies (every copy, whatever hist_copies says)
  unsigned long long *zero_copies2 = nullptr;   // FP_FLAG_SPECULATE: the sample's accumulators (zero_elems)
  // sweep_and_route (one rank's grid is the whole grid): the last block of
  // model route_model also writes {iB, iCS, iCL, ok} of its best split
  const uint32_t *edges = nullptr;
  uint32_t n_edges = 0, route_model = 0;
  uint32_t *route_out = nullptr;
  // NEXT-2 three pools (replicated grid): pairs (i | j << 16) of B-grid indices
  const uint32_t *pairs = nullptr;
  uint32_t n_pairs = 0;
  const uint16_t *b_win3 = nullptr;     // window index of each B
  uint64_t per_model3 = 0;
  fp_pool3_candidate *results3 = nullptr;
  fp_pool3_candidate *best3 = nullptr;  // [n_models]
  BlockBest *block_best3 = nullptr;
  unsigned int *done3 = nullptr;
  // NEXT-4 peak windows: cumulative per-window counts [n_windows][nbins]
  const uint32_t *colmax_pk = nullptr;  // NEXT-4 per-bin / per-(B, C_L) window maxima
  const uint32_t *pairmax_pk = nullptr;
  double inv_w_s = 0.0;                 // windows per second = 1e9 / window_ns
  fp_peak_candidate *results_pk = nullptr;
  fp_peak_candidate *best_pk = nullptr;
  BlockBest *block_best_pk = nullptr;
  unsigned int *done_pk = nullptr;
};
// K3 launch shape (chosen once per plan)
enum { kK3Cluster = 0, kK3Factored = 1, kK3Grid = 2 };
struct EvalLaunch {
  int shape = kK3Grid;
  int grid_x = 1, block = 256;   // blocks per model (cluster size for kK3Cluster)
  size_t smem = 0;
};
cudaError_t launch_eval(const EvalArgs &a, const EvalLaunch &L, cudaStream_t s);
// sum the trace pass's accumulator copies into one [2][nbins] histogram; with
// flag (FP_FLAG_P2P) also fence system-wide and publish `epoch` for the peers
cudaError_t launch_fold(const unsigned long long *copies, uint32_t n_copies, uint32_t nbins, unsigned long long *out,
                        unsigned int *flag, unsigned int epoch, cudaStream_t s);
// fills cap_nseq and rmu
cudaError_t launch_capacity(const EvalArgs &a, unsigned long long *cap, double *rmu, cudaStream_t s);
cudaError_t launch_eval3(const EvalArgs &a, int grid_x, int block, size_t smem, cudaStream_t s);
cudaError_t launch_eval_peak(const EvalArgs &a, int grid_x, int block, cudaStream_t s);
size_t eval_smem_bytes(const EvalArgs &a, int block);
size_t eval_factored_smem_bytes(const EvalArgs &a);
size_t eval_peak_smem_bytes(const EvalArgs &a);
uint32_t eval_factored_blocks_per_model(const EvalArgs &a);
int eval_max_cluster(int block, size_t smem);
cudaError_t eval_prepare();

// NEXT-4: peak-window provisioning (k_peak.cu + the k3 peak kernel)
struct PeakArgs {
  const uint32_t *len;
  const uint64_t *arrival;          // ns, non-decreasing
  uint64_t n;                       // < 2^32
  uint64_t window_ns;
  uint64_t n_windows;               // floor(arrival[n-1] / window_ns) + 1
  uint64_t *start;                  // [n_windows + 1]: first request of each window
  const void *lut;                  // as TraceArgs
  const uint32_t *edges;
  uint32_t lut_cells, lutw, clampv, round, shift, nbins;
  uint32_t *hist2d;                 // [n_windows][nbins] requests per (window, bin)
  const uint16_t *b_edge, *cl_edge; // index in E of each B / C_L
  uint32_t n_b, n_cl;
  uint32_t rows;                    // windows per K2w shared-memory chunk
  uint32_t *colmax;                 // [nbins]      max_w cnt_le[w][j]
  uint32_t *pairmax;                // [n_b * n_cl] max_w cnt_le[w][cl_edge[l]] - cnt_le[w][b_edge[k]]
  unsigned int *error;
  bool check_order;
};
size_t peak_smem_bytes(const PeakArgs &a);
size_t peak_scan_smem_bytes(const PeakArgs &a);
cudaError_t launch_peak_hist(const PeakArgs &a, int sm_count, cudaStream_t s);   // Kc?, K0w, K1w
cudaError_t launch_peak_scan(const PeakArgs &a, int sm_count, cudaStream_t s);   // K2w

// NEXT-3: calibration replay (k_calib.cu)
struct CalibArgs {
  const uint32_t *bytes, *tokens;
  const uint8_t *cat;
  uint64_t n;
  uint32_t n_cats;                  // <= 16
  double beta;
  const double *c0, *s0;            // device [n_cats] initial state
  uint64_t threads, blocks, seg;    // thread t owns [t*seg, (t+1)*seg); seg % 16 == 0; 256 threads / block
  double *thrA, *thrB;              // [n_cats][threads] within-block exclusive c_hat maps
  uint32_t *thrN;
  uint32_t *thrC;                   // [n_cats][threads] observations in each thread's own segment
  double *blkA, *blkB;              // [n_cats][blocks] c_hat block totals -> exclusive prefixes
  unsigned long long *blkN;
  double *sblkA, *sblkB;            // [n_cats][blocks] sigma block totals -> exclusive prefixes
  double *totA, *totSA;             // [n_cats] final c_hat / sigma
  unsigned long long *totN;         // [n_cats] observations
  double *mapA, *mapB;              // [n_cats] this stream's total c_hat map (world > 1 exchange)
  unsigned long long *mapN;
  double *smapA, *smapB;            // [n_cats] this stream's total sigma map
  unsigned long long snap_off[16];  // observations of each category on lower ranks
  uint64_t snap_at;
  double *snap_c, *snap_s;          // [n_cats]
  double *snap_sa, *snap_sb;        // [n_cats] sigma map from the snapshot's block start
  unsigned long long *snap_block;   // [n_cats] (~0: no snapshot)
  bool vec_bt, vec_c;               // 16-B aligned columns: vector loads
};
// one rank, n_cats <= 4: the streaming replay (k_calib.cu c_stream), every
// record read once; a persistent cooperative grid of G CTAs, chunks of G pieces
struct CalibStreamArgs {
  const uint32_t *bytes, *tokens;
  const uint8_t *cat;
  uint64_t n;
  uint32_t n_cats;                  // <= 4
  double beta;
  const double *c0, *s0;            // device [4] initial state
  uint32_t G, n_chunks;             // CTAs (<= 512), chunks of G pieces of calib_stream_piece() records
  unsigned int *done, *ready;       // [n_chunks] finished-A counters, [n_chunks + 1] chunk-start flags (zeroed)
  void *cagg;                       // [n_chunks][G][4] piece c_hat maps (k_calib.cu Aff, 24 B)
  double *pstate_c;                 // [n_chunks][G][4] c_hat at each piece's start
  unsigned long long *pstate_n;     // [n_chunks][G][4] observations before each piece
  double *cstart_c;                 // [n_chunks + 1][4] c_hat at each chunk's start (last: final)
  unsigned long long *cstart_n;     // [n_chunks + 1][4]
  double *sig_a, *sig_b;            // [n_chunks * G][4] piece sigma maps
  unsigned long long *snap_piece;   // [4] piece holding the snap_at-th observation (~0: none; preset)
  double *snap_v;                   // [4][4] sigma map piece start -> snapshot (a, b), snapshot c_hat
  void *fin_part, *fin_pre;         // c_stream_final: [4][fin_blocks] range maps, [4] snapshot range prefix (Aff)
  unsigned int *fin_done, *fin_snapb;   // [4] block counters (zeroed), [4] block holding the snapshot
  uint64_t snap_at;
  double *out;                      // [80]: c_hat[16], sigma[16], n_obs[16] (u64), snap_c[16], snap_s[16]
  unsigned long long *prof;         // FP_CALIB_PROFILE: [2 n_chunks + 2][8] phase stamps (nullptr: off)
};
size_t calib_stream_smem();
uint32_t calib_stream_piece();
uint32_t calib_stream_fin_blocks();
int calib_stream_blocks_per_sm();
cudaError_t launch_calib_stream(const CalibStreamArgs &a, cudaStream_t s);
size_t calib_scratch_bytes(uint64_t blocks, uint32_t n_cats);
int calib_blocks_per_sm(uint32_t n_cats);
cudaError_t launch_calibrate(CalibArgs a, cudaStream_t s);        // C1 C2 C3 C2 C4 (one rank)
cudaError_t launch_calib_maps(const CalibArgs &a, cudaStream_t s);   // C1 C2
cudaError_t launch_calib_replay(const CalibArgs &a, cudaStream_t s); // C3 C2
cudaError_t launch_calib_snap(const CalibArgs &a, cudaStream_t s);   // C4

}  // namespace fp
