// Plan runtime and C ABI (include/fleet_plan.h).
//
// fleet_plan_create validates the descriptor, builds the routing edge set
// E = sortuniq(B u C_L) and its fine-cell bin LUT, copies
// every table to one device blob, and (world > 1) initialises NCCL from the
// caller's unique id (NCCL is dlopen'ed: single-GPU plans never touch it).
// The compute entry points enqueue the kernels of k_trace.cu / k_eval.cu on
// the caller's stream; host-resident traces are streamed through two
// plan-owned device staging buffers on a copy stream, overlapping the
// host-to-device DMA of chunk i+1 with the trace pass over chunk i.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

using namespace fp;

// ---- minimal NCCL surface (types per nccl.h; functions resolved at runtime) ----
namespace {
typedef struct { char internal[128]; } NcclUniqueId;
typedef void *NcclComm;
enum { kNcclUint8 = 1, kNcclUint32 = 3, kNcclUint64 = 5 };
enum { kNcclSum = 0 };
struct NcclApi {
  void *h = nullptr;
  int (*GetUniqueId)(NcclUniqueId *) = nullptr;
  int (*CommInitRank)(NcclComm *, int, NcclUniqueId, int) = nullptr;
  int (*AllReduce)(const void *, void *, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*AllGather)(const void *, void *, size_t, int, NcclComm, cudaStream_t) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  const char *(*GetErrorString)(int) = nullptr;
  int (*CommCount)(NcclComm, int *) = nullptr;
  int (*CommGetAsyncError)(NcclComm, int *) = nullptr;
};

bool load_nccl(NcclApi &api, std::string &err) {
  if (api.h) return true;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *n : names) {
    api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) { err = std::string("dlopen libnccl failed: ") + dlerror(); return false; }
#define FP_SYM(field, name)                                                   \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, name));     \
  if (!api.field) { err = "missing NCCL symbol " name; return false; }
  FP_SYM(GetUniqueId, "ncclGetUniqueId");
  FP_SYM(CommInitRank, "ncclCommInitRank");
  FP_SYM(AllReduce, "ncclAllReduce");
  FP_SYM(AllGather, "ncclAllGather");
  FP_SYM(CommDestroy, "ncclCommDestroy");
  FP_SYM(GetErrorString, "ncclGetErrorString");
  FP_SYM(CommCount, "ncclCommCount");
  FP_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef FP_SYM
  return true;
}
NcclApi g_nccl;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

constexpr uint64_t kChunkElems = 32ull << 20;  // host streaming: 128 MB per chunk
}  // namespace

struct fp_plan {
  // descriptor copy
  std::vector<fp_model> models;
  std::vector<fp_gpu> gpus;
  std::vector<fp_deploy> deploy;
  std::vector<uint32_t> b, cs, cl, windows;
  std::vector<double> mu;
  double hours = 8760.0;
  uint32_t flags = 0;
  int device = 0, rank = 0, world = 1;
  bool dist = false;                       // cross-rank steps run (world > 1 or FP_FLAG_COLLECTIVES)
  // derived
  std::vector<uint32_t> edges;
  uint32_t shift = 0, lut_cells = 0, lut_u8 = 0, max_edge = 0, nbins = 0;
  uint64_t n_cand = 0, per_model = 0, cand_first = 0, cand_count = 0;
  uint32_t n_cs_eff = 1;
  int sm_count = 148, k1_grid = 0, k1_block = 512, k4_grid = 0, k4_block = 256;
  size_t k1_smem = 0, k3_smem = 0;
  // device
  unsigned char *d_blob = nullptr;
  size_t blob_bytes = 0;
  TraceArgs ta{};
  EvalArgs ea{};
  unsigned long long *d_hist = nullptr;    // [2][nbins] summed histogram (written by K3)
  // K1's accumulators [2 parities][hist_copies][2][nbins]: sweep number q uses
  // parity q & 1, and its K3 zeroes the other parity for sweep q + 1
  unsigned long long *d_hcopies = nullptr;
  uint32_t hist_copies = 1;
  size_t copies_elems = 0;                  // u64 elements per parity
  uint64_t sweep_seq = 0;
  bool parity_clean[2] = {true, true};      // that parity's copies are zero (stream-ordered)
  unsigned long long *d_fold = nullptr;     // dist (NCCL / hooks): [2][nbins] folded histogram, all-reduced
  // FP_FLAG_SPECULATE: the sample's accumulator copies (zeroed by the full K3),
  // its best records, its split {iB, iCS, iCL, ok} and a miss counter
  unsigned char *d_spec = nullptr;
  unsigned long long *spec_acc = nullptr;
  fp_candidate *spec_best = nullptr;
  uint32_t *spec_route = nullptr;
  unsigned int *spec_miss = nullptr;
  uint64_t spec_calls = 0;
  // sweep_and_route_graph: the captured step per accumulator parity, its key
  // and the scratch it was captured against
  struct StepGraph {
    bool valid = false;
    const uint32_t *len = nullptr;
    uint64_t n = 0;
    double rate = 0.0;
    uint32_t model = 0;
    uint8_t *dec = nullptr;
    const void *bins = nullptr, *spec_buf = nullptr;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    uint64_t launches[2] = {0, 0}, spec_n[2] = {0, 0};
  } graph;
  cudaStream_t graph_stream = nullptr;
  bool spec_dirty = false;                  // a speculative call failed before its full K3 (which zeroes spec_acc)
  // FP_FLAG_P2P: exchange buffer [2 parities][2][nbins] u64 (each rank's folded
  // histogram) + the arrival flag, the peers' buffers opened by CUDA IPC, and
  // device tables of their addresses
  unsigned long long *d_xbuf = nullptr;
  unsigned int *d_xflag = nullptr;
  size_t xbuf_elems = 0;                    // u64 elements per parity
  std::vector<void *> peer_open;            // opened IPC mappings (closed at destroy)
  unsigned long long **d_peer_hist = nullptr;
  unsigned int **d_peer_flag = nullptr;
  bool p2p_ready = false;
  uint32_t p2p_epoch = 0;
  unsigned long long *d_rcounts = nullptr; // [8]: route counts [5], mis-routes [2] (or the picked split)
  unsigned long long *d_cap = nullptr;     // [M][G][W] N_seq
  double *d_rmu = nullptr;                 // [M][G][W] RN(1/mu)
  unsigned int *d_err = nullptr;           // device error word (P2P wait timeout)
  double *d_calib = nullptr;               // [256][2] estimator snapshot
  fp_candidate *d_best = nullptr;          // [world][n_models]
  fp_candidate *d_results = nullptr;       // [cand_count] (lazy)
  BlockBest *d_block_best = nullptr;
  unsigned int *d_done = nullptr;
  unsigned long long *h_phase = nullptr;   // diagnostic K3 phase stamps (env FP_K3_PHASES, mapped host)
  double phase_sum[16] = {0};
  uint64_t phase_n = 0;
  EvalLaunch k3a;                          // K3 launch, argmin only (the step's)
  EvalLaunch k3r;                          // K3 launch with every record (want_results)
  int k3_grid_x = 1;                       // blocks per model of the grid-stride shape
  // host streaming
  uint32_t *d_stage[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  // pinned host mirrors
  fp_candidate *h_best = nullptr;          // [world][n_models]
  unsigned long long *h_small = nullptr;   // [2 * nbins + 8]: hist, route counts
  // device copy of a host trace / per-request bins for sweep_and_route
  uint32_t *d_resident = nullptr;
  uint64_t resident_cap = 0;
  uint8_t *d_bins = nullptr;
  uint64_t bins_cap = 0;
  // NEXT-2 three-pool state (lazy)
  unsigned char *d_p3 = nullptr;           // pairs, b_win3, best3, block_best3, done3
  fp_pool3_candidate *d_results3 = nullptr;
  EvalArgs ea3{};
  int k3p_grid_x = 1;
  uint64_t n_cand3 = 0;
  // NEXT-4 peak-window scratch (lazy)
  uint64_t *d_xch = nullptr;               // [world + 1][4] small all-gather exchange
  unsigned char *d_peak = nullptr;
  size_t peak_cap = 0;
  fp_peak_candidate *d_results_pk = nullptr;
  // NEXT-3 calibration scratch (lazy)
  unsigned char *d_calib_scratch = nullptr;
  size_t calib_cap = 0;
  // NCCL
  NcclComm comm = nullptr;
  fp_collectives coll{};                   // host hooks replacing NCCL (optional)
  bool has_coll = false;
  // per-kernel event timing (FP_FLAG_KERNEL_TIMING): a ring of event pairs;
  // the oldest pending pair is folded into the running total when the ring is
  // full, so a long-running process keeps a bounded number of events
  struct Timer {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;   // ring
    size_t head = 0, pending = 0;
    double total_ms = 0.0;
    uint64_t launches = 0;
  } timers[3];
  cudaEvent_t ev_order = nullptr;          // orders a call on another stream after the last sweep
  // state
  bool have_sweep = false;
  cudaStream_t last_stream = nullptr;
  uint64_t launches = 0;
  std::string err;
};

namespace {

fp_status fail(fp_plan *p, fp_status s, const char *fmt, ...) {
  if (p) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    p->err = buf;
  }
  return s;
}

fp_status cuda_fail(fp_plan *p, cudaError_t e, const char *what) {
  cudaGetLastError();
  return fail(p, e == cudaErrorMemoryAllocation ? FP_ERR_OOM : FP_ERR_CUDA, "%s: %s", what,
              cudaGetErrorString(e));
}

#define CUDA_TRY(p, expr, what)                              \
  do {                                                       \
    cudaError_t e_ = (expr);                                 \
    if (e_ != cudaSuccess) return cuda_fail((p), e_, what);  \
  } while (0)

fp_status nccl_check(fp_plan *p, int r, const char *what) {
  // a communicator failure raised asynchronously (a peer died, a network
  // error) is reported by the next collective's check
  constexpr int kNcclInProgress = 7;
  if (r == 0 && p && p->comm && g_nccl.CommGetAsyncError) {
    int ae = 0;
    if (g_nccl.CommGetAsyncError(p->comm, &ae) == 0 && ae != 0 && ae != kNcclInProgress) r = ae;
  }
  if (r == 0) return FP_OK;
  return fail(p, FP_ERR_NCCL, "%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
}

uint32_t index_of(const std::vector<uint32_t> &v, uint32_t x) {
  auto it = std::lower_bound(v.begin(), v.end(), x);
  return (it != v.end() && *it == x) ? (uint32_t)(it - v.begin()) : UINT32_MAX;
}

bool is_host_pointer(const void *ptr) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

fp_status validate_and_copy(fp_plan *p, const fp_plan_desc *d) {
  if (d->abi_version != FP_ABI_VERSION)
    return fail(p, FP_ERR_CONFIG, "abi_version %u != %u", d->abi_version, FP_ABI_VERSION);
  if (!d->models || !d->gpus || !d->deploy || !d->windows || !d->mu_table || !d->grid.b_short ||
      !d->grid.c_long || (d->grid.n_cs && !d->grid.c_short))
    return fail(p, FP_ERR_INVALID_ARG, "NULL array in descriptor");
  if (d->n_models == 0 || d->n_gpus == 0 || d->grid.n_b == 0 || d->grid.n_cl == 0 || d->n_windows == 0)
    return fail(p, FP_ERR_CONFIG, "empty models/gpus/grid/windows");
  if (d->world < 1 || d->rank < 0 || d->rank >= d->world)
    return fail(p, FP_ERR_CONFIG, "rank %d world %d", d->rank, d->world);
  if ((d->world > 1 || (d->flags & FP_FLAG_COLLECTIVES)) && !d->nccl_unique_id && !d->collectives)
    return fail(p, FP_ERR_CONFIG, "world > 1 (or FP_FLAG_COLLECTIVES) needs nccl_unique_id or collectives");
  if (d->collectives && (!d->collectives->allreduce_sum_u64 || !d->collectives->allgather_bytes))
    return fail(p, FP_ERR_CONFIG, "collectives hooks must both be set");
  if (d->collectives) {
    p->coll = *d->collectives;
    p->has_coll = true;
  }
  if (!(d->hours_per_year > 0.0) || !std::isfinite(d->hours_per_year))
    return fail(p, FP_ERR_CONFIG, "hours_per_year must be finite and > 0");
  p->models.assign(d->models, d->models + d->n_models);
  p->gpus.assign(d->gpus, d->gpus + d->n_gpus);
  p->deploy.assign(d->deploy, d->deploy + (size_t)d->n_models * d->n_gpus);
  p->b.assign(d->grid.b_short, d->grid.b_short + d->grid.n_b);
  if (d->grid.n_cs) p->cs.assign(d->grid.c_short, d->grid.c_short + d->grid.n_cs);
  p->cl.assign(d->grid.c_long, d->grid.c_long + d->grid.n_cl);
  p->windows.assign(d->windows, d->windows + d->n_windows);
  p->mu.assign(d->mu_table, d->mu_table + (size_t)d->n_models * d->n_gpus * d->n_windows);
  p->hours = d->hours_per_year;
  p->flags = d->flags;
  p->device = d->device;
  p->rank = d->rank;
  p->world = d->world;
  p->dist = d->world > 1 || (d->flags & FP_FLAG_COLLECTIVES);
  if (p->flags & FP_FLAG_P2P) {
    if (!p->dist) return fail(p, FP_ERR_CONFIG, "FP_FLAG_P2P needs world > 1 or FP_FLAG_COLLECTIVES");
    if (d->world > 64) return fail(p, FP_ERR_CONFIG, "FP_FLAG_P2P: world > 64");
    p->flags |= FP_FLAG_REPLICATED_GRID;   // every rank sums all ranks' histograms: no all-gather
  }

  for (auto &m : p->models) {
    if (!m.n_layers || !m.n_kv_heads || !m.head_dim ||
        !(m.kv_elem_bytes == 1 || m.kv_elem_bytes == 2 || m.kv_elem_bytes == 4))
      return fail(p, FP_ERR_CONFIG, "model %.32s: counts must be >= 1 and b in {1,2,4}", m.name);
  }
  for (auto &g : p->gpus) {
    if (g.hbm_bytes == 0 || g.hbm_bytes >= (1ull << 50))
      return fail(p, FP_ERR_CONFIG, "gpu %.32s: hbm_bytes must be in [1, 2^50)", g.name);
    if (g.util_num == 0 || g.util_den == 0 || g.util_num > g.util_den || g.util_den > 8192)
      return fail(p, FP_ERR_CONFIG, "gpu %.32s: need 0 < util_num <= util_den <= 8192", g.name);
    if (!(g.price_per_gpu_hour >= 0.0) || !std::isfinite(g.price_per_gpu_hour))
      return fail(p, FP_ERR_CONFIG, "gpu %.32s: price must be finite and >= 0", g.name);
  }
  for (auto &dp : p->deploy) {
    if (dp.tp_degree < 1 || dp.tp_degree > 8192)
      return fail(p, FP_ERR_CONFIG, "tp_degree must be in [1, 8192]");
    if (dp.gpus_per_instance < 1 || dp.gpus_per_instance > 512)
      return fail(p, FP_ERR_CONFIG, "gpus_per_instance must be in [1, 512]");
  }
  for (size_t i = 0; i < p->windows.size(); ++i)
    if (p->windows[i] == 0 || (i && p->windows[i] <= p->windows[i - 1]))
      return fail(p, FP_ERR_CONFIG, "windows must be >= 1 and strictly increasing");
  for (double v : p->mu)
    if (!(v >= 0.0) || !std::isfinite(v)) return fail(p, FP_ERR_CONFIG, "mu must be finite and >= 0");
  for (uint32_t v : p->b) if (!v) return fail(p, FP_ERR_CONFIG, "B_short values must be >= 1");
  for (uint32_t v : p->cs) if (!v) return fail(p, FP_ERR_CONFIG, "C_S values must be >= 1");
  for (uint32_t v : p->cl) if (!v) return fail(p, FP_ERR_CONFIG, "C_L values must be >= 1");
  // Eq. (1) products stay below 2^63 for every (model, window)
  for (auto &m : p->models) {
    unsigned __int128 per_tok = (unsigned __int128)2 * m.n_layers * m.n_kv_heads * m.head_dim * m.kv_elem_bytes;
    if (per_tok * p->windows.back() >= ((unsigned __int128)1 << 63))
      return fail(p, FP_ERR_CONFIG, "model %.32s: M_seq overflows 64 bits", m.name);
  }
  return FP_OK;
}

fp_status build_tables(fp_plan *p) {
  // edge set E = sortuniq(B u C_L): C_S never adds an edge since B <= C_S (R16)
  // E = sortuniq(B u C_S u C_L): B and C_L give every candidate's counts;
  // C_S (never needed for the counts since B <= C_S) is included so that every
  // comparison of Alg. 1 is a bin comparison (sweep_and_route's bin pass)
  p->edges = p->b;
  p->edges.insert(p->edges.end(), p->cl.begin(), p->cl.end());
  p->edges.insert(p->edges.end(), p->cs.begin(), p->cs.end());
  std::sort(p->edges.begin(), p->edges.end());
  p->edges.erase(std::unique(p->edges.begin(), p->edges.end()), p->edges.end());
  if (p->edges.size() > (size_t)kMaxEdges)
    return fail(p, FP_ERR_CONFIG, "|E| = %zu exceeds %d", p->edges.size(), kMaxEdges);
  p->nbins = (uint32_t)p->edges.size() + 1;
  p->max_edge = p->edges.back();
  // fine cells: s = largest k with 2^k | every edge; cell(L) = ceil(L / 2^s)
  uint32_t s = 31;
  for (uint32_t e : p->edges) s = std::min<uint32_t>(s, (uint32_t)__builtin_ctz(e));
  p->shift = s;
  uint64_t cell_max = p->max_edge >> s;
  // LUT mode needs a small table and e_max + 2^s < 2^32 (K1 computes
  // ceil(min(L, e_max + 1) / 2^s) in 32 bits); otherwise binary search over E
  const bool lut_ok = cell_max + 2 <= (uint64_t)kLutMaxCells &&
                      (uint64_t)p->max_edge + (1ull << s) <= 0xFFFFFFFFull;
  p->lut_cells = lut_ok ? (uint32_t)(cell_max + 2) : 0;
  p->lut_u8 = p->nbins <= 256;
  // window / edge index maps
  p->n_cs_eff = p->cs.empty() ? 1 : (uint32_t)p->cs.size();
  for (uint32_t v : p->b)
    if (p->cs.empty() && index_of(p->windows, v) == UINT32_MAX)
      return fail(p, FP_ERR_CONFIG, "window %u (B with n_cs = 0) missing from windows", v);
  for (uint32_t v : p->cs)
    if (index_of(p->windows, v) == UINT32_MAX) return fail(p, FP_ERR_CONFIG, "C_S %u missing from windows", v);
  for (uint32_t v : p->cl)
    if (index_of(p->windows, v) == UINT32_MAX) return fail(p, FP_ERR_CONFIG, "C_L %u missing from windows", v);
  p->per_model = (uint64_t)p->gpus.size() * p->cl.size() * p->n_cs_eff * p->b.size();
  p->n_cand = p->per_model * p->models.size();
  if (p->n_cand >= 0xffffffffull) return fail(p, FP_ERR_CONFIG, "grid has >= 2^32 - 1 candidates");
  if (p->flags & FP_FLAG_REPLICATED_GRID || !p->dist) {
    p->cand_first = 0;
    p->cand_count = p->n_cand;
  } else {
    fp_candidate_range(p->n_cand, p->rank, p->world, &p->cand_first, &p->cand_count);
  }
  return FP_OK;
}

int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// Copy every table into one device blob and fill ta / ea pointers.
fp_status upload(fp_plan *p) {
  const uint32_t G = (uint32_t)p->gpus.size(), M = (uint32_t)p->models.size();
  const uint32_t W = (uint32_t)p->windows.size();
  std::vector<unsigned char> blob;
  auto put = [&](const void *src, size_t bytes) {
    size_t off = (blob.size() + 15) & ~size_t(15);
    blob.resize(off + bytes);
    if (bytes) memcpy(blob.data() + off, src, bytes);
    return off;
  };
  // LUT: lut[c] = #{e in E : e < c * 2^s}
  std::vector<uint8_t> lut8;
  std::vector<uint16_t> lut16;
  size_t off_lut = 0;
  if (p->lut_cells) {
    std::vector<uint32_t> lut(p->lut_cells);
    size_t j = 0;
    for (uint32_t c = 0; c < p->lut_cells; ++c) {
      uint64_t bound = (uint64_t)c << p->shift;
      while (j < p->edges.size() && (uint64_t)p->edges[j] < bound) ++j;
      lut[c] = (uint32_t)j;
    }
    if (p->lut_u8) {
      lut8.assign(lut.begin(), lut.end());
      off_lut = put(lut8.data(), lut8.size());
    } else {
      lut16.assign(lut.begin(), lut.end());
      off_lut = put(lut16.data(), lut16.size() * 2);
    }
  }
  size_t off_edges = put(p->edges.data(), p->edges.size() * 4);
  size_t off_b = put(p->b.data(), p->b.size() * 4);
  size_t off_cs = put(p->cs.data(), p->cs.size() * 4);
  size_t off_cl = put(p->cl.data(), p->cl.size() * 4);
  std::vector<uint16_t> b_edge, cs_edge, cl_edge, b_win, cs_win, cl_win;
  for (uint32_t v : p->b) {
    b_edge.push_back((uint16_t)index_of(p->edges, v));
    b_win.push_back(p->cs.empty() ? (uint16_t)index_of(p->windows, v) : 0);
  }
  for (uint32_t v : p->cs) {
    cs_win.push_back((uint16_t)index_of(p->windows, v));
    cs_edge.push_back((uint16_t)index_of(p->edges, v));
  }
  for (uint32_t v : p->cl) {
    cl_edge.push_back((uint16_t)index_of(p->edges, v));
    cl_win.push_back((uint16_t)index_of(p->windows, v));
  }
  if (p->windows.size() > 65535) return fail(p, FP_ERR_CONFIG, "too many windows");
  size_t off_be = put(b_edge.data(), b_edge.size() * 2);
  size_t off_ce = put(cl_edge.data(), cl_edge.size() * 2);
  size_t off_bw = put(b_win.data(), b_win.size() * 2);
  size_t off_sw = put(cs_win.data(), cs_win.size() * 2);
  size_t off_se = put(cs_edge.data(), cs_edge.size() * 2);
  size_t off_lw = put(cl_win.data(), cl_win.size() * 2);
  std::vector<uint32_t> arch;
  for (auto &m : p->models) {
    arch.push_back(m.n_layers); arch.push_back(m.n_kv_heads);
    arch.push_back(m.head_dim); arch.push_back(m.kv_elem_bytes);
  }
  size_t off_arch = put(arch.data(), arch.size() * 4);
  std::vector<unsigned long long> gu;
  std::vector<double> price;
  for (auto &g : p->gpus) {
    gu.push_back(g.hbm_bytes); gu.push_back(g.util_num); gu.push_back(g.util_den);
    gu.push_back(g.activation_reserve_bytes);
    price.push_back(g.price_per_gpu_hour);
  }
  size_t off_gu = put(gu.data(), gu.size() * 8);
  size_t off_price = put(price.data(), price.size() * 8);
  std::vector<unsigned long long> dep;
  for (auto &d : p->deploy) {
    dep.push_back(d.tp_degree); dep.push_back(d.gpus_per_instance); dep.push_back(d.weight_bytes_per_gpu);
  }
  size_t off_dep = put(dep.data(), dep.size() * 8);
  size_t off_win = put(p->windows.data(), p->windows.size() * 4);
  size_t off_mu = put(p->mu.data(), p->mu.size() * 8);

  p->blob_bytes = blob.size();
  CUDA_TRY(p, cudaMalloc(&p->d_blob, p->blob_bytes), "cudaMalloc tables");
  CUDA_TRY(p, cudaMemcpy(p->d_blob, blob.data(), p->blob_bytes, cudaMemcpyHostToDevice), "upload tables");
  CUDA_TRY(p, cudaMalloc(&p->d_hist, 2ull * p->nbins * 8), "cudaMalloc hist");
  CUDA_TRY(p, cudaMemset(p->d_hist, 0, 2ull * p->nbins * 8), "memset hist");
  // K1's accumulator copies: 16 for small |E| (a few KB), one for large ones
  // (K3 sums them per block)
  p->hist_copies = p->nbins <= 256 ? 16u : 1u;
  p->copies_elems = (size_t)p->hist_copies * 2 * p->nbins;
  CUDA_TRY(p, cudaMalloc(&p->d_hcopies, 2 * p->copies_elems * 8), "cudaMalloc hist copies");
  CUDA_TRY(p, cudaMemset(p->d_hcopies, 0, 2 * p->copies_elems * 8), "memset hist copies");
  if (p->dist && !(p->flags & FP_FLAG_P2P)) {
    CUDA_TRY(p, cudaMalloc(&p->d_fold, 2ull * p->nbins * 8), "cudaMalloc folded histogram");
  }
  CUDA_TRY(p, cudaMalloc(&p->d_err, 16), "cudaMalloc error word");
  CUDA_TRY(p, cudaMemset(p->d_err, 0, 16), "memset error word");
  if (p->flags & FP_FLAG_P2P) {
    p->xbuf_elems = 2ull * p->nbins;
    const size_t bytes = 2 * p->xbuf_elems * 8 + 256;
    CUDA_TRY(p, cudaMalloc(&p->d_xbuf, bytes), "cudaMalloc p2p exchange");
    CUDA_TRY(p, cudaMemset(p->d_xbuf, 0, bytes), "memset p2p exchange");
    p->d_xflag = reinterpret_cast<unsigned int *>(p->d_xbuf + 2 * p->xbuf_elems);
  }
  CUDA_TRY(p, cudaMalloc(&p->d_rcounts, 8 * 8), "cudaMalloc counts");
  CUDA_TRY(p, cudaMalloc(&p->d_best, (size_t)p->world * M * sizeof(fp_candidate)), "cudaMalloc best");
  CUDA_TRY(p, cudaMemset(p->d_best, 0, (size_t)p->world * M * sizeof(fp_candidate)), "memset best");

  unsigned char *B0 = p->d_blob;
  TraceArgs &ta = p->ta;
  ta.lut = p->lut_cells ? (const void *)(B0 + off_lut) : nullptr;
  ta.edges = reinterpret_cast<const uint32_t *>(B0 + off_edges);
  ta.lut_cells = p->lut_cells;
  ta.lut_u8 = p->lut_u8;
  ta.shift = p->shift;
  ta.n_edges = (uint32_t)p->edges.size();
  ta.max_edge = p->max_edge;
  ta.want_mass = !(p->flags & FP_FLAG_NO_MASS);
  ta.g_cnt = p->d_hcopies;              // (per sweep: the sweep's parity)
  ta.g_mass = p->d_hcopies + p->nbins;
  ta.hist_copies = p->hist_copies;

  EvalArgs &ea = p->ea;
  ea.hist_cnt = p->d_hcopies;
  ea.hist_mass = p->d_hcopies + p->nbins;
  ea.hist_copies = p->hist_copies;
  ea.hist_out = p->d_hist;
  ea.nbins = p->nbins;
  ea.b = reinterpret_cast<const uint32_t *>(B0 + off_b);
  ea.cs = reinterpret_cast<const uint32_t *>(B0 + off_cs);
  ea.cl = reinterpret_cast<const uint32_t *>(B0 + off_cl);
  ea.b_edge = reinterpret_cast<const uint16_t *>(B0 + off_be);
  ea.cl_edge = reinterpret_cast<const uint16_t *>(B0 + off_ce);
  ea.b_win = reinterpret_cast<const uint16_t *>(B0 + off_bw);
  ea.cs_win = reinterpret_cast<const uint16_t *>(B0 + off_sw);
  ea.cs_edge = reinterpret_cast<const uint16_t *>(B0 + off_se);
  ea.cl_win = reinterpret_cast<const uint16_t *>(B0 + off_lw);
  ea.n_b = (uint32_t)p->b.size();
  ea.n_cs = (uint32_t)p->cs.size();
  ea.n_cl = (uint32_t)p->cl.size();
  ea.n_cs_eff = p->n_cs_eff;
  ea.n_models = M;
  ea.n_gpus = G;
  ea.n_windows = W;
  // K3's index decomposition multipliers: ceil(2^64 / d), 0 for d = 1
  auto magic = [](uint64_t d) -> unsigned long long { return d <= 1 ? 0ull : (~0ull) / d + 1ull; };
  ea.div_b = magic(ea.n_b);
  ea.div_cs = magic(ea.n_cs_eff);
  ea.div_cl = magic(ea.n_cl);
  ea.div_g = magic(G);
  ea.model_arch = reinterpret_cast<const uint32_t *>(B0 + off_arch);
  ea.gpu_u64 = reinterpret_cast<const unsigned long long *>(B0 + off_gu);
  ea.price = reinterpret_cast<const double *>(B0 + off_price);
  ea.deploy = reinterpret_cast<const unsigned long long *>(B0 + off_dep);
  ea.windows = reinterpret_cast<const uint32_t *>(B0 + off_win);
  ea.mu = reinterpret_cast<const double *>(B0 + off_mu);
  ea.hours = p->hours;
  ea.per_model = p->per_model;
  ea.cand_first = p->cand_first;
  ea.cand_count = p->cand_count;
  ea.best_out = p->d_best + (size_t)((p->dist && !(p->flags & FP_FLAG_REPLICATED_GRID)) ? p->rank : 0) * M;
  ea.edges = ta.edges;
  ea.n_edges = ta.n_edges;
  // capacity table N_seq[m][g][w] (Eq. 2) and RN(1/mu): plan data only, computed once here
  CUDA_TRY(p, cudaMalloc(&p->d_cap, (size_t)M * G * W * 8), "cudaMalloc capacity table");
  CUDA_TRY(p, cudaMalloc(&p->d_rmu, (size_t)M * G * W * 8), "cudaMalloc reciprocal table");
  {
    cudaError_t e = launch_capacity(ea, p->d_cap, p->d_rmu, 0);
    if (e != cudaSuccess) return cuda_fail(p, e, "capacity table launch");
    CUDA_TRY(p, cudaDeviceSynchronize(), "capacity table");
  }
  ea.cap_nseq = p->d_cap;
  ea.rmu = p->d_rmu;
  ea.err_word = p->d_err;
  if (env_int("FP_K3_PHASES", 0)) {
    CUDA_TRY(p, cudaHostAlloc(&p->h_phase, 16 * 8, cudaHostAllocMapped), "cudaHostAlloc phases");
    memset(p->h_phase, 0, 16 * 8);
    unsigned long long *dptr = nullptr;
    CUDA_TRY(p, cudaHostGetDevicePointer(&dptr, p->h_phase, 0), "phase pointer");
    ea.phase_ts = dptr;
  }
  ea.p2p_timeout_ns = (unsigned long long)std::max(1, env_int("FP_P2P_TIMEOUT_MS", 10000)) * 1000000ull;

  // K3 grid: enough blocks for the largest per-model part of this rank's slice
  uint64_t widest = 0;
  for (uint32_t m = 0; m < M; ++m) {
    uint64_t lo = std::max<uint64_t>((uint64_t)m * p->per_model, p->cand_first);
    uint64_t hi = std::min<uint64_t>((uint64_t)(m + 1) * p->per_model, p->cand_first + p->cand_count);
    if (hi > lo) widest = std::max(widest, hi - lo);
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  CUDA_TRY(p, eval_prepare(), "k3 attributes");
  const size_t tab_smem = eval_smem_bytes(ea, 256);
  if (tab_smem > 190 * 1024)
    return fail(p, FP_ERR_CONFIG, "histogram + capacity table need %zu B of shared memory", tab_smem);
  // grid-stride shape (full records of large grids): one thread per candidate
  // up to ~8 blocks per SM in total, then grid-stride
  const uint64_t cap = std::max<uint64_t>(1, (uint64_t)sms * 8 / M);
  p->k3_grid_x = (int)std::min<uint64_t>(cap, std::max<uint64_t>(1, (widest + 255) / 256));
  p->k3_grid_x = std::max(1, std::min(p->k3_grid_x, env_int("FP_K3_GRID", p->k3_grid_x)));
  if (p->k3_grid_x > 65535 * 64) return fail(p, FP_ERR_CONFIG, "candidate grid too large for one launch");
  EvalLaunch grid;
  grid.shape = kK3Grid;
  grid.grid_x = p->k3_grid_x;
  grid.block = 256;
  grid.smem = tab_smem;
  // cluster shape: the paper-size grids, one cluster per model reduced in DSMEM
  // (<= 4 candidates per thread); FP_K3_SHAPE=grid|factored|cluster forces a shape
  const char *force = getenv("FP_K3_SHAPE");
  // 128-thread blocks when <= 2 candidates per thread: they fit beside the
  // trace pass's 3 x 512 threads on an SM, so the early-launched K3 loads its
  // tables while K1 drains; each thread keeps its best full record in shared memory
  EvalLaunch clu;
  clu.shape = kK3Cluster;
  clu.block = widest <= 2048 ? 128 : 256;
  clu.smem = tab_smem + (size_t)clu.block * sizeof(fp_candidate);
  const int max_cl = eval_max_cluster(clu.block, clu.smem);
  clu.grid_x = (int)std::min<uint64_t>(max_cl, std::max<uint64_t>(1, (widest + clu.block - 1) / clu.block));
  const bool cluster_ok = widest <= (uint64_t)clu.grid_x * clu.block * 4 && clu.smem <= 190 * 1024;
  // factored shape: large grids, argmin only
  // C_L values per block: the smallest power of two >= 16 whose grid fits in
  // one resident wave (2 blocks per SM): fewer blocks rebuild the short-pool
  // table fewer times, but a second partial wave costs more (2^24 grid:
  // 16 -> 41.1 us, 32 -> 29.6 us, 64 -> 31.1 us; profiles/r02/k3_factored_lc.md)
  {
    uint32_t lc = 16;
    const uint64_t kt = ((uint64_t)ea.n_b + 31) / 32;
    while (lc < 64 && (uint64_t)ea.n_gpus * ((ea.n_cl + lc - 1) / lc) * kt * M > (uint64_t)sms * 2) lc *= 2;
    ea.fac_lc = (uint32_t)std::max(1, std::min(64, env_int("FP_K3_LC", (int)lc)));
  }
  EvalLaunch fac;
  fac.shape = kK3Factored;
  fac.grid_x = (int)eval_factored_blocks_per_model(ea);
  fac.block = 256;
  fac.smem = eval_factored_smem_bytes(ea);
  const bool fac_ok = fac.smem <= 190 * 1024 && fac.grid_x <= 65535 * 64;
  if (force && !strcmp(force, "grid")) {
    p->k3a = grid;
    p->k3r = grid;
  } else if (force && !strcmp(force, "factored") && fac_ok) {
    p->k3a = fac;
    p->k3r = grid;
  } else if (cluster_ok && !(force && !strcmp(force, "factored"))) {
    p->k3a = clu;
    p->k3r = clu;
  } else {
    p->k3a = fac_ok ? fac : grid;
    p->k3r = grid;
  }
  const int bb_blocks = std::max(p->k3_grid_x, p->k3a.shape == kK3Factored ? p->k3a.grid_x : 1);
  CUDA_TRY(p, cudaMalloc(&p->d_block_best, (size_t)M * bb_blocks * sizeof(BlockBest)), "cudaMalloc block_best");
  CUDA_TRY(p, cudaMalloc(&p->d_done, M * sizeof(unsigned int)), "cudaMalloc done");
  CUDA_TRY(p, cudaMemset(p->d_done, 0, M * sizeof(unsigned int)), "memset done");
  ea.block_best = p->d_block_best;
  ea.done = p->d_done;
  p->k3_smem = tab_smem;
  return FP_OK;
}

fp_status configure_launch(fp_plan *p) {
  CUDA_TRY(p, cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, p->device), "attr");
  // tuning knobs (measurement only; defaults are the measured best on B200)
  p->ta.flush_iters = 1;  // set per launch by launch_trace's smem config
  p->k1_block = env_int("FP_K1_BLOCK", 512);
  if (p->k1_block < 64 || p->k1_block > 512 || (p->k1_block & 31))
    return fail(p, FP_ERR_CONFIG, "FP_K1_BLOCK must be a multiple of 32 in [64, 512]");
  p->k1_smem = trace_smem_bytes(p->ta, p->k1_block);
  if (p->k1_smem > 200 * 1024)
    return fail(p, FP_ERR_CONFIG, "trace-pass shared memory %zu B too large", p->k1_smem);
  int per_sm = 0;
  CUDA_TRY(p, trace_occupancy(p->ta, p->k1_block, p->k1_smem, &per_sm), "occupancy");
  // 3 x 512 threads per SM measured best for the grid-stride trace pass
  // (C5: 0.592 ms at 3, 0.605 at 4, 0.667 at 2; profiles/r01_tune_launch_*)
  const int k1_bps = env_int("FP_K1_BLOCKS_PER_SM", 3);
  if (k1_bps > 0) per_sm = std::min(per_sm, k1_bps);
  p->k1_grid = p->sm_count * std::max(1, per_sm);
  p->k4_block = env_int("FP_K4_BLOCK", 512);
  if (p->k4_block < 64 || p->k4_block > 512 || (p->k4_block & 31))
    return fail(p, FP_ERR_CONFIG, "FP_K4_BLOCK must be a multiple of 32 in [64, 512]");
  // persistent grid = every block resident (2 x 512 threads per SM with
  // __launch_bounds__(512, 2) and the next tile's loads in flight)
  int k4_res = 1;
  CUDA_TRY(p, route_occupancy(p->k4_block, &k4_res), "k4 occupancy");
  p->k4_grid = p->sm_count * std::min(k4_res, env_int("FP_K4_BLOCKS_PER_SM", k4_res));
  // pinned host mirrors for the small synchronous results
  CUDA_TRY(p, cudaMallocHost(&p->h_best, (size_t)p->world * p->models.size() * sizeof(fp_candidate)),
           "cudaMallocHost best");
  CUDA_TRY(p, cudaMallocHost(&p->h_small, (2ull * p->nbins + 8) * 8), "cudaMallocHost small");
  return FP_OK;
}

constexpr size_t kTimerRing = 256;

// The trace pass's grid for n requests: the plan's resident grid, but no more
// blocks than there is work for (16 requests per thread per grid-stride step),
// so a small trace does not pay 444 block prologues and flushes.
int k1_grid_for(const fp_plan *p, uint64_t n) {
  const uint64_t per_block = (uint64_t)p->k1_block * 16;
  const uint64_t want = std::max<uint64_t>(1, (n + per_block - 1) / per_block);
  return (int)std::min<uint64_t>((uint64_t)p->k1_grid, want);
}

// Fold the oldest pending event pair of `t` into its running total.
void timer_fold_one(fp_plan::Timer &t) {
  const size_t i = (t.head + t.ev.size() - t.pending) % t.ev.size();
  float ms = 0.f;
  if (cudaEventSynchronize(t.ev[i].second) == cudaSuccess &&
      cudaEventElapsedTime(&ms, t.ev[i].first, t.ev[i].second) == cudaSuccess)
    t.total_ms += ms;
  cudaGetLastError();
  --t.pending;
}

// Record an event pair around one launch of kernel `kind` (timing flags only).
struct LaunchTimer {
  fp_plan *p;
  cudaStream_t s;
  cudaEvent_t stop = nullptr;
  LaunchTimer(fp_plan *p_, int kind, cudaStream_t s_) : p(p_), s(s_) {
    if (!(p->flags & FP_FLAG_KERNEL_TIMING) && !((p->flags & FP_FLAG_TIME_TRACE) && kind == FP_KERNEL_TRACE))
      return;
    auto &t = p->timers[kind];
    if (t.pending == t.ev.size()) {
      if (t.ev.size() < kTimerRing) {
        // grow the ring: the new slot goes right after the newest pending pair
        cudaEvent_t a, b;
        if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) { cudaGetLastError(); return; }
        t.ev.insert(t.ev.begin() + t.head, std::make_pair(a, b));
      } else {
        timer_fold_one(t);               // ring full: fold the oldest (long finished) launch
      }
    }
    auto &pr = t.ev[t.head];
    t.head = (t.head + 1) % t.ev.size();
    ++t.pending;
    ++t.launches;
    cudaEventRecord(pr.first, s);
    stop = pr.second;
  }
  ~LaunchTimer() {
    if (stop) cudaEventRecord(stop, s);
  }
};

// NVTX range around a host-side phase (header-only NVTX3: a no-op unless a
// tool such as Nsight injects itself)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// The device error word (the P2P wait's timeout), read at the synchronising calls.
fp_status check_device_error(fp_plan *p) {
  unsigned int *h = reinterpret_cast<unsigned int *>(p->h_small + 2ull * p->nbins + 7);
  CUDA_TRY(p, cudaMemcpy(h, p->d_err, 4, cudaMemcpyDeviceToHost), "D2H error word");
  if (*h) {
    const unsigned int v = *h;
    CUDA_TRY(p, cudaMemset(p->d_err, 0, 4), "clear error word");
    return fail(p, FP_ERR_NCCL, "P2P exchange: rank %u did not publish its histogram within %d ms (a peer "
                "failed or stopped sweeping); results of that sweep are invalid", v >> 8,
                std::max(1, env_int("FP_P2P_TIMEOUT_MS", 10000)));
  }
  return FP_OK;
}

fp_status ensure_staging(fp_plan *p) {
  if (p->d_stage[0]) return FP_OK;
  for (int i = 0; i < 2; ++i) {
    CUDA_TRY(p, cudaMalloc(&p->d_stage[i], kChunkElems * 4), "cudaMalloc staging");
    CUDA_TRY(p, cudaEventCreateWithFlags(&p->ev_copied[i], cudaEventDisableTiming), "event");
    CUDA_TRY(p, cudaEventCreateWithFlags(&p->ev_used[i], cudaEventDisableTiming), "event");
  }
  CUDA_TRY(p, cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking), "copy stream");
  return FP_OK;
}

// Run `body(dev_ptr, n, offset)` over a trace that may live on the host: device
// traces go straight through, host traces are DMA'd chunk by chunk into two
// staging buffers on the copy stream (double-buffered, event-ordered).
// With `resident` (device, >= n elements) a host trace is copied there in
// full (each chunk processed as soon as it lands) instead of through the ring.
template <class F>
fp_status over_trace(fp_plan *p, const uint32_t *len, uint64_t n, cudaStream_t s, F body,
                     uint32_t *resident = nullptr) {
  if (n == 0) return FP_OK;
  if (!is_host_pointer(len)) return body(len, n, 0ull);
  fp_status st = ensure_staging(p);
  if (st != FP_OK) return st;
  // the copy stream must not run ahead of work already queued on s
  cudaEvent_t start;
  CUDA_TRY(p, cudaEventCreateWithFlags(&start, cudaEventDisableTiming), "event");
  cudaEventRecord(start, s);
  cudaStreamWaitEvent(p->copy_stream, start, 0);
  cudaEventDestroy(start);
  for (uint64_t off = 0, i = 0; off < n; off += kChunkElems, ++i) {
    const int k = (int)(i & 1);
    const uint64_t cnt = std::min<uint64_t>(kChunkElems, n - off);
    uint32_t *dst = resident ? resident + off : p->d_stage[k];
    if (i >= 2 && !resident) CUDA_TRY(p, cudaStreamWaitEvent(p->copy_stream, p->ev_used[k], 0), "wait used");
    CUDA_TRY(p, cudaMemcpyAsync(dst, len + off, cnt * 4, cudaMemcpyHostToDevice, p->copy_stream), "H2D chunk");
    CUDA_TRY(p, cudaEventRecord(p->ev_copied[k], p->copy_stream), "record copied");
    CUDA_TRY(p, cudaStreamWaitEvent(s, p->ev_copied[k], 0), "wait copied");
    st = body(dst, cnt, off);
    if (st != FP_OK) return st;
    CUDA_TRY(p, cudaEventRecord(p->ev_used[k], s), "record used");
  }
  return FP_OK;
}

// ---- the two cross-rank operations of the path (NCCL or host hooks) ----------
fp_status all_reduce_u64(fp_plan *p, unsigned long long *dbuf, size_t count, cudaStream_t s, const char *what) {
  if (!p->has_coll)
    return nccl_check(p, g_nccl.AllReduce(dbuf, dbuf, count, kNcclUint64, kNcclSum, p->comm, s), what);
  std::vector<uint64_t> h(count);
  CUDA_TRY(p, cudaMemcpyAsync(h.data(), dbuf, count * 8, cudaMemcpyDeviceToHost, s), what);
  CUDA_TRY(p, cudaStreamSynchronize(s), what);
  if (p->coll.allreduce_sum_u64(h.data(), count, p->coll.user) != 0)
    return fail(p, FP_ERR_NCCL, "%s: collectives hook failed", what);
  CUDA_TRY(p, cudaMemcpyAsync(dbuf, h.data(), count * 8, cudaMemcpyHostToDevice, s), what);
  CUDA_TRY(p, cudaStreamSynchronize(s), what);
  return FP_OK;
}

fp_status all_reduce_u32(fp_plan *p, uint32_t *dbuf, size_t count, cudaStream_t s, const char *what) {
  if (!p->has_coll)
    return nccl_check(p, g_nccl.AllReduce(dbuf, dbuf, count, kNcclUint32, kNcclSum, p->comm, s), what);
  // host hooks carry u64 sums: widen, reduce, narrow (sums are bounded by the caller)
  std::vector<uint32_t> h(count);
  CUDA_TRY(p, cudaMemcpyAsync(h.data(), dbuf, count * 4, cudaMemcpyDeviceToHost, s), what);
  CUDA_TRY(p, cudaStreamSynchronize(s), what);
  std::vector<uint64_t> w(h.begin(), h.end());
  if (p->coll.allreduce_sum_u64(w.data(), count, p->coll.user) != 0)
    return fail(p, FP_ERR_NCCL, "%s: collectives hook failed", what);
  for (size_t i = 0; i < count; ++i) h[i] = (uint32_t)w[i];
  CUDA_TRY(p, cudaMemcpyAsync(dbuf, h.data(), count * 4, cudaMemcpyHostToDevice, s), what);
  CUDA_TRY(p, cudaStreamSynchronize(s), what);
  return FP_OK;
}

fp_status all_gather_bytes(fp_plan *p, const void *dsend, void *drecv, size_t bytes, cudaStream_t s,
                           const char *what) {
  if (!p->has_coll)
    return nccl_check(p, g_nccl.AllGather(dsend, drecv, bytes, kNcclUint8, p->comm, s), what);
  std::vector<unsigned char> hs(bytes), hr(bytes * (size_t)p->world);
  CUDA_TRY(p, cudaMemcpyAsync(hs.data(), dsend, bytes, cudaMemcpyDeviceToHost, s), what);
  CUDA_TRY(p, cudaStreamSynchronize(s), what);
  if (p->coll.allgather_bytes(hs.data(), hr.data(), bytes, p->coll.user) != 0)
    return fail(p, FP_ERR_NCCL, "%s: collectives hook failed", what);
  CUDA_TRY(p, cudaMemcpyAsync(drecv, hr.data(), hr.size(), cudaMemcpyHostToDevice, s), what);
  CUDA_TRY(p, cudaStreamSynchronize(s), what);
  return FP_OK;
}

}  // namespace

// ============================== ABI ==========================================

extern "C" {

const char *fp_status_string(fp_status s) {
  switch (s) {
    case FP_OK: return "ok";
    case FP_ERR_INVALID_ARG: return "invalid argument";
    case FP_ERR_CONFIG: return "invalid configuration";
    case FP_ERR_EMPTY_TRACE: return "empty trace";
    case FP_ERR_ALIGNMENT: return "misaligned buffer";
    case FP_ERR_OOM: return "out of memory";
    case FP_ERR_CUDA: return "CUDA error";
    case FP_ERR_NCCL: return "NCCL error";
    case FP_ERR_STATE: return "invalid call order";
  }
  return "unknown status";
}

const char *fp_last_error(const fp_plan *plan) { return plan ? plan->err.c_str() : "no plan"; }

void fp_shard_range(uint64_t n_total, int32_t rank, int32_t world, uint64_t *first, uint64_t *count) {
  if (world < 1) world = 1;
  uint64_t per = (n_total + (uint64_t)world - 1) / (uint64_t)world;
  per = (per + 31) / 32 * 32;
  uint64_t lo = std::min<uint64_t>(n_total, (uint64_t)rank * per);
  uint64_t hi = std::min<uint64_t>(n_total, lo + per);
  *first = lo;
  *count = hi - lo;
}

void fp_candidate_range(uint64_t n_candidates, int32_t rank, int32_t world, uint64_t *first, uint64_t *count) {
  if (world < 1) world = 1;
  uint64_t per = (n_candidates + (uint64_t)world - 1) / (uint64_t)world;
  uint64_t lo = std::min<uint64_t>(n_candidates, (uint64_t)rank * per);
  uint64_t hi = std::min<uint64_t>(n_candidates, lo + per);
  *first = lo;
  *count = hi - lo;
}

void fp_merge_best(const fp_candidate *recs, int32_t world, uint32_t n_models, fp_candidate *out) {
  for (uint32_t m = 0; m < n_models; ++m) {
    const fp_candidate *best = nullptr;
    for (int32_t r = 0; r < world; ++r) {
      const fp_candidate *c = recs + (size_t)r * n_models + m;
      if (!(c->flags & FP_CAND_FEASIBLE)) continue;
      if (!best || c->cost_dual < best->cost_dual ||
          (c->cost_dual == best->cost_dual && c->index < best->index))
        best = c;
    }
    if (best) {
      out[m] = *best;
    } else {
      memset(&out[m], 0, sizeof(fp_candidate));
      out[m].index = 0xffffffffu;
      out[m].model = m;
      out[m].cost_dual = out[m].cost_homo = INFINITY;
    }
  }
}

fp_status fp_nccl_get_unique_id(void *out128) {
  if (!out128) return FP_ERR_INVALID_ARG;
  std::string err;
  if (!load_nccl(g_nccl, err)) return FP_ERR_NCCL;
  NcclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != 0) return FP_ERR_NCCL;
  memcpy(out128, &id, sizeof id);
  return FP_OK;
}

fp_status fp_p2p_export(fp_plan *p, void *handle_out) {
  if (!p || !handle_out) return FP_ERR_INVALID_ARG;
  if (!(p->flags & FP_FLAG_P2P) || !p->d_xbuf) return fail(p, FP_ERR_STATE, "plan created without FP_FLAG_P2P");
  static_assert(sizeof(cudaIpcMemHandle_t) == FP_P2P_HANDLE_BYTES, "IPC handle size");
  DeviceGuard g(p->device);
  cudaIpcMemHandle_t h;
  CUDA_TRY(p, cudaIpcGetMemHandle(&h, p->d_xbuf), "cudaIpcGetMemHandle");
  memcpy(handle_out, &h, sizeof h);
  return FP_OK;
}

fp_status fp_p2p_import(fp_plan *p, const void *handles) {
  if (!p || !handles) return FP_ERR_INVALID_ARG;
  if (!(p->flags & FP_FLAG_P2P) || !p->d_xbuf) return fail(p, FP_ERR_STATE, "plan created without FP_FLAG_P2P");
  if (p->p2p_ready) return fail(p, FP_ERR_STATE, "fp_p2p_import called twice");
  DeviceGuard g(p->device);
  std::vector<unsigned long long *> hist(p->world);
  std::vector<unsigned int *> flag(p->world);
  for (int r = 0; r < p->world; ++r) {
    unsigned long long *base = p->d_xbuf;
    if (r != p->rank) {
      cudaIpcMemHandle_t h;
      memcpy(&h, static_cast<const unsigned char *>(handles) + (size_t)r * FP_P2P_HANDLE_BYTES, sizeof h);
      void *q = nullptr;
      CUDA_TRY(p, cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      p->peer_open.push_back(q);
      base = static_cast<unsigned long long *>(q);
    }
    hist[r] = base;
    flag[r] = reinterpret_cast<unsigned int *>(base + 2 * p->xbuf_elems);
  }
  CUDA_TRY(p, cudaMalloc(&p->d_peer_hist, p->world * sizeof(void *)), "cudaMalloc peer table");
  CUDA_TRY(p, cudaMalloc(&p->d_peer_flag, p->world * sizeof(void *)), "cudaMalloc peer table");
  CUDA_TRY(p, cudaMemcpy(p->d_peer_hist, hist.data(), p->world * sizeof(void *), cudaMemcpyHostToDevice), "H2D");
  CUDA_TRY(p, cudaMemcpy(p->d_peer_flag, flag.data(), p->world * sizeof(void *), cudaMemcpyHostToDevice), "H2D");
  p->p2p_ready = true;
  return FP_OK;
}

fp_status fleet_plan_create(const fp_plan_desc *desc, fp_plan **out) {
  if (!out) return FP_ERR_INVALID_ARG;
  *out = nullptr;
  if (!desc) return FP_ERR_INVALID_ARG;
  fp_plan *p = new fp_plan();
  fp_status st = validate_and_copy(p, desc);
  if (st == FP_OK) st = build_tables(p);
  if (st == FP_OK) {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      st = fail(p, FP_ERR_CUDA, "no CUDA device (%s)", cudaGetErrorString(e));
    } else if (p->device < 0 || p->device >= ndev) {
      st = fail(p, FP_ERR_CONFIG, "device %d out of range (%d devices)", p->device, ndev);
    }
  }
  if (st == FP_OK) {
    DeviceGuard g(p->device);
    st = upload(p);
    if (st == FP_OK) st = configure_launch(p);
    if (st == FP_OK && p->dist && !p->has_coll) {
      std::string err;
      if (!load_nccl(g_nccl, err)) {
        st = fail(p, FP_ERR_NCCL, "%s", err.c_str());
      } else {
        NcclUniqueId id;
        memcpy(&id, desc->nccl_unique_id, sizeof id);
        st = nccl_check(p, g_nccl.CommInitRank(&p->comm, p->world, id, p->rank), "ncclCommInitRank");
      }
    }
  }
  if (st != FP_OK) {
    fprintf(stderr, "fleet_plan_create: %s: %s\n", fp_status_string(st), p->err.c_str());
    fleet_plan_destroy(p);
    return st;
  }
  *out = p;
  return FP_OK;
}

void fleet_plan_destroy(fp_plan *p) {
  if (!p) return;
  {
    DeviceGuard g(p->device);
    if (p->last_stream || p->have_sweep) cudaDeviceSynchronize();
    if (p->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(p->comm);
    cudaFree(p->d_blob);
    cudaFree(p->d_hist);
    cudaFree(p->d_hcopies);
    for (void *q : p->peer_open) cudaIpcCloseMemHandle(q);
    cudaFree(p->d_peer_hist);
    cudaFree(p->d_peer_flag);
    cudaFree(p->d_xbuf);
    cudaFree(p->d_rcounts);
    cudaFree(p->d_cap);
    cudaFree(p->d_best);
    cudaFree(p->d_results);
    cudaFree(p->d_block_best);
    cudaFree(p->d_done);
    cudaFree(p->d_fold);
    cudaFree(p->d_spec);
    cudaFree(p->d_rmu);
    cudaFree(p->d_err);
    if (p->ev_order) cudaEventDestroy(p->ev_order);
    for (cudaGraphExec_t &x : p->graph.exec)
      if (x) cudaGraphExecDestroy(x);
    if (p->graph_stream) cudaStreamDestroy(p->graph_stream);
    cudaFree(p->d_resident);
    cudaFree(p->d_bins);
    cudaFree(p->d_p3);
    cudaFree(p->d_calib_scratch);
    cudaFree(p->d_peak);
    cudaFree(p->d_xch);
    cudaFree(p->d_results_pk);
    cudaFree(p->d_results3);
    cudaFree(p->d_calib);
    for (int i = 0; i < 2; ++i) {
      cudaFree(p->d_stage[i]);
      if (p->ev_copied[i]) cudaEventDestroy(p->ev_copied[i]);
      if (p->ev_used[i]) cudaEventDestroy(p->ev_used[i]);
    }
    if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
    if (p->h_phase) {
      if (p->phase_n) {
        fprintf(stderr, "[fp] K3 phases over %llu sweeps (us after entry): ", (unsigned long long)p->phase_n);
        for (int i = 1; i <= 10; ++i) fprintf(stderr, "%d:%.2f ", i, p->phase_sum[i] / p->phase_n / 1e3);
        fprintf(stderr, "\n");
      }
      cudaFreeHost(p->h_phase);
    }
    if (p->h_best) cudaFreeHost(p->h_best);
    if (p->h_small) cudaFreeHost(p->h_small);
    for (auto &t : p->timers)
      for (auto &pr : t.ev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    cudaGetLastError();
  }
  delete p;
}

fp_status fleet_plan_info(const fp_plan *p, fp_plan_info *o) {
  if (!p || !o) return FP_ERR_INVALID_ARG;
  o->n_candidates = p->n_cand;
  o->cand_first = p->cand_first;
  o->cand_count = p->cand_count;
  o->n_edges = (uint32_t)p->edges.size();
  o->lut_shift = p->shift;
  o->lut_cells = p->lut_cells;
  o->n_windows = (uint32_t)p->windows.size();
  o->device = p->device;
  o->rank = p->rank;
  o->world = p->world;
  o->sm_count = (uint32_t)p->sm_count;
  o->k1_grid = (uint32_t)p->k1_grid;
  o->k1_block = (uint32_t)p->k1_block;
  o->nccl_comm_size = 0;
  if (p->comm && g_nccl.CommCount) {
    int n = 0;
    if (g_nccl.CommCount(p->comm, &n) == 0) o->nccl_comm_size = n;
  }
  o->k3_shape = (uint32_t)p->k3a.shape;
  o->k3_blocks_per_model = (uint32_t)p->k3a.grid_x;
  o->spec_calls = (uint32_t)p->spec_calls;
  o->spec_misses = 0;
  if (p->spec_miss) {
    DeviceGuard g(p->device);
    if (p->last_stream) cudaStreamSynchronize(p->last_stream);
    unsigned int m = 0;
    if (cudaMemcpy(&m, p->spec_miss, 4, cudaMemcpyDeviceToHost) == cudaSuccess) o->spec_misses = m;
    cudaGetLastError();
  }
  return FP_OK;
}

uint64_t fp_kernel_launches(const fp_plan *p) { return p ? p->launches : 0; }

fp_status fp_kernel_time(fp_plan *p, int32_t kind, double *total_ms, uint64_t *launches) {
  if (!p || kind < 0 || kind > 2) return FP_ERR_INVALID_ARG;
  if (!(p->flags & FP_FLAG_KERNEL_TIMING) && !((p->flags & FP_FLAG_TIME_TRACE) && kind == FP_KERNEL_TRACE))
    return fail(p, FP_ERR_STATE, "kernel kind %d is not timed (FP_FLAG_KERNEL_TIMING / FP_FLAG_TIME_TRACE)", kind);
  DeviceGuard g(p->device);
  auto &t = p->timers[kind];
  while (t.pending) timer_fold_one(t);
  if (total_ms) *total_ms = t.total_ms;
  if (launches) *launches = t.launches;
  return FP_OK;
}

fp_status fp_kernel_time_reset(fp_plan *p) {
  if (!p) return FP_ERR_INVALID_ARG;
  DeviceGuard g(p->device);
  for (auto &t : p->timers) {
    while (t.pending) timer_fold_one(t);
    t.total_ms = 0.0;
    t.launches = 0;
  }
  return FP_OK;
}

fp_status route_batch(fp_plan *p, const uint32_t *d_len, uint64_t n_local, uint32_t b_short,
                      uint32_t c_short, uint32_t c_long, uint8_t *d_decision, fp_route_counts *h_counts,
                      void *stream) {
  if (!p) return FP_ERR_INVALID_ARG;
  if (n_local && !d_len) return fail(p, FP_ERR_INVALID_ARG, "d_len is NULL");
  if (!(b_short >= 1 && b_short <= c_short && c_short <= c_long))
    return fail(p, FP_ERR_INVALID_ARG, "need 1 <= B_short <= C_S <= C_L (S:316-321)");
  if (d_decision && n_local && is_host_pointer(d_decision))
    return fail(p, FP_ERR_INVALID_ARG, "d_decision must be device memory");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(p, cudaMemsetAsync(p->d_rcounts, 0, 5 * 8, s), "memset counts");
  RouteArgs ra{};
  ra.b = b_short;
  ra.cs = c_short;
  ra.cl = c_long;
  ra.g_counts = p->d_rcounts;
  fp_status st = over_trace(p, d_len, n_local, s, [&](const uint32_t *ptr, uint64_t n, uint64_t off) {
    RouteArgs r = ra;
    r.len = ptr;
    r.n = n;
    r.decision = d_decision ? d_decision + off : nullptr;
    LaunchTimer lt(p, FP_KERNEL_ROUTE, s);
    cudaError_t e = launch_route(r, p->k4_grid, p->k4_block, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "route_batch launch");
    ++p->launches;
    return FP_OK;
  });
  if (st != FP_OK) return st;
  if (p->dist) {
    st = all_reduce_u64(p, p->d_rcounts, 5, s, "all-reduce(route counts)");
    if (st != FP_OK) return st;
  }
  p->last_stream = s;
  if (h_counts) {
    unsigned long long *c = p->h_small + 2ull * p->nbins;
    CUDA_TRY(p, cudaMemcpyAsync(c, p->d_rcounts, 5 * 8, cudaMemcpyDeviceToHost, s), "D2H counts");
    CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
    h_counts->n_short = c[0];
    h_counts->n_long = c[1];
    h_counts->n_reject = c[2];
    h_counts->mass_short = c[3];
    h_counts->mass_long = c[4];
  }
  return FP_OK;
}

namespace {
fp_status sweep_impl(fp_plan *p, const uint32_t *d_len, uint64_t n_local, double rate_rps,
                     fp_candidate *h_results, void *stream, uint32_t *resident,
                     const TraceArgs *raw = nullptr, uint8_t *bins = nullptr, uint32_t *route_out = nullptr,
                     uint32_t route_model = 0, uint8_t *bins_side = nullptr, uint8_t *bins_hi = nullptr,
                     const uint32_t *dec_route = nullptr, unsigned long long *zero2 = nullptr);
}

fp_status sweep_thresholds(fp_plan *p, const uint32_t *d_len, uint64_t n_local, double rate_rps,
                           fp_candidate *h_results, void *stream) {
  return sweep_impl(p, d_len, n_local, rate_rps, h_results, stream, nullptr);
}

namespace {
// FP_FLAG_SPECULATE path of sweep_and_route (preconditions checked by the caller).
// raw != NULL: the raw-column form (sweep_and_route_raw): *raw is the trace
// pass's TraceArgs with the columns and estimator set, rr the verify's args.
// the smallest trace (log2 requests per rank) that speculates with a u16 LUT:
// the wide grids' K3 (~14 us for C3's 30,720 candidates) runs twice per step,
// which 2 B/request saved pays for only above ~2e8 requests (C3 at 1e8: 0.191
// ms speculative vs 0.174 ms with the bin pass; profiles/r02/spec_wide/)
static unsigned spec_min_wide_log2() {
  return (unsigned)std::min(40, std::max(1, env_int("FP_SPEC_MIN_WIDE_LOG2", 28)));
}

fp_status sweep_route_speculative(fp_plan *p, const uint32_t *len, uint64_t n_local, double rate_rps,
                                  uint32_t route_model, uint8_t *d_decision, fp_candidate *h_best,
                                  fp_route_counts *h_counts, cudaStream_t s, const TraceArgs *raw = nullptr,
                                  const RouteRawArgs *rr = nullptr) {
  const size_t M = p->models.size();
  if (!p->d_spec) {
    const size_t acc_b = p->copies_elems * 8, best_b = M * sizeof(fp_candidate);
    CUDA_TRY(p, cudaMalloc(&p->d_spec, acc_b + best_b + 32), "cudaMalloc speculation state");
    CUDA_TRY(p, cudaMemset(p->d_spec, 0, acc_b + best_b + 32), "memset speculation state");
    p->spec_acc = reinterpret_cast<unsigned long long *>(p->d_spec);
    p->spec_best = reinterpret_cast<fp_candidate *>(p->d_spec + acc_b);
    p->spec_route = reinterpret_cast<uint32_t *>(p->d_spec + acc_b + best_b);
    p->spec_miss = reinterpret_cast<unsigned int *>(p->d_spec + acc_b + best_b + 16);
  }
  ++p->spec_calls;
  // (a failed earlier call left the sample's accumulators dirty: only the
  // speculation would suffer -- the verify keeps the result exact -- but clear them)
  if (p->spec_dirty) CUDA_TRY(p, cudaMemsetAsync(p->spec_acc, 0, p->copies_elems * 8, s), "memset sample hist");
  p->spec_dirty = true;
  // 1. the sample: every stride-th grid-wide stripe of the trace pass (~4 stripes;
  //    6 -> 4 -> 2 stripes: 0.833 -> 0.827 -> 0.823 ms per C5 step, 0 misses each)
  {
    NvtxRange r("fp:K1s sample pass");
    TraceArgs t = raw ? *raw : p->ta;
    t.len = raw ? nullptr : len;
    t.n = n_local;
    t.g_cnt = p->spec_acc;
    t.g_mass = p->spec_acc + p->nbins;
    const int grid = k1_grid_for(p, n_local);
    // uint4 per grid step of k1_trace (kUnroll = 4; raw columns: 2)
    const uint64_t stripe = (uint64_t)grid * p->k1_block * (raw ? 2 : 4);
    const uint64_t nsteps = (n_local / 4 + stripe - 1) / stripe;
    static const uint64_t stripes = (uint64_t)std::max(1, env_int("FP_SPEC_STRIPES", 4));
    t.step_stride = (uint32_t)std::max<uint64_t>(1, nsteps / stripes);
    t.pdl = 1;          // its prologue overlaps the previous kernel's tail (it waits before reading)
    cudaError_t e = launch_trace(t, grid, p->k1_block, p->k1_smem, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "sample pass launch");
    ++p->launches;
  }
  // 2. its K3: the speculated split of route_model
  {
    NvtxRange r("fp:K3s sample evaluation");
    EvalArgs es = p->ea;
    es.hist_cnt = p->spec_acc;
    es.hist_mass = p->spec_acc + p->nbins;
    es.hist_copies = p->hist_copies;
    es.rate = rate_rps;
    es.results = nullptr;
    es.zero_copies = nullptr;
    es.zero_copies2 = nullptr;
    es.hist_out = nullptr;
    es.best_out = p->spec_best;
    es.route_out = p->spec_route;
    es.route_model = route_model;
    es.p2p_world = 0;
    es.phase_ts = nullptr;
    es.cand_first = 0;                   // the whole grid on every rank (its own sample)
    es.cand_count = p->n_cand;
    cudaError_t e = launch_eval(es, p->k3a, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "sample evaluation launch");
    ++p->launches;
  }
  // 3. + 4. the full trace pass writing decisions for the speculated split, the full K3
  // (ranks that split the grid: the final split is picked after the all-gather)
  uint32_t *route = reinterpret_cast<uint32_t *>(p->d_rcounts);
  const bool sliced = p->dist && !(p->flags & FP_FLAG_REPLICATED_GRID);
  TraceArgs traw;
  if (raw) {                                 // the raw branch of sweep_impl takes the decision output here
    traw = *raw;
    traw.bins_out = d_decision;
    traw.dec_route = p->spec_route;
    traw.pdl = 1;
  }
  fp_status st = sweep_impl(p, raw ? nullptr : len, n_local, rate_rps, nullptr, s, nullptr, raw ? &traw : nullptr,
                            d_decision, sliced ? nullptr : route, route_model, nullptr, nullptr, p->spec_route,
                            p->spec_acc);
  if (st != FP_OK) return st;
  p->spec_dirty = false;                    // the full K3 zeroes the sample's accumulators
  if (sliced) {
    cudaError_t e = launch_pick_route(p->d_best, p->world, (uint32_t)M, route_model, p->ta.edges,
                                      (uint32_t)p->edges.size(), route, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "route pick launch");
    ++p->launches;
  }
  // 5. verify: re-route from L_total when the final split differs
  {
    NvtxRange r("fp:K4v verify");
    LaunchTimer lt(p, FP_KERNEL_ROUTE, s);
    cudaError_t e = raw ? launch_route_verify_raw(*rr, p->spec_route, route, p->ta.edges, p->spec_miss, p->k4_grid,
                                                  p->k4_block, s)
                        : launch_route_verify(len, d_decision, n_local, p->spec_route, route, p->ta.edges,
                                              p->spec_miss, p->k4_grid, p->k4_block, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "verify launch");
    ++p->launches;
  }
  p->last_stream = s;
  if (!h_best && !h_counts) return FP_OK;
  std::vector<fp_candidate> best(M);
  st = best_split(p, best.data());
  if (st != FP_OK) return st;
  if (h_best) memcpy(h_best, best.data(), best.size() * sizeof(fp_candidate));
  const fp_candidate &b = best[route_model];
  if (!(b.flags & FP_CAND_FEASIBLE))
    return fail(p, FP_ERR_STATE, "model %u has no feasible split to route with", route_model);
  if (h_counts) {
    h_counts->n_short = b.n_short;
    h_counts->n_long = b.n_long;
    h_counts->n_reject = b.n_reject;
    h_counts->mass_short = b.mass_short;
    h_counts->mass_long = b.mass_long;
  }
  return FP_OK;
}
}  // namespace

fp_status sweep_and_route(fp_plan *p, const uint32_t *len, uint64_t n_local, double rate_rps,
                          uint32_t route_model, uint8_t *d_decision, fp_candidate *h_best,
                          fp_route_counts *h_counts, void *stream) {
  if (!p) return FP_ERR_INVALID_ARG;
  if (route_model >= p->models.size()) return fail(p, FP_ERR_INVALID_ARG, "route_model out of range");
  if (d_decision && n_local && is_host_pointer(d_decision))
    return fail(p, FP_ERR_INVALID_ARG, "d_decision must be device memory");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  // Bin pass (|E| < 256, u8 LUT): the trace pass also writes every request's
  // bin (1 B); the routing pass maps bins to decisions (1 B in, 1 B out) and
  // the route counts are the best record's counts (same histogram). A host
  // trace then never needs a device copy. Otherwise: K4 re-reads L_total
  // (from a device copy for host traces).
  // |E| >= 256 (u16 LUT): clamped bytes (k1_trace bin_byte) for device traces,
  // the routing pass reading L_total back for requests above the 255th edge
  // when the split needs it
  const bool bin_pass = p->lut_cells && (p->lut_u8 || (len && !is_host_pointer(len)));
  // |E| + 1 <= 64 bins, device trace: 6-bit packed bins (0.75 B per request each way)
  const bool pack = bin_pass && p->nbins <= 64 && !(len && is_host_pointer(len));
  const uint32_t *src = len;
  uint32_t *resident = nullptr;
  uint8_t *bins = nullptr, *side = nullptr, *bins_hi = nullptr;
  uint32_t head = 0;
  int k1_grid_used = p->k1_grid;
  if (bin_pass) {
    if (d_decision && n_local) {
      // elements before the trace pass's first 16-B aligned uint4 (host traces
      // are processed from 256-B aligned staging chunks: none)
      const uintptr_t lp = is_host_pointer(len) ? 0 : reinterpret_cast<uintptr_t>(len);
      const uint64_t head_phase = (4 - ((lp & 15u) >> 2)) & 3u;
      head = (uint32_t)head_phase;
      // packed: [16 B side bytes (head / tail bins)][u64 x chunks][u32 x chunks],
      // one chunk per (step, thread) of the trace pass (TraceArgs::bins_pack);
      // bytes: one bin per request, placed so that bins + i and len + i share
      // the 4-B phase the trace pass needs for its 32-bit stores of 4 bins
      uint64_t chunks = 0;
      if (pack) {
        TraceArgs tq = p->ta;
        tq.bins_out = reinterpret_cast<uint8_t *>(16);   // any non-null: the bin variant's grid
        tq.bins_pack = 1;
        k1_grid_used = trace_grid(tq, k1_grid_for(p, n_local), p->k1_block);
        const uint64_t S = (uint64_t)k1_grid_used * p->k1_block;
        const uint64_t n4 = (n_local - std::min<uint64_t>(n_local, head_phase)) / 4;
        chunks = std::max<uint64_t>(1, (n4 + 4 * S - 1) / (4 * S)) * S;
      }
      const uint64_t need = pack ? 16 + 12 * chunks + 16 : n_local + 16;
      if (p->bins_cap < need) {
        cudaFree(p->d_bins);
        p->d_bins = nullptr;
        p->bins_cap = 0;
        CUDA_TRY(p, cudaMalloc(&p->d_bins, need), "cudaMalloc bins");
        p->bins_cap = need;
      }
      if (pack) {
        side = p->d_bins;
        bins = p->d_bins + 16;                 // u64 low nibbles [chunks]
        bins_hi = bins + 8 * chunks;           // u32 high parts [chunks]
      } else {
        bins = p->d_bins + ((4 - head_phase) & 3u);
      }
    }
  } else if (n_local && len && is_host_pointer(len)) {
    if (p->resident_cap < n_local) {
      cudaFree(p->d_resident);
      p->d_resident = nullptr;
      p->resident_cap = 0;
      CUDA_TRY(p, cudaMalloc(&p->d_resident, n_local * 4), "cudaMalloc resident trace");
      p->resident_cap = n_local;
    }
    resident = p->d_resident;
    src = resident;
  }
  // FP_FLAG_SPECULATE (header): sample pass -> its K3 picks a split -> the full
  // trace pass writes decisions for it -> full K3 -> verify / re-route
  {
    const uintptr_t lp = len ? reinterpret_cast<uintptr_t>(len) : 0;
    const uint64_t hph = (4 - ((lp & 15u) >> 2)) & 3u;
    const bool spec = (p->flags & FP_FLAG_SPECULATE) && d_decision && len && !is_host_pointer(len) &&
                      n_local >= (1ull << (p->lut_u8 ? 26 : spec_min_wide_log2())) && p->lut_cells &&
                      (!p->lut_u8 || p->nbins <= 127) &&
                      p->k3a.shape == kK3Cluster && (reinterpret_cast<uintptr_t>(d_decision + hph) & 3u) == 0;
    if (spec) return sweep_route_speculative(p, len, n_local, rate_rps, route_model, d_decision, h_best, h_counts, s);
  }
  // pick the split and route on the device: no host round trip in the step.
  // With one rank's grid = the whole grid, K3's last block of route_model
  // writes the split's edge indices; otherwise a one-warp kernel merges the
  // ranks' records after the all-gather.
  const bool routing = bin_pass && d_decision && n_local;
  const bool sliced = p->dist && !(p->flags & FP_FLAG_REPLICATED_GRID);   // ranks split the grid
  uint32_t *route = reinterpret_cast<uint32_t *>(p->d_rcounts);
  fp_status st = sweep_impl(p, len, n_local, rate_rps, nullptr, stream, resident, nullptr, bins,
                            routing && !sliced ? route : nullptr, route_model, side, bins_hi);
  if (st != FP_OK) return st;
  if (routing) {
    LaunchTimer lt(p, FP_KERNEL_ROUTE, s);
    const fp_candidate *recs = sliced ? p->d_best : nullptr;
    const int ranks = sliced ? p->world : 1;
    cudaError_t e =
        pack ? launch_route_packed(bins, bins_hi, side, head, d_decision, n_local, recs, ranks,
                                   (uint32_t)p->models.size(), route_model, p->ta.edges, (uint32_t)p->edges.size(),
                                   route, k1_grid_used, p->k1_block, s)
             : launch_route_bins(bins, d_decision, n_local, recs, ranks, (uint32_t)p->models.size(), route_model,
                                 p->ta.edges, (uint32_t)p->edges.size(), route, p->k4_grid, p->k4_block, s, len);
    if (e != cudaSuccess) return cuda_fail(p, e, "route (bins) launch");
    p->launches += sliced ? 2 : 1;
  }
  if (bin_pass && !h_best && !h_counts && !is_host_pointer(len)) {
    p->last_stream = s;                     // asynchronous: the records stay on the device
    return FP_OK;
  }
  std::vector<fp_candidate> best(p->models.size());
  st = best_split(p, best.data());          // D2H of the records, after the routing pass
  if (st != FP_OK) return st;
  if (h_best) memcpy(h_best, best.data(), best.size() * sizeof(fp_candidate));
  const fp_candidate &b = best[route_model];
  if (!(b.flags & FP_CAND_FEASIBLE))
    return fail(p, FP_ERR_STATE, "model %u has no feasible split to route with", route_model);
  if (!bin_pass) return route_batch(p, src, n_local, b.b_short, b.c_short, b.c_long, d_decision, h_counts, stream);
  if (h_counts) {
    h_counts->n_short = b.n_short;
    h_counts->n_long = b.n_long;
    h_counts->n_reject = b.n_reject;
    h_counts->mass_short = b.mass_short;
    h_counts->mass_long = b.mass_long;
  }
  p->last_stream = s;
  return FP_OK;
}

fp_status sweep_and_route_graph(fp_plan *p, const uint32_t *len, uint64_t n_local, double rate_rps,
                                uint32_t route_model, uint8_t *d_decision, void *stream) {
  if (!p) return FP_ERR_INVALID_ARG;
  if (p->dist || (p->flags & (FP_FLAG_COLLECTIVES | FP_FLAG_P2P)))
    return fail(p, FP_ERR_CONFIG, "sweep_and_route_graph: one rank only");
  if (p->flags & (FP_FLAG_KERNEL_TIMING | FP_FLAG_TIME_TRACE))
    return fail(p, FP_ERR_CONFIG, "sweep_and_route_graph: no per-kernel timing inside a graph");
  if (!len || !d_decision || !n_local || is_host_pointer(len) || is_host_pointer(d_decision))
    return fail(p, FP_ERR_INVALID_ARG, "sweep_and_route_graph: device trace and decision buffer, n_local > 0");
  if (route_model >= p->models.size()) return fail(p, FP_ERR_INVALID_ARG, "route_model out of range");
  if (!p->lut_cells) return fail(p, FP_ERR_CONFIG, "sweep_and_route_graph: bin mode needs the LUT");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  auto &G = p->graph;
  auto drop = [&]() {
    for (cudaGraphExec_t &x : G.exec)
      if (x) { cudaGraphExecDestroy(x); x = nullptr; }
    G.valid = false;
  };
  const bool same = G.valid && G.len == len && G.n == n_local && G.rate == rate_rps && G.model == route_model &&
                    G.dec == d_decision && G.bins == p->d_bins && G.spec_buf == p->d_spec;
  if (!same) {
    drop();
    // one eager step: allocates every scratch buffer the step uses (no
    // allocation may happen during capture) and leaves the plan in a state
    // whose bookkeeping (accumulator parity) the graphs reproduce
    fp_status st = sweep_and_route(p, len, n_local, rate_rps, route_model, d_decision, nullptr, nullptr, s);
    if (st != FP_OK) return st;
    if (!p->graph_stream)
      CUDA_TRY(p, cudaStreamCreateWithFlags(&p->graph_stream, cudaStreamNonBlocking), "graph stream");
    // the captures read the plan's device state only when replayed; order the
    // eager step before the first replay on `stream` (it is: same stream)
    for (int q = 0; q < 2; ++q) {
      const uint32_t par = (uint32_t)(p->sweep_seq & 1u);
      const uint64_t l0 = p->launches, s0 = p->spec_calls;
      CUDA_TRY(p, cudaStreamBeginCapture(p->graph_stream, cudaStreamCaptureModeRelaxed), "begin capture");
      fp_status st2 = sweep_and_route(p, len, n_local, rate_rps, route_model, d_decision, nullptr, nullptr,
                                      p->graph_stream);
      cudaGraph_t graph = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(p->graph_stream, &graph);
      if (st2 != FP_OK || ec != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        drop();
        cudaGetLastError();
        // the captured calls advanced the host bookkeeping without running:
        // the histogram copies of both parities are cleared before the next step
        p->parity_clean[0] = p->parity_clean[1] = false;
        p->spec_dirty = true;
        return st2 != FP_OK ? st2 : cuda_fail(p, ec, "end capture");
      }
      const cudaError_t ei = cudaGraphInstantiate(&G.exec[par], graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) {
        drop();
        p->parity_clean[0] = p->parity_clean[1] = false;
        p->spec_dirty = true;
        return cuda_fail(p, ei, "graph instantiate");
      }
      G.launches[par] = p->launches - l0;
      G.spec_n[par] = p->spec_calls - s0;
      p->launches = l0;                 // counted when replayed
      p->spec_calls = s0;
    }
    // the two captures advanced the parity by two: back where the eager step left it
    G.valid = true;
    G.len = len;
    G.n = n_local;
    G.rate = rate_rps;
    G.model = route_model;
    G.dec = d_decision;
    G.bins = p->d_bins;
    G.spec_buf = p->d_spec;
  }
  const uint32_t par = (uint32_t)(p->sweep_seq & 1u);
  // the graphs assume what every completed step leaves behind: this parity's
  // accumulator copies (and the sample's) cleared by the previous step's K3;
  // after a step that failed before its K3, clear them here as the eager call would
  if (!p->parity_clean[par])
    CUDA_TRY(p, cudaMemsetAsync(p->d_hcopies + par * p->copies_elems, 0, p->copies_elems * 8, s), "memset hist");
  if (p->spec_dirty && p->spec_acc) {
    CUDA_TRY(p, cudaMemsetAsync(p->spec_acc, 0, p->copies_elems * 8, s), "memset sample hist");
    p->spec_dirty = false;
  }
  CUDA_TRY(p, cudaGraphLaunch(G.exec[par], s), "graph launch");
  // the bookkeeping of the step the graph replays (sweep_impl / sweep_route_speculative)
  p->parity_clean[par] = false;
  p->parity_clean[par ^ 1u] = true;
  ++p->sweep_seq;
  p->launches += G.launches[par];
  p->spec_calls += G.spec_n[par];
  p->have_sweep = true;
  p->last_stream = s;
  return FP_OK;
}

namespace {
// Validate an estimator and upload its snapshot (c_hat, sigma) to d_calib.
fp_status upload_estimator(fp_plan *p, const fp_estimator *est, cudaStream_t s) {
  if (!est || !est->cats || est->n_cats == 0 || est->n_cats > 256)
    return fail(p, FP_ERR_INVALID_ARG, "estimator needs 1..256 categories");
  if (!std::isfinite(est->gamma) || est->gamma < 0.0 || !std::isfinite(est->c_floor) || !(est->c_floor > 0.0))
    return fail(p, FP_ERR_INVALID_ARG, "estimator needs gamma >= 0 and c_floor > 0 (finite)");
  std::vector<double> v(2 * est->n_cats);
  for (uint32_t k = 0; k < est->n_cats; ++k) {
    if (!std::isfinite(est->cats[k].c_hat) || !std::isfinite(est->cats[k].sigma_hat) || est->cats[k].sigma_hat < 0)
      return fail(p, FP_ERR_INVALID_ARG, "category %u: c_hat finite, sigma_hat finite and >= 0", k);
    v[2 * k] = est->cats[k].c_hat;
    v[2 * k + 1] = est->cats[k].sigma_hat;
  }
  if (!p->d_calib) CUDA_TRY(p, cudaMalloc(&p->d_calib, 512 * sizeof(double)), "cudaMalloc calib");
  // pageable source: staged by the driver before the call returns
  CUDA_TRY(p, cudaMemcpyAsync(p->d_calib, v.data(), v.size() * 8, cudaMemcpyHostToDevice, s), "H2D calib");
  return FP_OK;
}

fp_status check_raw(fp_plan *p, const fp_raw_trace *t, uint64_t n, bool need_true) {
  if (!t) return fail(p, FP_ERR_INVALID_ARG, "raw trace is NULL");
  if (!n) return FP_OK;
  if (!t->body_bytes || !t->max_output_tokens || !t->category)
    return fail(p, FP_ERR_INVALID_ARG, "raw trace columns must be set");
  if (is_host_pointer(t->body_bytes) || is_host_pointer(t->max_output_tokens) || is_host_pointer(t->category) ||
      (need_true && t->true_prompt_tokens && is_host_pointer(t->true_prompt_tokens)))
    return fail(p, FP_ERR_INVALID_ARG, "raw trace columns must be device memory");
  return FP_OK;
}
}  // namespace

fp_status sweep_thresholds_raw(fp_plan *p, const fp_raw_trace *t, uint64_t n_local, const fp_estimator *est,
                               double rate_rps, fp_candidate *h_results, void *stream) {
  if (!p) return FP_ERR_INVALID_ARG;
  fp_status st = check_raw(p, t, n_local, false);
  if (st != FP_OK) return st;
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  st = upload_estimator(p, est, s);
  if (st != FP_OK) return st;
  TraceArgs a = p->ta;
  a.len = nullptr;
  a.n = n_local;
  a.body = t->body_bytes;
  a.maxout = t->max_output_tokens;
  a.cat = t->category;
  a.calib = p->d_calib;
  a.n_cats = est->n_cats;
  a.gamma = est->gamma;
  a.c_floor = est->c_floor;
  return sweep_impl(p, nullptr, n_local, rate_rps, h_results, stream, nullptr, &a);
}

fp_status sweep_and_route_raw(fp_plan *p, const fp_raw_trace *t, uint64_t n_local, const fp_estimator *est,
                              double rate_rps, uint32_t route_model, uint8_t *d_decision, fp_candidate *h_best,
                              fp_route_counts *h_counts, void *stream) {
  if (!p) return FP_ERR_INVALID_ARG;
  fp_status st = check_raw(p, t, n_local, false);
  if (st != FP_OK) return st;
  if (route_model >= p->models.size()) return fail(p, FP_ERR_INVALID_ARG, "route_model out of range");
  if (d_decision && n_local && is_host_pointer(d_decision))
    return fail(p, FP_ERR_INVALID_ARG, "d_decision must be device memory");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  // speculative form: the columns and the decision buffer in the trace pass's
  // vector phase (k1_trace raw_vec; bins + i in the 4-B phase of body + i)
  const uintptr_t b = reinterpret_cast<uintptr_t>(t->body_bytes), m = reinterpret_cast<uintptr_t>(t->max_output_tokens),
                  k = reinterpret_cast<uintptr_t>(t->category);
  const uint64_t head = ((b & 15u) >> 2) ? 4 - ((b & 15u) >> 2) : 0;
  const bool vec = ((b & 3u) == 0) && ((m & 15u) == (b & 15u)) && (((k + head) & 3u) == 0);
  const bool spec = (p->flags & FP_FLAG_SPECULATE) && d_decision && n_local >= (1ull << 26) && vec &&
                    p->lut_cells && p->lut_u8 && p->nbins <= 127 && p->k3a.shape == kK3Cluster &&
                    (reinterpret_cast<uintptr_t>(d_decision + head) & 3u) == 0;
  if (!spec) {
    // sweep, argmin on the host, route with the split
    st = sweep_thresholds_raw(p, t, n_local, est, rate_rps, nullptr, stream);
    if (st != FP_OK) return st;
    std::vector<fp_candidate> best(p->models.size());
    st = best_split(p, best.data());
    if (st != FP_OK) return st;
    if (h_best) memcpy(h_best, best.data(), best.size() * sizeof(fp_candidate));
    const fp_candidate &c = best[route_model];
    if (!(c.flags & FP_CAND_FEASIBLE))
      return fail(p, FP_ERR_STATE, "model %u has no feasible split to route with", route_model);
    return route_batch_raw(p, t, n_local, est, c.b_short, c.c_short, c.c_long, d_decision, nullptr, h_counts, nullptr,
                           stream);
  }
  st = upload_estimator(p, est, s);
  if (st != FP_OK) return st;
  TraceArgs a = p->ta;
  a.len = nullptr;
  a.n = n_local;
  a.body = t->body_bytes;
  a.maxout = t->max_output_tokens;
  a.cat = t->category;
  a.calib = p->d_calib;
  a.n_cats = est->n_cats;
  a.gamma = est->gamma;
  a.c_floor = est->c_floor;
  RouteRawArgs rr{};
  rr.body = t->body_bytes;
  rr.maxout = t->max_output_tokens;
  rr.cat = t->category;
  rr.calib = p->d_calib;
  rr.n_cats = est->n_cats;
  rr.gamma = est->gamma;
  rr.c_floor = est->c_floor;
  rr.decision = d_decision;
  rr.n = n_local;
  return sweep_route_speculative(p, nullptr, n_local, rate_rps, route_model, d_decision, h_best, h_counts, s, &a,
                                 &rr);
}

fp_status route_batch_raw(fp_plan *p, const fp_raw_trace *t, uint64_t n_local, const fp_estimator *est,
                          uint32_t b_short, uint32_t c_short, uint32_t c_long, uint8_t *d_decision,
                          uint32_t *d_l_total, fp_route_counts *h_counts, uint64_t *h_misroute, void *stream) {
  if (!p) return FP_ERR_INVALID_ARG;
  if (!(b_short >= 1 && b_short <= c_short && c_short <= c_long))
    return fail(p, FP_ERR_INVALID_ARG, "need 1 <= B_short <= C_S <= C_L (S:316-321)");
  fp_status st = check_raw(p, t, n_local, true);
  if (st != FP_OK) return st;
  if (n_local && ((d_decision && is_host_pointer(d_decision)) || (d_l_total && is_host_pointer(d_l_total))))
    return fail(p, FP_ERR_INVALID_ARG, "outputs must be device memory");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  st = upload_estimator(p, est, s);
  if (st != FP_OK) return st;
  CUDA_TRY(p, cudaMemsetAsync(p->d_rcounts, 0, 7 * 8, s), "memset counts");
  if (n_local) {
    RouteRawArgs a{};
    a.body = t->body_bytes;
    a.maxout = t->max_output_tokens;
    a.cat = t->category;
    a.true_prompt = t->true_prompt_tokens;
    a.calib = p->d_calib;
    a.n_cats = est->n_cats;
    a.gamma = est->gamma;
    a.c_floor = est->c_floor;
    a.decision = d_decision;
    a.l_total = d_l_total;
    a.n = n_local;
    a.b = b_short;
    a.cs = c_short;
    a.cl = c_long;
    a.g_counts = p->d_rcounts;
    a.g_mis = p->d_rcounts + 5;
    LaunchTimer lt(p, FP_KERNEL_ROUTE, s);
    cudaError_t e = launch_route_raw(a, p->k4_grid, p->k4_block, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "route_batch_raw launch");
    ++p->launches;
  }
  if (p->dist) {
    st = all_reduce_u64(p, p->d_rcounts, 7, s, "all-reduce(route counts)");
    if (st != FP_OK) return st;
  }
  p->last_stream = s;
  if (h_counts || h_misroute) {
    unsigned long long *c = p->h_small + 2ull * p->nbins;
    CUDA_TRY(p, cudaMemcpyAsync(c, p->d_rcounts, 7 * 8, cudaMemcpyDeviceToHost, s), "D2H counts");
    CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
    if (h_counts) {
      h_counts->n_short = c[0];
      h_counts->n_long = c[1];
      h_counts->n_reject = c[2];
      h_counts->mass_short = c[3];
      h_counts->mass_long = c[4];
    }
    if (h_misroute) {
      h_misroute[0] = c[5];
      h_misroute[1] = c[6];
    }
  }
  return FP_OK;
}

namespace {
fp_status sweep_impl(fp_plan *p, const uint32_t *d_len, uint64_t n_local, double rate_rps,
                     fp_candidate *h_results, void *stream, uint32_t *resident, const TraceArgs *raw,
                     uint8_t *bins, uint32_t *route_out, uint32_t route_model, uint8_t *bins_side,
                     uint8_t *bins_hi, const uint32_t *dec_route, unsigned long long *zero2) {
  if (!p) return FP_ERR_INVALID_ARG;
  if (n_local && !d_len && !raw) return fail(p, FP_ERR_INVALID_ARG, "d_len is NULL");
  if (!(rate_rps > 0.0) || !std::isfinite(rate_rps))
    return fail(p, FP_ERR_INVALID_ARG, "rate_rps must be finite and > 0");
  if (!p->dist && n_local == 0) return fail(p, FP_ERR_EMPTY_TRACE, "empty trace (S:170)");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  // this sweep's accumulator parity (its K3 clears the other one for the next sweep)
  const uint32_t par = (uint32_t)(p->sweep_seq & 1u);
  unsigned long long *acc = p->d_hcopies + par * p->copies_elems;
  unsigned long long *other = p->d_hcopies + (par ^ 1u) * p->copies_elems;
  // a memset only when an earlier sweep failed before its K3 ran
  if (!p->parity_clean[par])
    CUDA_TRY(p, cudaMemsetAsync(acc, 0, p->copies_elems * 8, s), "memset hist");
  const bool p2p = (p->flags & FP_FLAG_P2P) != 0;
  if (p2p && !p->p2p_ready) return fail(p, FP_ERR_STATE, "FP_FLAG_P2P plan: call fp_p2p_import first");
  // FP_FLAG_P2P: the step's epoch is committed only once this rank has
  // published it (a failure before that leaves the peers waiting for the same
  // epoch, which a retried sweep then publishes)
  const uint32_t epoch = p2p ? p->p2p_epoch + 1u : 0u;
  p->parity_clean[par] = false;
  fp_status st = FP_OK;
  {
    NvtxRange r("fp:K1 trace pass");
    if (raw) {
      if (n_local) {
        LaunchTimer lt(p, FP_KERNEL_TRACE, s);
        TraceArgs t = *raw;
        t.g_cnt = acc;
        t.g_mass = acc + p->nbins;
        cudaError_t e = launch_trace(t, k1_grid_for(p, n_local), p->k1_block, p->k1_smem, s);
        if (e != cudaSuccess) return cuda_fail(p, e, "trace pass (raw) launch");
        ++p->launches;
      }
    } else st = over_trace(p, d_len, n_local, s, [&](const uint32_t *ptr, uint64_t n, uint64_t off) {
      TraceArgs t = p->ta;
      t.len = ptr;
      t.n = n;
      t.g_cnt = acc;
      t.g_mass = acc + p->nbins;
      // packed bins: this chunk's body starts at global uint4 off / 4 (chunks are
      // whole multiples of 4 elements except the last, and have no head)
      t.bins_out = bins ? bins + (bins_side ? 0 : off) : nullptr;   // packed: device traces (one call, off = 0)
      t.bins_hi = bins_hi;
      t.bins_pack = bins_side ? 1u : 0u;
      t.bins_side = bins_side;
      t.dec_route = dec_route;             // speculative routing: decision bytes into bins_out
      t.pdl = dec_route ? 1u : 0u;
      LaunchTimer lt(p, FP_KERNEL_TRACE, s);
      // packed bins: the grid the routing pass will use (bins_pack: one piece, n_local)
      cudaError_t e = launch_trace(t, k1_grid_for(p, bins_side ? n_local : n), p->k1_block, p->k1_smem, s);
      if (e != cudaSuccess) return cuda_fail(p, e, "trace pass launch");
      ++p->launches;
      return FP_OK;
    }, resident);
  }
  if (st != FP_OK) return st;
  // C1: sum the per-rank histograms. The accumulator copies are folded into
  // one [2][nbins] histogram first (one small kernel), then either published
  // to the peers (FP_FLAG_P2P: K3's prologue reads every rank's over NVLink)
  // or all-reduced (2 (|E| + 1) u64).
  EvalArgs ea = p->ea;
  if (p2p) {
    NvtxRange r("fp:C1 p2p publish");
    unsigned long long *xb = p->d_xbuf + (size_t)(epoch & 1u) * p->xbuf_elems;
    cudaError_t e = launch_fold(acc, p->hist_copies, p->nbins, xb, p->d_xflag, epoch, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "p2p fold/publish launch");
    ++p->launches;
    p->p2p_epoch = epoch;
    ea.peer_hist = p->d_peer_hist;
    ea.peer_flag = p->d_peer_flag;
    ea.p2p_world = (uint32_t)p->world;
    ea.p2p_epoch = epoch;
    ea.p2p_off = (size_t)(epoch & 1u) * p->xbuf_elems;
  } else if (p->dist) {
    NvtxRange r("fp:C1 all-reduce(histogram)");
    cudaError_t e = launch_fold(acc, p->hist_copies, p->nbins, p->d_fold, nullptr, 0, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "fold launch");
    ++p->launches;
    st = all_reduce_u64(p, p->d_fold, 2ull * p->nbins, s, "all-reduce(histogram)");
    if (st != FP_OK) return st;
    ea.hist_cnt = p->d_fold;
    ea.hist_mass = p->d_fold + p->nbins;
    ea.hist_copies = 1;
  } else {
    ea.hist_cnt = acc;
    ea.hist_mass = acc + p->nbins;
  }
  // K2 + K3: scan, evaluate this rank's candidates, per-model argmin
  if (h_results && !p->d_results && p->cand_count)
    CUDA_TRY(p, cudaMalloc(&p->d_results, p->cand_count * sizeof(fp_candidate)), "cudaMalloc results");
  ea.rate = rate_rps;
  ea.results = h_results ? p->d_results : nullptr;
  ea.zero_copies = other;
  ea.zero_elems = p->copies_elems;
  ea.zero_copies2 = zero2;
  ea.route_out = route_out;
  ea.route_model = route_model;
  cudaError_t e;
  {
    NvtxRange r("fp:K3 candidate evaluation");
    LaunchTimer lt(p, FP_KERNEL_EVAL, s);
    e = launch_eval(ea, h_results ? p->k3r : p->k3a, s);
  }
  if (e != cudaSuccess) return cuda_fail(p, e, "candidate evaluation launch");
  p->parity_clean[par ^ 1u] = true;        // K3 zeroes them (stream-ordered)
  ++p->sweep_seq;
  ++p->launches;
  // C2: gather every rank's per-model best
  if (p->dist && !(p->flags & FP_FLAG_REPLICATED_GRID)) {
    NvtxRange r("fp:C2 all-gather(best)");
    const size_t bytes = p->models.size() * sizeof(fp_candidate);
    st = all_gather_bytes(p, p->d_best + (size_t)p->rank * p->models.size(), p->d_best, bytes, s,
                          "all-gather(best)");
    if (st != FP_OK) return st;
  }
  p->have_sweep = true;
  p->last_stream = s;
  if (h_results && p->cand_count) {
    CUDA_TRY(p, cudaMemcpyAsync(h_results, p->d_results, p->cand_count * sizeof(fp_candidate),
                                cudaMemcpyDeviceToHost, s),
             "D2H results");
    CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
    if (p2p) return check_device_error(p);
  }
  return FP_OK;
}

}  // namespace

fp_status sweep_three_pools(fp_plan *p, double rate_rps, fp_pool3_candidate *h_results,
                            fp_pool3_candidate *h_best, void *stream) {
  if (!p || !h_best) return FP_ERR_INVALID_ARG;
  if (!p->have_sweep) return fail(p, FP_ERR_STATE, "sweep_three_pools before a sweep");
  if (!(rate_rps > 0.0) || !std::isfinite(rate_rps))
    return fail(p, FP_ERR_INVALID_ARG, "rate_rps must be finite and > 0");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t nb = (uint32_t)p->b.size(), M = (uint32_t)p->models.size();
  if (!p->d_p3) {
    if (nb < 2 || nb > 4096) return fail(p, FP_ERR_CONFIG, "three pools need 2 <= n_b <= 4096");
    std::vector<uint16_t> bw(nb);
    for (uint32_t k = 0; k < nb; ++k) {
      uint32_t w = index_of(p->windows, p->b[k]);
      if (w == UINT32_MAX) return fail(p, FP_ERR_CONFIG, "B %u missing from windows (three pools)", p->b[k]);
      bw[k] = (uint16_t)w;
    }
    std::vector<uint32_t> pairs;
    pairs.reserve((size_t)nb * (nb - 1) / 2);
    for (uint32_t i = 0; i < nb; ++i)
      for (uint32_t j = i + 1; j < nb; ++j) pairs.push_back(i | (j << 16));
    const uint64_t per = (uint64_t)p->gpus.size() * p->cl.size() * pairs.size();
    if (per * M >= 0xffffffffull) return fail(p, FP_ERR_CONFIG, "three-pool grid has >= 2^32 candidates");
    p->k3p_grid_x = (int)std::min<uint64_t>(std::max<uint64_t>(1, (uint64_t)p->sm_count * 8 / M),
                                            std::max<uint64_t>(1, (per + 255) / 256));
    const size_t off_bw = pairs.size() * 4;
    const size_t off_best = (off_bw + nb * 2 + 15) & ~size_t(15);
    const size_t off_bb = off_best + M * sizeof(fp_pool3_candidate);
    const size_t off_done = off_bb + (size_t)M * p->k3p_grid_x * sizeof(BlockBest);
    const size_t bytes = off_done + M * sizeof(unsigned int);
    CUDA_TRY(p, cudaMalloc(&p->d_p3, bytes), "cudaMalloc three-pool state");
    CUDA_TRY(p, cudaMemcpy(p->d_p3, pairs.data(), pairs.size() * 4, cudaMemcpyHostToDevice), "H2D pairs");
    CUDA_TRY(p, cudaMemcpy(p->d_p3 + off_bw, bw.data(), nb * 2, cudaMemcpyHostToDevice), "H2D b_win3");
    CUDA_TRY(p, cudaMemset(p->d_p3 + off_done, 0, M * sizeof(unsigned int)), "memset done3");
    p->ea3 = p->ea;
    // the last sweep's summed histogram (K3 of that sweep published it)
    p->ea3.hist_cnt = p->d_hist;
    p->ea3.hist_mass = p->d_hist + p->nbins;
    p->ea3.hist_copies = 1;
    p->ea3.hist_out = nullptr;
    p->ea3.zero_copies = nullptr;
    p->ea3.p2p_world = 0;
    p->ea3.pairs = reinterpret_cast<const uint32_t *>(p->d_p3);
    p->ea3.n_pairs = (uint32_t)pairs.size();
    p->ea3.b_win3 = reinterpret_cast<const uint16_t *>(p->d_p3 + off_bw);
    p->ea3.per_model3 = per;
    p->ea3.best3 = reinterpret_cast<fp_pool3_candidate *>(p->d_p3 + off_best);
    p->ea3.block_best3 = reinterpret_cast<BlockBest *>(p->d_p3 + off_bb);
    p->ea3.done3 = reinterpret_cast<unsigned int *>(p->d_p3 + off_done);
    p->n_cand3 = per * M;
  }
  if (h_results && !p->d_results3)
    CUDA_TRY(p, cudaMalloc(&p->d_results3, p->n_cand3 * sizeof(fp_pool3_candidate)), "cudaMalloc results3");
  // the last sweep's histogram was written on last_stream: order this call after it
  if (p->last_stream != s) {
    if (!p->ev_order) CUDA_TRY(p, cudaEventCreateWithFlags(&p->ev_order, cudaEventDisableTiming), "event");
    CUDA_TRY(p, cudaEventRecord(p->ev_order, p->last_stream), "record order");
    CUDA_TRY(p, cudaStreamWaitEvent(s, p->ev_order, 0), "wait order");
  }
  EvalArgs ea = p->ea3;
  ea.rate = rate_rps;
  ea.results3 = h_results ? p->d_results3 : nullptr;
  {
    LaunchTimer lt(p, FP_KERNEL_EVAL, s);
    cudaError_t e = launch_eval3(ea, p->k3p_grid_x, 256, p->k3_smem, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "three-pool evaluation launch");
  }
  ++p->launches;
  CUDA_TRY(p, cudaMemcpyAsync(h_best, ea.best3, M * sizeof(fp_pool3_candidate), cudaMemcpyDeviceToHost, s),
           "D2H best3");
  if (h_results)
    CUDA_TRY(p, cudaMemcpyAsync(h_results, p->d_results3, p->n_cand3 * sizeof(fp_pool3_candidate),
                                cudaMemcpyDeviceToHost, s), "D2H results3");
  CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
  return FP_OK;
}

namespace {
struct HostAff {
  double a = 1.0, b = 0.0;
  uint64_t n = 0;
};
// e first, then l (as the device's compose)
HostAff host_compose(const HostAff &e, const HostAff &l) {
  return HostAff{l.a * e.a, std::fma(l.a, e.b, l.b), e.n + l.n};
}

fp_status ensure_xch(fp_plan *p) {
  if (!p->d_xch) CUDA_TRY(p, cudaMalloc(&p->d_xch, (size_t)(p->world + 1) * 512), "cudaMalloc exchange");
  return FP_OK;
}
}  // namespace

fp_status calibrate_replay(fp_plan *p, const uint32_t *d_body_bytes, const uint32_t *d_prompt_tokens,
                           const uint8_t *d_category, uint64_t n, uint32_t n_cats, double beta,
                           const fp_category_calibration *init, uint64_t snap_at,
                           fp_category_calibration *h_final, uint64_t *h_n_obs,
                           fp_category_calibration *h_snap, void *stream) {
  if (!p || !init || !h_final || !h_n_obs) return FP_ERR_INVALID_ARG;
  if (n_cats < 1 || n_cats > 16) return fail(p, FP_ERR_INVALID_ARG, "calibrate_replay needs 1 <= n_cats <= 16");
  if (!(beta > 0.0 && beta < 1.0)) return fail(p, FP_ERR_INVALID_ARG, "beta must be in (0, 1)");
  for (uint32_t k = 0; k < n_cats; ++k)
    if (!std::isfinite(init[k].c_hat) || !std::isfinite(init[k].sigma_hat))
      return fail(p, FP_ERR_INVALID_ARG, "initial state must be finite");
  // a rank-specific failure is exchanged (world > 1) so that all ranks fail together
  const bool bad = n && (!d_body_bytes || !d_prompt_tokens || !d_category || is_host_pointer(d_body_bytes) ||
                         is_host_pointer(d_prompt_tokens) || is_host_pointer(d_category));
  if (bad && !p->dist) return fail(p, FP_ERR_INVALID_ARG, "feedback columns must be device memory");
  if (bad) n = 0;
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int stream_bps = (!p->dist && n_cats <= 4 && n > 0 && env_int("FP_CALIB_STREAM", 0))
                             ? calib_stream_blocks_per_sm() : 0;
  if (stream_bps > 0) {
    // one rank, n_cats <= 4, FP_CALIB_STREAM=1: the streaming replay (k_calib.cu
    // c_stream) -- every record read from HBM once, c_obs computed once, no
    // per-record category dispatch. Correct, but slower than the two-pass
    // kernels below on a B200 (17.5 vs 4.7 ms per 1e9 records: each iteration
    // is a chain of latencies -- column loads, fence + chunk counter, the
    // chunk scanner's hand-off -- with two CTAs per SM to hide them;
    // profiles/r02/next3_stream_profile.log).
    const uint32_t G = (uint32_t)std::min<int64_t>(512, (int64_t)stream_bps * p->sm_count);
    const uint64_t chunk = (uint64_t)G * calib_stream_piece();
    const uint64_t nch = (n + chunk - 1) / chunk;
    if (env_int("FP_CALIB_VERBOSE", 0))
      fprintf(stderr, "[fp] calibrate_replay: streaming kernel, %d CTAs/SM, G = %u, %llu chunks of %llu records\n",
              stream_bps, G, (unsigned long long)nch, (unsigned long long)chunk);
    const uint64_t np = nch * G * 4;                          // (piece, category) entries
    const size_t flag_bytes = ((2 * nch + 9) * 4 + 255) & ~size_t(255);
    const size_t fin = (size_t)4 * (calib_stream_fin_blocks() + 1) * 24;
    const bool prof = env_int("FP_CALIB_PROFILE", 0) != 0;
    const size_t prof_bytes = prof ? (2 * nch + 2) * 64 : 0;
    const size_t need = 16 * 16 * 8 + flag_bytes + np * (24 + 8 + 8 + 8 + 8) + (nch + 1) * 4 * 16 + fin + prof_bytes + 256;
    if (p->calib_cap < need) {
      cudaFree(p->d_calib_scratch);
      p->d_calib_scratch = nullptr;
      p->calib_cap = 0;
      CUDA_TRY(p, cudaMalloc(&p->d_calib_scratch, need), "cudaMalloc calibration scratch");
      p->calib_cap = need;
    }
    unsigned char *base = p->d_calib_scratch;
    double *sm = reinterpret_cast<double *>(base);                       // 16 slots of 16 doubles
    unsigned int *flags = reinterpret_cast<unsigned int *>(base + 16 * 16 * 8);
    unsigned char *q = base + 16 * 16 * 8 + flag_bytes;
    CalibStreamArgs a{};
    a.bytes = d_body_bytes;
    a.tokens = d_prompt_tokens;
    a.cat = d_category;
    a.n = n;
    a.n_cats = n_cats;
    a.beta = beta;
    a.G = G;
    a.n_chunks = (uint32_t)nch;
    a.done = flags;
    a.ready = flags + nch;
    a.cagg = q;                                      q += np * 24;
    a.pstate_c = reinterpret_cast<double *>(q);      q += np * 8;
    a.pstate_n = reinterpret_cast<unsigned long long *>(q); q += np * 8;
    a.sig_a = reinterpret_cast<double *>(q);         q += np * 8;
    a.sig_b = reinterpret_cast<double *>(q);         q += np * 8;
    a.cstart_c = reinterpret_cast<double *>(q);      q += (nch + 1) * 4 * 8;
    a.cstart_n = reinterpret_cast<unsigned long long *>(q); q += (nch + 1) * 4 * 8;
    a.fin_part = q;                                  q += (size_t)4 * calib_stream_fin_blocks() * 24;
    a.fin_pre = q;                                   q += 4 * 24;
    a.prof = prof ? reinterpret_cast<unsigned long long *>(q) : nullptr;
    a.fin_done = flags + 2 * nch + 1;
    a.fin_snapb = flags + 2 * nch + 5;
    double *c0 = sm + 16 * 8, *s0 = sm + 16 * 9;
    a.c0 = c0;
    a.s0 = s0;
    a.snap_piece = reinterpret_cast<unsigned long long *>(sm + 16 * 10);
    a.snap_v = sm + 16 * 11;
    a.snap_at = snap_at;
    a.out = sm;
    std::vector<double> init_c(16, 0.0), init_s(16, 0.0), outv(80, 0.0);
    for (uint32_t k = 0; k < n_cats; ++k) {
      init_c[k] = init[k].c_hat;
      init_s[k] = init[k].sigma_hat;
    }
    for (int k = 48; k < 80; ++k) outv[k] = std::nan("");
    CUDA_TRY(p, cudaMemcpyAsync(c0, init_c.data(), 16 * 8, cudaMemcpyHostToDevice, s), "H2D init");
    CUDA_TRY(p, cudaMemcpyAsync(s0, init_s.data(), 16 * 8, cudaMemcpyHostToDevice, s), "H2D init");
    CUDA_TRY(p, cudaMemcpyAsync(sm, outv.data(), 80 * 8, cudaMemcpyHostToDevice, s), "H2D outputs");
    CUDA_TRY(p, cudaMemsetAsync(a.snap_piece, 0xFF, 4 * 8, s), "memset snapshot pieces");
    CUDA_TRY(p, cudaMemsetAsync(flags, 0, (2 * nch + 9) * 4, s), "memset chunk flags");
    {
      LaunchTimer lt(p, FP_KERNEL_EVAL, s);
      cudaError_t e = launch_calib_stream(a, s);
      if (e != cudaSuccess) return cuda_fail(p, e, "calibration replay launch");
    }
    p->launches += 2;
    if (prof) {
      std::vector<unsigned long long> t((2 * nch + 2) * 8);
      CUDA_TRY(p, cudaMemcpyAsync(t.data(), a.prof, t.size() * 8, cudaMemcpyDeviceToHost, s), "D2H profile");
      CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
      double sc[3] = {0, 0, 0}, it[5] = {0, 0, 0, 0, 0};
      for (uint64_t i = 1; i + 1 < nch; ++i)
        for (int j = 0; j < 3; ++j) sc[j] += (double)(t[i * 8 + j + 1] - t[i * 8 + j]);
      uint64_t m = 0;
      for (uint64_t i = 2; i + 2 < nch; ++i, ++m) {
        const unsigned long long *r = &t[(nch + i) * 8];
        it[0] += (double)(r[1] - r[0]); it[1] += (double)(r[2] - r[1]); it[2] += (double)(r[3] - r[2]);
        it[3] += (double)(r[4] - r[3]); it[4] += (double)(r[5] - r[4]);
      }
      const double ns = (double)std::max<uint64_t>(1, nch - 2), nm = (double)std::max<uint64_t>(1, m);
      fprintf(stderr, "[fp] c_stream scanner ns: scan %.0f wait %.0f publish %.0f | CTA 0 iteration ns: A %.0f "
              "scan %.0f gap %.0f C-wait %.0f C %.0f | total %.3f ms\n", sc[0] / ns, sc[1] / ns, sc[2] / ns,
              it[0] / nm, it[1] / nm, it[2] / nm, it[3] / nm, it[4] / nm,
              (double)(t[(2 * nch + 1) * 8 + 5] - t[nch * 8]) * 1e-6);
    }
    std::vector<double> h(80);
    CUDA_TRY(p, cudaMemcpyAsync(h.data(), sm, 80 * 8, cudaMemcpyDeviceToHost, s), "D2H calibration");
    CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
    for (uint32_t k = 0; k < n_cats; ++k) {
      uint64_t nobs;
      memcpy(&nobs, &h[32 + k], 8);
      h_final[k].c_hat = h[k];
      h_final[k].sigma_hat = h[16 + k];
      h_n_obs[k] = nobs;
      if (h_snap) {
        h_snap[k].c_hat = h[48 + k];
        h_snap[k].sigma_hat = h[64 + k];
      }
    }
    return FP_OK;
  }
  // one contiguous segment per thread (a multiple of 16 records), one resident wave
  const int bps = calib_blocks_per_sm(n_cats);
  if (bps < 1) return fail(p, FP_ERR_CUDA, "calibration kernels do not fit an SM");
  const uint64_t max_blocks = (uint64_t)p->sm_count * bps;
  // (segments stay below 65,536 records: the n_cats <= 4 kernels pack 16-bit counters)
  const uint64_t blocks = std::max<uint64_t>({1, std::min<uint64_t>(max_blocks, (n + 256 * 64 - 1) / (256 * 64)),
                                              (n + 256ull * 65520 - 1) / (256ull * 65520)});
  const uint64_t threads = blocks * 256;
  const uint64_t seg = std::max<uint64_t>(16, ((n + threads - 1) / threads + 15) / 16 * 16);
  const size_t scratch = calib_scratch_bytes(blocks, n_cats);
  const size_t small = 16 * 16 * 8;
  if (p->calib_cap < scratch + small) {
    cudaFree(p->d_calib_scratch);
    p->d_calib_scratch = nullptr;
    p->calib_cap = 0;
    CUDA_TRY(p, cudaMalloc(&p->d_calib_scratch, scratch + small), "cudaMalloc calibration scratch");
    p->calib_cap = scratch + small;
  }
  unsigned char *base = p->d_calib_scratch;
  const uint64_t KT = (uint64_t)n_cats * threads, KB = (uint64_t)n_cats * blocks;
  CalibArgs a{};
  a.bytes = d_body_bytes;
  a.tokens = d_prompt_tokens;
  a.cat = d_category;
  a.n = n;
  a.n_cats = n_cats;
  a.beta = beta;
  a.threads = threads;
  a.blocks = blocks;
  a.seg = seg;
  a.thrA = reinterpret_cast<double *>(base);
  a.thrB = a.thrA + KT;
  a.blkA = a.thrB + KT;
  a.blkB = a.blkA + KB;
  a.sblkA = a.blkB + KB;
  a.sblkB = a.sblkA + KB;
  a.blkN = reinterpret_cast<unsigned long long *>(a.sblkB + KB);
  a.thrN = reinterpret_cast<uint32_t *>(a.blkN + KB);
  a.thrC = a.thrN + KT;
  // 16 slots of 16 doubles; slots 3-5 and 10-13 / 14-15 are the exchange records
  double *sm = reinterpret_cast<double *>(base + scratch);
  auto slot = [&](int i) { return sm + 16 * i; };
  a.totA = slot(0);
  a.totSA = slot(1);
  a.totN = reinterpret_cast<unsigned long long *>(slot(2));
  a.snap_c = slot(3);
  a.snap_s = slot(4);
  a.snap_block = reinterpret_cast<unsigned long long *>(slot(5));
  a.snap_sa = slot(6);
  a.snap_sb = slot(7);
  double *c0 = slot(8), *s0 = slot(9);
  a.c0 = c0;
  a.s0 = s0;
  a.mapA = slot(10);
  a.mapB = slot(11);
  a.mapN = reinterpret_cast<unsigned long long *>(slot(12));
  double *flag = slot(13);
  a.smapA = slot(14);
  a.smapB = slot(15);
  a.snap_at = snap_at;
  a.vec_bt = !(((uintptr_t)d_body_bytes | (uintptr_t)d_prompt_tokens) & 15);
  a.vec_c = !((uintptr_t)d_category & 15);
  std::vector<double> init_c(16, 0.0), init_s(16, 0.0);
  for (uint32_t k = 0; k < n_cats; ++k) { init_c[k] = init[k].c_hat; init_s[k] = init[k].sigma_hat; }
  CUDA_TRY(p, cudaMemcpyAsync(c0, init_c.data(), 16 * 8, cudaMemcpyHostToDevice, s), "H2D init");
  CUDA_TRY(p, cudaMemcpyAsync(s0, init_s.data(), 16 * 8, cudaMemcpyHostToDevice, s), "H2D init");
  // snapshots start as NaN (all-ones bytes), no snapshot block (~0)
  CUDA_TRY(p, cudaMemsetAsync(a.snap_c, 0xFF, 48 * 8, s), "memset snapshots");
  if (!p->dist) {
    {
      LaunchTimer lt(p, FP_KERNEL_EVAL, s);
      cudaError_t e = launch_calibrate(a, s);
      if (e != cudaSuccess) return cuda_fail(p, e, "calibration replay launch");
    }
    p->launches += 5;
    std::vector<double> h(96);
    CUDA_TRY(p, cudaMemcpyAsync(h.data(), sm, 96 * 8, cudaMemcpyDeviceToHost, s), "D2H calibration");
    CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
    for (uint32_t k = 0; k < n_cats; ++k) {
      uint64_t nobs;
      memcpy(&nobs, &h[32 + k], 8);
      h_final[k].c_hat = h[k];
      h_final[k].sigma_hat = h[16 + k];
      h_n_obs[k] = nobs;
      if (h_snap) {
        h_snap[k].c_hat = h[48 + k];
        h_snap[k].sigma_hat = h[64 + k];
      }
    }
    return FP_OK;
  }

  // world > 1: the stream is sharded in order over the ranks (rank r holds the
  // r-th contiguous piece). Each rank composes its piece's maps; an all-gather
  // gives every rank the maps of the ranks before it, hence its start state
  // and the observations that precede it; the same for the sigma maps.
  fp_status st = ensure_xch(p);
  if (st != FP_OK) return st;
  const int W = p->world, R = p->rank;
  const double flagv = bad ? 1.0 : 0.0;
  CUDA_TRY(p, cudaMemcpyAsync(flag, &flagv, 8, cudaMemcpyHostToDevice, s), "H2D flag");
  {
    LaunchTimer lt(p, FP_KERNEL_EVAL, s);
    cudaError_t e = launch_calib_maps(a, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "calibration maps launch");
  }
  st = all_gather_bytes(p, slot(10), p->d_xch, 64 * 8, s, "all-gather(calibration maps)");
  if (st != FP_OK) return st;
  std::vector<double> g1((size_t)W * 64);
  CUDA_TRY(p, cudaMemcpyAsync(g1.data(), p->d_xch, g1.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
  CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
  for (int r = 0; r < W; ++r)
    if (g1[64 * r + 48] != 0.0) return fail(p, FP_ERR_INVALID_ARG, "feedback columns must be device memory");
  auto map_of = [&](const std::vector<double> &g, int r, uint32_t k, bool with_n) {
    HostAff m;
    m.a = g[(size_t)r * 64 + k];
    m.b = g[(size_t)r * 64 + 16 + k];
    if (with_n) memcpy(&m.n, &g[(size_t)r * 64 + 32 + k], 8);
    return m;
  };
  std::vector<double> c0r(16, 0.0), s0r(16, 0.0);
  for (uint32_t k = 0; k < n_cats; ++k) {
    HostAff pre, tot;
    for (int r = 0; r < W; ++r) {
      if (r == R) pre = tot;
      tot = host_compose(tot, map_of(g1, r, k, true));
    }
    c0r[k] = std::fma(pre.a, init_c[k], pre.b);
    a.snap_off[k] = pre.n;
    h_final[k].c_hat = std::fma(tot.a, init_c[k], tot.b);
    h_n_obs[k] = tot.n;
  }
  CUDA_TRY(p, cudaMemcpyAsync(c0, c0r.data(), 16 * 8, cudaMemcpyHostToDevice, s), "H2D rank start");
  {
    LaunchTimer lt(p, FP_KERNEL_EVAL, s);
    cudaError_t e = launch_calib_replay(a, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "calibration replay launch");
  }
  st = all_gather_bytes(p, slot(14), p->d_xch, 32 * 8, s, "all-gather(sigma maps)");
  if (st != FP_OK) return st;
  std::vector<double> g2((size_t)W * 32);
  CUDA_TRY(p, cudaMemcpyAsync(g2.data(), p->d_xch, g2.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
  CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
  for (uint32_t k = 0; k < n_cats; ++k) {
    HostAff pre, tot;
    for (int r = 0; r < W; ++r) {
      if (r == R) pre = tot;
      tot = host_compose(tot, HostAff{g2[(size_t)r * 32 + k], g2[(size_t)r * 32 + 16 + k], 0});
    }
    s0r[k] = std::fma(pre.a, init_s[k], pre.b);
    h_final[k].sigma_hat = std::fma(tot.a, init_s[k], tot.b);
  }
  CUDA_TRY(p, cudaMemcpyAsync(s0, s0r.data(), 16 * 8, cudaMemcpyHostToDevice, s), "H2D rank sigma start");
  {
    LaunchTimer lt(p, FP_KERNEL_EVAL, s);
    cudaError_t e = launch_calib_snap(a, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "calibration snapshot launch");
  }
  p->launches += 5;
  st = all_gather_bytes(p, slot(3), p->d_xch, 48 * 8, s, "all-gather(snapshots)");
  if (st != FP_OK) return st;
  std::vector<double> g3((size_t)W * 48);
  CUDA_TRY(p, cudaMemcpyAsync(g3.data(), p->d_xch, g3.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
  CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
  if (h_snap)
    for (uint32_t k = 0; k < n_cats; ++k) {
      h_snap[k].c_hat = std::nan("");
      h_snap[k].sigma_hat = std::nan("");
      for (int r = 0; r < W; ++r) {
        uint64_t blk;
        memcpy(&blk, &g3[(size_t)r * 48 + 32 + k], 8);
        if (blk != ~0ull) {
          h_snap[k].c_hat = g3[(size_t)r * 48 + k];
          h_snap[k].sigma_hat = g3[(size_t)r * 48 + 16 + k];
        }
      }
    }
  return FP_OK;
}

fp_status sweep_peak_windows(fp_plan *p, const uint32_t *d_len, const uint64_t *d_arrival_ns, uint64_t n_local,
                             uint64_t window_ns, fp_peak_candidate *h_results, fp_peak_candidate *h_best,
                             void *stream) {
  if (!p || !h_best) return FP_ERR_INVALID_ARG;
  // checks every rank takes identically come first; rank-specific ones are
  // exchanged below so that all ranks fail together (no rank left waiting)
  if (window_ns == 0) return fail(p, FP_ERR_INVALID_ARG, "window_ns must be > 0");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t *ends = reinterpret_cast<uint64_t *>(p->h_small);
  uint64_t bad = 0;
  if (n_local && (!d_len || !d_arrival_ns || is_host_pointer(d_len) || is_host_pointer(d_arrival_ns)))
    bad = 1;
  else if (n_local && (((uintptr_t)d_len & 3) || ((uintptr_t)d_arrival_ns & 7)))
    bad = 2;
  uint64_t first = 0, last = 0;
  if (!bad && n_local) {
    CUDA_TRY(p, cudaMemcpyAsync(ends, d_arrival_ns, 8, cudaMemcpyDeviceToHost, s), "D2H first arrival");
    CUDA_TRY(p, cudaMemcpyAsync(ends + 1, d_arrival_ns + (n_local - 1), 8, cudaMemcpyDeviceToHost, s),
             "D2H last arrival");
    CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
    first = ends[0];
    last = ends[1];
    if (first > last) bad = 3;
  }
  // global extent: every rank's (bad, n_local, last)
  uint64_t n_total = n_local, last_all = last, bad_all = bad;
  if (p->dist) {
    fp_status st = ensure_xch(p);
    if (st != FP_OK) return st;
    const uint64_t mine[4] = {bad, n_local, last, 0};
    CUDA_TRY(p, cudaMemcpyAsync(p->d_xch, mine, 32, cudaMemcpyHostToDevice, s), "H2D exchange");
    st = all_gather_bytes(p, p->d_xch, p->d_xch + 4, 32, s, "all-gather(peak extents)");
    if (st != FP_OK) return st;
    std::vector<uint64_t> all(4 * (size_t)p->world);
    CUDA_TRY(p, cudaMemcpyAsync(all.data(), p->d_xch + 4, all.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
    CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
    n_total = 0;
    last_all = 0;
    bad_all = 0;
    for (int r = 0; r < p->world; ++r) {
      bad_all = std::max<uint64_t>(bad_all, all[4 * r]);
      n_total += all[4 * r + 1];
      if (all[4 * r + 1]) last_all = std::max<uint64_t>(last_all, all[4 * r + 2]);
    }
  }
  if (bad_all == 1) return fail(p, FP_ERR_INVALID_ARG, "length and arrival columns must be device memory");
  if (bad_all == 2) return fail(p, FP_ERR_INVALID_ARG, "misaligned column");
  if (bad_all == 3) return fail(p, FP_ERR_INVALID_ARG, "arrivals not in order (first > last)");
  if (n_total == 0) return fail(p, FP_ERR_EMPTY_TRACE, "empty trace");
  if (n_total > 0xffffffffull) return fail(p, FP_ERR_INVALID_ARG, "trace must be < 2^32 requests (u32 window counters)");
  if (last_all > ~0ull - window_ns) return fail(p, FP_ERR_INVALID_ARG, "arrival + window_ns overflows");
  const uint64_t n_twin = last_all / window_ns + 1;
  const size_t hbytes = (size_t)n_twin * p->nbins * 4;
  if (n_twin > (1ull << 26) || hbytes > (4ull << 30))
    return fail(p, FP_ERR_INVALID_ARG, "%llu windows x %u bins is too many", (unsigned long long)n_twin, p->nbins);
  const uint32_t M = (uint32_t)p->models.size();
  const uint32_t n_b = (uint32_t)p->b.size(), n_cl = (uint32_t)p->cl.size();
  const int grid_x = (int)std::min<uint64_t>(std::max<uint64_t>(1, (uint64_t)p->sm_count * 8 / M),
                                             std::max<uint64_t>(1, (p->per_model + 255) / 256));
  // scratch: [hist2d | colmax | pairmax | error] (zeroed together), start, best, block bests, done
  const size_t zbytes = ((hbytes + ((size_t)p->nbins + (size_t)n_b * n_cl + 1) * 4) + 15) & ~size_t(15);
  const size_t sbytes = (n_twin + 1) * 8;
  const size_t need = zbytes + sbytes + M * sizeof(fp_peak_candidate) + (size_t)M * grid_x * sizeof(BlockBest) +
                      M * sizeof(unsigned int) + 64;
  if (p->peak_cap < need) {
    cudaFree(p->d_peak);
    p->d_peak = nullptr;
    p->peak_cap = 0;
    CUDA_TRY(p, cudaMalloc(&p->d_peak, need), "cudaMalloc peak scratch");
    p->peak_cap = need;
  }
  unsigned char *base = p->d_peak;
  uint32_t *hist2d = reinterpret_cast<uint32_t *>(base);
  uint32_t *colmax = hist2d + (size_t)n_twin * p->nbins;
  uint32_t *pairmax = colmax + p->nbins;
  unsigned int *err = pairmax + (size_t)n_b * n_cl;
  size_t off = zbytes;
  uint64_t *start = reinterpret_cast<uint64_t *>(base + off);
  off += (sbytes + 15) & ~size_t(15);
  fp_peak_candidate *best = reinterpret_cast<fp_peak_candidate *>(base + off);
  off += M * sizeof(fp_peak_candidate);
  BlockBest *bb = reinterpret_cast<BlockBest *>(base + off);
  off += (size_t)M * grid_x * sizeof(BlockBest);
  unsigned int *done = reinterpret_cast<unsigned int *>(base + off);
  CUDA_TRY(p, cudaMemsetAsync(hist2d, 0, zbytes, s), "memset hist2d");
  CUDA_TRY(p, cudaMemsetAsync(done, 0, M * sizeof(unsigned int), s), "memset done");
  PeakArgs pa{};
  pa.len = d_len;
  pa.arrival = d_arrival_ns;
  pa.n = n_local;
  pa.window_ns = window_ns;
  pa.n_windows = n_twin;
  pa.start = start;
  pa.lut = p->ta.lut;
  pa.edges = p->ta.edges;
  pa.lut_cells = p->lut_cells;
  pa.lutw = p->lut_cells ? (p->lut_u8 ? 1 : 2) : 0;
  pa.clampv = p->max_edge + 1u;
  pa.round = (1u << p->shift) - 1u;
  pa.shift = p->shift;
  pa.nbins = p->nbins;
  pa.hist2d = hist2d;
  pa.b_edge = p->ea.b_edge;
  pa.cl_edge = p->ea.cl_edge;
  pa.n_b = n_b;
  pa.n_cl = n_cl;
  pa.colmax = colmax;
  pa.pairmax = pairmax;
  pa.error = err;
  pa.check_order = (p->flags & FP_FLAG_CHECK_ORDER) != 0;
  {
    const size_t fixed = ((size_t)n_b * n_cl + p->nbins) * 4;
    const size_t budget = 96 * 1024;
    if (fixed + (size_t)p->nbins * 4 > 200 * 1024) return fail(p, FP_ERR_CONFIG, "too many (B, C_L) pairs");
    pa.rows = (uint32_t)std::max<size_t>(1, std::min<size_t>(64, (budget > fixed ? budget - fixed : 0) /
                                                                     ((size_t)p->nbins * 4)));
  }
  if (peak_smem_bytes(pa) > 200 * 1024) return fail(p, FP_ERR_CONFIG, "peak LUT too large");
  {
    LaunchTimer lt(p, FP_KERNEL_TRACE, s);
    cudaError_t e = n_local ? launch_peak_hist(pa, p->sm_count, s) : cudaSuccess;
    if (e != cudaSuccess) return cuda_fail(p, e, "peak histogram launch");
  }
  if (n_local) p->launches += pa.check_order ? 3 : 2;
  if (p->dist) {
    // global windows: sum the per-rank 2-D histograms (and order-check flags)
    fp_status st = all_reduce_u32(p, hist2d, zbytes / 4, s, "all-reduce(window histogram)");
    if (st != FP_OK) return st;
  }
  {
    LaunchTimer lt(p, FP_KERNEL_TRACE, s);
    cudaError_t e = launch_peak_scan(pa, p->sm_count, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "peak scan launch");
  }
  ++p->launches;
  EvalArgs ea = p->ea;
  ea.colmax_pk = colmax;
  ea.pairmax_pk = pairmax;
  ea.inv_w_s = 1e9 / (double)window_ns;
  ea.best_pk = best;
  ea.block_best_pk = bb;
  ea.done_pk = done;
  if (h_results && !p->d_results_pk)
    CUDA_TRY(p, cudaMalloc(&p->d_results_pk, p->n_cand * sizeof(fp_peak_candidate)), "cudaMalloc peak results");
  ea.results_pk = h_results ? p->d_results_pk : nullptr;
  {
    LaunchTimer lt(p, FP_KERNEL_EVAL, s);
    cudaError_t e = launch_eval_peak(ea, grid_x, 256, s);
    if (e != cudaSuccess) return cuda_fail(p, e, "peak evaluation launch");
  }
  ++p->launches;
  unsigned int *herr = reinterpret_cast<unsigned int *>(ends);
  CUDA_TRY(p, cudaMemcpyAsync(herr, err, 4, cudaMemcpyDeviceToHost, s), "D2H error flag");
  CUDA_TRY(p, cudaMemcpyAsync(h_best, best, M * sizeof(fp_peak_candidate), cudaMemcpyDeviceToHost, s), "D2H best");
  if (h_results)
    CUDA_TRY(p, cudaMemcpyAsync(h_results, p->d_results_pk, p->n_cand * sizeof(fp_peak_candidate),
                                cudaMemcpyDeviceToHost, s), "D2H peak results");
  CUDA_TRY(p, cudaStreamSynchronize(s), "sync");
  if (*herr) return fail(p, FP_ERR_INVALID_ARG, "arrivals not in order (FP_FLAG_CHECK_ORDER)");
  return FP_OK;
}

fp_status best_split(fp_plan *p, fp_candidate *h_best) {
  if (!p || !h_best) return FP_ERR_INVALID_ARG;
  if (!p->have_sweep) return fail(p, FP_ERR_STATE, "best_split before sweep_thresholds");
  DeviceGuard g(p->device);
  const int ranks = (p->dist && !(p->flags & FP_FLAG_REPLICATED_GRID)) ? p->world : 1;
  const size_t M = p->models.size();
  const size_t nrec = (size_t)ranks * M;
  // records and the per-bin counts in one stream-ordered round trip (pinned)
  CUDA_TRY(p, cudaMemcpyAsync(p->h_best, p->d_best, nrec * sizeof(fp_candidate), cudaMemcpyDeviceToHost,
                              p->last_stream), "D2H best");
  CUDA_TRY(p, cudaMemcpyAsync(p->h_small, p->d_hist, p->nbins * 8, cudaMemcpyDeviceToHost, p->last_stream),
           "D2H hist");
  CUDA_TRY(p, cudaStreamSynchronize(p->last_stream), "sync");
  if (p->flags & FP_FLAG_P2P) {
    fp_status st = check_device_error(p);
    if (st != FP_OK) return st;
  }
  if (p->h_phase && p->h_phase[0]) {
    for (int i = 1; i <= 10; ++i)
      if (p->h_phase[i] >= p->h_phase[0]) p->phase_sum[i] += (double)(p->h_phase[i] - p->h_phase[0]);
    ++p->phase_n;
  }
  unsigned long long total = 0;
  for (uint32_t j = 0; j < p->nbins; ++j) total += p->h_small[j];
  if (total == 0) return fail(p, FP_ERR_EMPTY_TRACE, "global trace is empty");
  fp_merge_best(p->h_best, ranks, (uint32_t)M, h_best);
  return FP_OK;
}

fp_status sweep_histogram(fp_plan *p, uint32_t *h_edges, uint64_t *h_bin_cnt, uint64_t *h_bin_mass) {
  if (!p) return FP_ERR_INVALID_ARG;
  if (!p->have_sweep) return fail(p, FP_ERR_STATE, "sweep_histogram before sweep_thresholds");
  DeviceGuard g(p->device);
  CUDA_TRY(p, cudaStreamSynchronize(p->last_stream), "sync");
  if (p->flags & FP_FLAG_P2P) {
    fp_status st = check_device_error(p);
    if (st != FP_OK) return st;
  }
  if (h_edges) memcpy(h_edges, p->edges.data(), p->edges.size() * 4);
  if (h_bin_cnt) CUDA_TRY(p, cudaMemcpy(h_bin_cnt, p->d_hist, p->nbins * 8, cudaMemcpyDeviceToHost), "D2H hist");
  if (h_bin_mass)
    CUDA_TRY(p, cudaMemcpy(h_bin_mass, p->d_hist + p->nbins, p->nbins * 8, cudaMemcpyDeviceToHost), "D2H hist");
  return FP_OK;
}

}  // extern "C"
