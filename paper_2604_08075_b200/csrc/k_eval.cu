// K2 + K3: prefix scan of the trace histogram, candidate-grid evaluation and
// per-model argmin.
//
// One thread per candidate; blockIdx.y = model. Prologue (per block): the
// |E|+1-bin histogram is scanned into cnt_le / mass_le (K2, P:589 alpha =
// F(B)) and the capacity table N_seq[g][w] (Eq. 1-2) and mu[g][w]
// are staged in shared memory. Each thread then sizes its candidate with the
// Sec. 3 formulas in IEEE binary64 with explicit round-to-nearest
// intrinsics and no contraction (DESIGN R14; the library is also built with
// --fmad=false), and the block reduces (cost, index) with warp shuffles. The
// last block of each model (self-resetting arrival counter) reduces the
// per-block winners and re-evaluates the winning index into a full record.
#include <cfloat>
#include <cmath>
#include "internal.cuh"

namespace fp {

namespace {

struct Shared {
  unsigned long long *cnt_le;   // [nbins]
  unsigned long long *mass_le;  // [nbins]
  unsigned long long *nseq;     // [n_gpus][n_windows]
  double *mu;                   // [n_gpus][n_windows]
  double *rmu;                  // [n_gpus][n_windows] RN(1/mu), 0 = use the IEEE division
  double rN;                    // RN(1/N), 0 = use the IEEE division
};

// RN(x / d) for x >= 0. With y = RN(1/d) (y != 0: d and x in range) it is
// Markstein's correction q0 = x y, r = x - d q0 (exact, one FMA), q = q0 + r y,
// which returns the correctly rounded quotient -- the IEEE division the oracle
// performs -- in 3 FP64 operations instead of a DDIV sequence (~40
// instructions with a MUFU and a slow-path branch). Its preconditions are
// exponent ranges: |x|, |d| in [2^-400, 2^400] keep the quotient, the
// residual and its correction normal. Otherwise: the IEEE division itself.
__device__ __forceinline__ double mdiv(double x, double d, double y) {
  if (y != 0.0 && x <= 0x1p400 && (x >= 0x1p-400 || x == 0.0)) {
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-d, q0, x);
    return __fma_rn(y, r, q0);
  }
  return __ddiv_rn(x, d);
}

// the reciprocal mdiv may use for divisor d (0 when d is out of its range)
__device__ __forceinline__ double mrcp(double d) {
  return (d >= 0x1p-400 && d <= 0x1p400) ? __ddiv_rn(1.0, d) : 0.0;
}

__device__ __forceinline__ double u2d(unsigned long long x) { return __ull2double_rn(x); }

// Eq. (2): N_seq = floor(budget * tp / M_seq), M_seq = 2 n_l n_h d_h b C (Eq. 1).
// Bounds validated at plan creation keep every product below 2^64.
__device__ __forceinline__ unsigned long long max_seqs(unsigned long long budget, uint32_t tp,
                                                       const uint32_t *arch, uint32_t c) {
  unsigned long long mseq = 2ull * arch[0] * arch[1] * arch[2] * arch[3] * (unsigned long long)c;
  if (mseq == 0) return 0;
  return (budget * tp) / mseq;
}

// budget = floor(M_gpu * u) - M_model - M_act, clamped at 0.
__device__ __forceinline__ unsigned long long kv_budget(const unsigned long long *gu,
                                                        unsigned long long weights) {
  unsigned long long usable = (gu[0] * gu[1]) / gu[2];
  unsigned long long need = weights + gu[3];
  return usable > need ? usable - need : 0ull;
}

// One pool: I = ceil(lambda / mu); lambda == 0 -> 0; no capacity -> infeasible (R13).
// rmu = RN(1/mu) or 0 (mdiv).
__device__ __forceinline__ bool pool_instances(double lam, double mu, double rmu, uint64_t nseq,
                                               uint64_t *inst) {
  *inst = 0;
  if (lam == 0.0) return true;
  if (nseq == 0 || !(mu > 0.0)) return false;
  double x = mdiv(lam, mu, rmu);
  if (!(x <= 9007199254740992.0)) return false;
  *inst = (unsigned long long)ceil(x);
  return true;
}

// x / d and x % d for x < 2^32 by a precomputed multiplier mul = ceil(2^64 / d)
// (0 for d = 1): floor(x mul / 2^64) = floor(x / d + delta), delta < 2^-32 <= 1/d,
// so the quotient is exact (a 32-bit IDIV sequence costs ~20 instructions)
__device__ __forceinline__ uint32_t divmod(uint32_t x, uint32_t d, unsigned long long mul, uint32_t &rem) {
  const uint32_t q = mul ? (uint32_t)__umul64hi((unsigned long long)x, mul) : x;
  rem = x - q * d;
  return q;
}

// FULL: the whole record; otherwise only what the argmin needs (index,
// flags, cost_dual -- bit-identical to the full record's), skipping the
// savings / rho / predicted / occupancy divisions (large grids without results)
template <bool FULL>
__device__ void evaluate(const EvalArgs &a, const Shared &sh, uint32_t m, uint64_t idx,
                         fp_candidate &c) {
  // decompose idx = (((m * G + g) * n_cl + l) * n_cs' + s) * n_b + k
  // 32-bit index math: the plan guarantees < 2^32 candidates
  uint32_t r = (uint32_t)idx, k, s, l, g;
  r = divmod(r, a.n_b, a.div_b, k);
  r = divmod(r, a.n_cs_eff, a.div_cs, s);
  r = divmod(r, a.n_cl, a.div_cl, l);
  divmod(r, a.n_gpus, a.div_g, g);
  uint32_t B = a.b[k], CL = a.cl[l];
  uint32_t CS = a.n_cs ? a.cs[s] : B;
  c.index = (uint32_t)idx; c.model = m; c.gpu = g;
  c.b_short = B; c.c_short = CS; c.c_long = CL; c.flags = 0; c._pad = 0;
  c.nseq_short = c.nseq_long = 0;
  c.n_short = c.n_long = c.n_reject = c.mass_short = c.mass_long = 0;
  c.inst_short = c.inst_long = c.inst_homo = c.gpus_dual = c.gpus_homo = 0;
  c.alpha = c.rho = c.predicted_savings = c.savings = 0.0;
  c.cost_dual = c.cost_homo = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  c.occupancy_short = c.occupancy_long = 0.0;
  if (!(B <= CS && CS <= CL)) return;  // invalid split

  const unsigned long long N = sh.cnt_le[a.nbins - 1];
  const uint32_t eb = a.b_edge[k], el = a.cl_edge[l];
  const unsigned long long n_s = sh.cnt_le[eb], n_sl = sh.cnt_le[el];
  c.n_short = n_s;
  c.n_long = n_sl - n_s;
  c.n_reject = N - n_sl;
  c.mass_short = sh.mass_le[eb];
  c.mass_long = sh.mass_le[el] - sh.mass_le[eb];

  const uint32_t ws = a.n_cs ? a.cs_win[s] : a.b_win[k];
  const uint32_t wl = a.cl_win[l];
  const uint32_t gw = g * a.n_windows;
  c.nseq_short = sh.nseq[gw + ws];
  c.nseq_long = sh.nseq[gw + wl];
  const double mu_s = sh.mu[gw + ws], mu_l = sh.mu[gw + wl];
  const double rmu_s = sh.rmu[gw + ws], rmu_l = sh.rmu[gw + wl];

  const double dN = u2d(N);
  c.alpha = mdiv(u2d(n_s), dN, sh.rN);
  const double lam_s = __dmul_rn(c.alpha, a.rate);
  const double lam_l = __dmul_rn(mdiv(u2d(c.n_long), dN, sh.rN), a.rate);
  const double lam_h = __dmul_rn(mdiv(u2d(n_sl), dN, sh.rN), a.rate);

  const bool ok_s = pool_instances(lam_s, mu_s, rmu_s, c.nseq_short, &c.inst_short);
  const bool ok_l = pool_instances(lam_l, mu_l, rmu_l, c.nseq_long, &c.inst_long);
  const bool ok_h = pool_instances(lam_h, mu_l, rmu_l, c.nseq_long, &c.inst_homo);
  const bool ok_d = ok_s && ok_l;
  if (!ok_d) { c.inst_short = 0; c.inst_long = 0; }
  const unsigned long long gpi = a.deploy[((uint64_t)m * a.n_gpus + g) * 3 + 1];
  c.gpus_dual = gpi * (c.inst_short + c.inst_long);
  c.gpus_homo = gpi * c.inst_homo;
  const double price = a.price[g];
  if (ok_d) c.cost_dual = __dmul_rn(__dmul_rn(u2d(c.gpus_dual), price), a.hours);
  if (ok_h) c.cost_homo = __dmul_rn(__dmul_rn(u2d(c.gpus_homo), price), a.hours);
  c.flags = FP_CAND_VALID | (ok_d ? FP_CAND_FEASIBLE : 0u) | (ok_h ? FP_CAND_HOMO_FEASIBLE : 0u);
  if constexpr (!FULL) return;
  if (ok_d && ok_h && c.gpus_homo > 0)
    c.savings = __ddiv_rn(__dsub_rn(u2d(c.gpus_homo), u2d(c.gpus_dual)), u2d(c.gpus_homo));
  if (mu_s > 0.0 && mu_l > 0.0) {
    c.rho = mdiv(mu_s, mu_l, rmu_l);
    // the oracle's guard: a rho that underflows to 0 leaves predicted at 0
    if (c.rho > 0.0) c.predicted_savings = __dmul_rn(c.alpha, __dsub_rn(1.0, __ddiv_rn(1.0, c.rho)));
  }
  if (c.n_short)
    c.occupancy_short = __ddiv_rn(u2d(c.mass_short), __dmul_rn(u2d(c.n_short), u2d(CS)));
  if (c.n_long)
    c.occupancy_long = __ddiv_rn(u2d(c.mass_long), __dmul_rn(u2d(c.n_long), u2d(CL)));
}

// NEXT-2: three pools. idx = ((m * G + g) * n_cl + l) * n_pairs + p,
// pair p = (i, j), i < j over the B grid; windows C1 = B1, C2 = B2, C3 = C_L;
// first-fit routing (L <= B1, else L <= B2, else L <= C_L, else rejected) and
// the Sec. 3 sizing per pool, in the oracle's operation order (or_sweep3).
__device__ void evaluate3(const EvalArgs &a, const Shared &sh, uint32_t m, uint64_t idx, fp_pool3_candidate &c) {
  uint32_t r = (uint32_t)idx;
  const uint32_t p = r % a.n_pairs; r /= a.n_pairs;
  const uint32_t l = r % a.n_cl; r /= a.n_cl;
  const uint32_t g = r % a.n_gpus;
  const uint32_t pr = a.pairs[p], i = pr & 0xFFFFu, j = pr >> 16;
  const uint32_t B1 = a.b[i], B2 = a.b[j], CL = a.cl[l];
  c.index = (uint32_t)idx; c.model = m; c.gpu = g; c.b1 = B1; c.b2 = B2; c.c_long = CL;
  c.flags = 0; c._pad = 0;
  c.n1 = c.n2 = c.n3 = c.n_reject = 0;
  c.nseq1 = c.nseq2 = c.nseq3 = 0;
  c.inst1 = c.inst2 = c.inst3 = c.inst_homo = c.gpus = c.gpus_homo = 0;
  c.cost = c.cost_homo = __longlong_as_double(0x7ff0000000000000ll);
  c.savings = 0.0;
  if (!(B1 < B2 && B2 <= CL)) return;
  const unsigned long long N = sh.cnt_le[a.nbins - 1];
  const unsigned long long c1 = sh.cnt_le[a.b_edge[i]], c2 = sh.cnt_le[a.b_edge[j]], c3 = sh.cnt_le[a.cl_edge[l]];
  c.n1 = c1;
  c.n2 = c2 - c1;
  c.n3 = c3 - c2;
  c.n_reject = N - c3;
  const uint32_t gw = g * a.n_windows;
  const uint32_t w1 = gw + a.b_win3[i], w2 = gw + a.b_win3[j], w3 = gw + a.cl_win[l];
  c.nseq1 = sh.nseq[w1];
  c.nseq2 = sh.nseq[w2];
  c.nseq3 = sh.nseq[w3];
  const double dN = u2d(N);
  const double lam1 = __dmul_rn(mdiv(u2d(c.n1), dN, sh.rN), a.rate);
  const double lam2 = __dmul_rn(mdiv(u2d(c.n2), dN, sh.rN), a.rate);
  const double lam3 = __dmul_rn(mdiv(u2d(c.n3), dN, sh.rN), a.rate);
  const double lamh = __dmul_rn(mdiv(u2d(c3), dN, sh.rN), a.rate);
  const bool ok1 = pool_instances(lam1, sh.mu[w1], sh.rmu[w1], c.nseq1, &c.inst1);
  const bool ok2 = pool_instances(lam2, sh.mu[w2], sh.rmu[w2], c.nseq2, &c.inst2);
  const bool ok3 = pool_instances(lam3, sh.mu[w3], sh.rmu[w3], c.nseq3, &c.inst3);
  const bool okh = pool_instances(lamh, sh.mu[w3], sh.rmu[w3], c.nseq3, &c.inst_homo);
  const bool ok = ok1 && ok2 && ok3;
  if (!ok) { c.inst1 = c.inst2 = c.inst3 = 0; }
  const unsigned long long gpi = a.deploy[((uint64_t)m * a.n_gpus + g) * 3 + 1];
  c.gpus = gpi * (c.inst1 + c.inst2 + c.inst3);
  c.gpus_homo = gpi * c.inst_homo;
  const double price = a.price[g];
  if (ok) c.cost = __dmul_rn(__dmul_rn(u2d(c.gpus), price), a.hours);
  if (okh) c.cost_homo = __dmul_rn(__dmul_rn(u2d(c.gpus_homo), price), a.hours);
  if (ok && okh && c.gpus_homo > 0)
    c.savings = __ddiv_rn(__dsub_rn(u2d(c.gpus_homo), u2d(c.gpus)), u2d(c.gpus_homo));
  c.flags = FP_CAND_VALID | (ok ? FP_CAND_FEASIBLE : 0u) | (okh ? FP_CAND_HOMO_FEASIBLE : 0u);
}

template <bool POOL3> struct RecOf { using T = fp_candidate; };
template <> struct RecOf<true> { using T = fp_pool3_candidate; };

template <bool FULL = true>
__device__ __forceinline__ void eval_any(const EvalArgs &a, const Shared &sh, uint32_t m, uint64_t idx,
                                         fp_candidate &c, double &cost) {
  evaluate<FULL>(a, sh, m, idx, c);
  cost = c.cost_dual;
}
template <bool FULL = true>
__device__ __forceinline__ void eval_any(const EvalArgs &a, const Shared &sh, uint32_t m, uint64_t idx,
                                         fp_pool3_candidate &c, double &cost) {
  evaluate3(a, sh, m, idx, c);
  cost = c.cost;
}

// (cost, index) lexicographic min; non-candidates carry valid = 0.
__device__ __forceinline__ void better(double &c0, uint32_t &i0, uint32_t &v0, double c1, uint32_t i1,
                                       uint32_t v1) {
  bool take = v1 && (!v0 || c1 < c0 || (c1 == c0 && i1 < i0));
  if (take) { c0 = c1; i0 = i1; v0 = v1; }
}

__device__ __forceinline__ void warp_argmin(double &c, uint32_t &i, uint32_t &v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double c1 = __shfl_down_sync(0xffffffffu, c, o);
    uint32_t i1 = __shfl_down_sync(0xffffffffu, i, o);
    uint32_t v1 = __shfl_down_sync(0xffffffffu, v, o);
    better(c, i, v, c1, i1, v1);
  }
}

// Block-wide exclusive/inclusive scan helper: inclusive prefix of x over the block.
__device__ void block_scan_inclusive(unsigned long long *data, uint32_t n,
                                     unsigned long long *warp_tot) {
  // each thread owns a contiguous run of ceil(n / blockDim) elements
  const uint32_t T = blockDim.x, t = threadIdx.x;
  const uint32_t per = (n + T - 1) / T;
  const uint32_t lo = min(n, t * per), hi = min(n, lo + per);
  unsigned long long run = 0;
  for (uint32_t j = lo; j < hi; ++j) run += data[j];
  // inclusive warp scan of run
  unsigned long long x = run;
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    const int nw = (T + 31) >> 5;
    unsigned long long z = lane < nw ? warp_tot[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < nw) warp_tot[lane] = z;
  }
  __syncthreads();
  unsigned long long off = (x - run) + (w ? warp_tot[w - 1] : 0ull);
  for (uint32_t j = lo; j < hi; ++j) { off += data[j]; data[j] = off; }
  __syncthreads();
}

template <bool POOL3>
__global__ void __launch_bounds__(256, 3) k3_eval(EvalArgs a) {
  using Rec = typename RecOf<POOL3>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long warp_tot[32];
  __shared__ double red_c[32];
  __shared__ uint32_t red_i[32], red_v[32];
  __shared__ uint32_t route_v[4];
  __shared__ bool is_last, zero_last;
  const uint32_t m = blockIdx.y;

  Shared sh;
  sh.cnt_le = reinterpret_cast<unsigned long long *>(smem);
  sh.mass_le = sh.cnt_le + a.nbins;
  sh.nseq = sh.mass_le + a.nbins;
  sh.mu = reinterpret_cast<double *>(sh.nseq + (size_t)a.n_gpus * a.n_windows);
  sh.rmu = sh.mu + (size_t)a.n_gpus * a.n_windows;

  // ---- prologue: K2 scan + capacity table for model m ----
  // the plan's tables first: they do not depend on the trace pass, so with a
  // programmatic (PDL) launch they load while K1's last blocks drain
  for (uint32_t j = threadIdx.x; j < a.n_gpus * a.n_windows; j += blockDim.x) {
    sh.nseq[j] = a.cap_nseq[(uint64_t)m * a.n_gpus * a.n_windows + j];
    const double mu = a.mu[(uint64_t)m * a.n_gpus * a.n_windows + j];
    sh.mu[j] = mu;
    sh.rmu[j] = mrcp(mu);
  }
  // K1's histogram is complete and visible after this (no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // sum K1's accumulator copies; block (0, 0) also publishes the summed
  // histogram (sweep_histogram, best_split's empty-trace check)
  if (a.p2p_world) {
    // peer-memory exchange (FP_FLAG_P2P): wait until every rank has released
    // this step's accumulators (its K1 done, fenced system-wide), then read
    // all ranks' copies directly -- the cross-rank sum fused into this prologue
    if (threadIdx.x < a.p2p_world) {
      const unsigned int *f = a.peer_flag[threadIdx.x];
      unsigned int v;
      for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int)(v - a.p2p_epoch) >= 0) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < a.nbins; j += blockDim.x) {
      unsigned long long cnt = 0, mass = 0;
      for (uint32_t r = 0; r < a.p2p_world; ++r) {
        const unsigned long long *h = a.peer_hist[r] + a.p2p_off;
        for (uint32_t c = 0; c < a.hist_copies; ++c) {
          cnt += __ldcv(h + (size_t)c * 2 * a.nbins + j);
          mass += __ldcv(h + (size_t)c * 2 * a.nbins + a.nbins + j);
        }
      }
      sh.cnt_le[j] = cnt;
      sh.mass_le[j] = mass;
      if (a.hist_out && blockIdx.x == 0 && blockIdx.y == 0) {
        a.hist_out[j] = cnt;
        a.hist_out[a.nbins + j] = mass;
      }
    }
  } else
  for (uint32_t j = threadIdx.x; j < a.nbins; j += blockDim.x) {
    unsigned long long cnt = 0, mass = 0;
    if (a.hist_copies == 16) {
      // all 32 loads in flight at once (one L2 round trip, not sixteen)
      unsigned long long vc[16], vm[16];
#pragma unroll
      for (uint32_t c = 0; c < 16; ++c) {
        vc[c] = a.hist_cnt[(size_t)c * 2 * a.nbins + j];
        vm[c] = a.hist_mass[(size_t)c * 2 * a.nbins + j];
      }
#pragma unroll
      for (uint32_t c = 0; c < 16; ++c) { cnt += vc[c]; mass += vm[c]; }
    } else {
      for (uint32_t c = 0; c < a.hist_copies; ++c) {
        cnt += a.hist_cnt[(size_t)c * 2 * a.nbins + j];
        mass += a.hist_mass[(size_t)c * 2 * a.nbins + j];
      }
    }
    sh.cnt_le[j] = cnt;
    sh.mass_le[j] = mass;
    if (a.hist_out && blockIdx.x == 0 && blockIdx.y == 0) {
      a.hist_out[j] = cnt;
      a.hist_out[a.nbins + j] = mass;
    }
  }
  __syncthreads();
  if (a.zero_copies) {
    // every block has its sums in shared memory now; the last one to get here
    // zeroes the copies (stream order puts this before the next sweep's K1)
    if (threadIdx.x == 0) {
      __threadfence();
      zero_last = atomicAdd(a.read_done, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (zero_last) {
      const size_t total = (size_t)a.hist_copies * 2 * a.nbins;
      for (size_t i = threadIdx.x; i < total; i += blockDim.x) a.zero_copies[i] = 0ull;
      if (threadIdx.x == 0) *a.read_done = 0u;
    }
  }
  block_scan_inclusive(sh.cnt_le, a.nbins, warp_tot);
  block_scan_inclusive(sh.mass_le, a.nbins, warp_tot);
  sh.rN = mrcp(u2d(sh.cnt_le[a.nbins - 1]));

  // ---- this block's candidates: model m's part of the rank slice ----
  const uint64_t per = POOL3 ? a.per_model3 : a.per_model;
  const uint64_t m_lo = (uint64_t)m * per, m_hi = m_lo + per;
  // the three-pool grid is evaluated whole on every rank (replicated)
  const uint64_t lo = POOL3 ? m_lo : max(m_lo, a.cand_first);
  const uint64_t hi = POOL3 ? m_hi : min(m_hi, a.cand_first + a.cand_count);
  // grid-stride over the model's candidates: the per-block prologue (scan,
  // capacity table) and epilogue (argmin, arrival fence) are amortised over
  // many candidates per thread on large grids (ncu r01_k3L: one candidate per
  // thread spent most of its time in the prologue and the arrival fence)
  double bc = 0.0;
  uint32_t bi = 0xffffffffu, bv = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool want = POOL3 ? a.results3 != nullptr : a.results != nullptr;
  if (want) {
    for (uint64_t idx = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < hi; idx += stride) {
      Rec c;
      double cost;
      eval_any<true>(a, sh, m, idx, c, cost);
      if (POOL3) reinterpret_cast<Rec *>(a.results3)[idx] = c;
      else reinterpret_cast<Rec *>(a.results)[idx - a.cand_first] = c;
      // indices increase along the loop, so strict '<' keeps the lowest index on ties
      if ((c.flags & FP_CAND_FEASIBLE) && (!bv || cost < bc)) { bc = cost; bi = c.index; bv = 1; }
    }
  } else {
    // no records requested: the argmin's fields only (the winner is
    // re-evaluated in full by the last block)
    for (uint64_t idx = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < hi; idx += stride) {
      Rec c;
      double cost;
      eval_any<false>(a, sh, m, idx, c, cost);
      if ((c.flags & FP_CAND_FEASIBLE) && (!bv || cost < bc)) { bc = cost; bi = c.index; bv = 1; }
    }
  }
  warp_argmin(bc, bi, bv);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) { red_c[w] = bc; red_i[w] = bi; red_v[w] = bv; }
  __syncthreads();
  if (w == 0) {
    bc = lane < nw ? red_c[lane] : 0.0;
    bi = lane < nw ? red_i[lane] : 0xffffffffu;
    bv = lane < nw ? red_v[lane] : 0u;
    warp_argmin(bc, bi, bv);
    if (lane == 0) {
      BlockBest *bb = (POOL3 ? a.block_best3 : a.block_best) + (size_t)m * gridDim.x + blockIdx.x;
      bb->cost = bc; bb->index = bi; bb->valid = bv;
      if (gridDim.x == 1) {
        is_last = true;                 // one block per model: no arrival protocol
      } else {
        __threadfence();
        unsigned int prev = atomicAdd((POOL3 ? a.done3 : a.done) + m, 1u);
        is_last = (prev == gridDim.x - 1);
      }
    }
  }
  __syncthreads();
  if (!is_last) return;

  // ---- last block of model m: reduce the per-block winners, emit the record ----
  if (gridDim.x > 1) __threadfence();
  bc = 0.0; bi = 0xffffffffu; bv = 0;
  for (uint32_t j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
    const volatile BlockBest *bb = (POOL3 ? a.block_best3 : a.block_best) + (size_t)m * gridDim.x + j;
    better(bc, bi, bv, bb->cost, bb->index, bb->valid);
  }
  warp_argmin(bc, bi, bv);
  if (lane == 0) { red_c[w] = bc; red_i[w] = bi; red_v[w] = bv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < nw; ++j) better(bc, bi, bv, red_c[j], red_i[j], red_v[j]);
    Rec c;
    double cost;
    if (bv) {
      eval_any(a, sh, m, bi, c, cost);
    } else {
      memset(&c, 0, sizeof c);
      c.index = 0xffffffffu;
      c.model = m;
      if constexpr (POOL3) c.cost = c.cost_homo = __longlong_as_double(0x7ff0000000000000ll);
      else c.cost_dual = c.cost_homo = __longlong_as_double(0x7ff0000000000000ll);
    }
    if constexpr (POOL3) {
      a.best3[m] = c;
      a.done3[m] = 0;
    } else {
      a.best_out[m] = c;
      a.done[m] = 0;  // self-reset for the next launch / graph replay
      if (a.route_out && m == a.route_model) {
        route_v[0] = c.b_short; route_v[1] = c.c_short; route_v[2] = c.c_long;
        route_v[3] = (c.flags & FP_CAND_FEASIBLE) ? 1u : 0u;
      }
    }
  }
  if constexpr (!POOL3) {
    // the split to route with: edge indices #{e in E : e < v} of its B, C_S, C_L
    if (a.route_out && m == a.route_model) {
      __syncthreads();
      if (w == 0) {
        uint32_t nb = 0, ns = 0, nl = 0;
        for (uint32_t base = 0; base < a.n_edges; base += 32) {
          const uint32_t e = base + lane < a.n_edges ? a.edges[base + lane] : 0xffffffffu;
          nb += __popc(__ballot_sync(0xffffffffu, e < route_v[0]));
          ns += __popc(__ballot_sync(0xffffffffu, e < route_v[1]));
          nl += __popc(__ballot_sync(0xffffffffu, e < route_v[2]));
        }
        if (lane == 0) *reinterpret_cast<uint4 *>(a.route_out) = make_uint4(nb, ns, nl, route_v[3]);
      }
    }
  }
}

// N_seq (Eq. 2) for every (model, GPU, window): plan data only, computed once
__global__ void k_capacity(EvalArgs a, unsigned long long *cap) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (uint64_t)a.n_models * a.n_gpus * a.n_windows) return;
  const uint32_t w = (uint32_t)(j % a.n_windows), g = (uint32_t)(j / a.n_windows % a.n_gpus);
  const uint32_t m = (uint32_t)(j / ((uint64_t)a.n_windows * a.n_gpus));
  const unsigned long long *dp = a.deploy + ((uint64_t)m * a.n_gpus + g) * 3;
  cap[j] = max_seqs(kv_budget(a.gpu_u64 + 4 * g, dp[2]), (uint32_t)dp[0], a.model_arch + 4 * m, a.windows[w]);
}

// NEXT-4: peak-window sizing. Same grid and index decomposition
// as evaluate(); the routing counts of a pool become its busiest window's
// counts (max over windows of the cumulative per-window histogram), the rates
// peak * (1e9 / window_ns), and each pool is sized with the Sec. 3 formula in
// the oracle's operation order (or_sweep_peak).
__device__ void evaluate_peak(const EvalArgs &a, const Shared &sh, uint32_t m, uint64_t idx, fp_peak_candidate &c) {
  uint32_t r = (uint32_t)idx;
  const uint32_t k = r % a.n_b; r /= a.n_b;
  const uint32_t s = r % a.n_cs_eff; r /= a.n_cs_eff;
  const uint32_t l = r % a.n_cl; r /= a.n_cl;
  const uint32_t g = r % a.n_gpus;
  const uint32_t B = a.b[k], CL = a.cl[l], CS = a.n_cs ? a.cs[s] : B;
  c.index = (uint32_t)idx; c.model = m; c.gpu = g; c.b_short = B; c.c_short = CS; c.c_long = CL;
  c.flags = 0; c._pad = 0;
  c.peak_short = c.peak_long = c.peak_homo = 0;
  c.inst_short = c.inst_long = c.inst_homo = c.gpus_dual = c.gpus_homo = 0;
  c.lambda_short = c.lambda_long = c.lambda_homo = 0.0;
  c.cost_dual = c.cost_homo = __longlong_as_double(0x7ff0000000000000ll);
  c.savings = 0.0;
  if (!(B <= CS && CS <= CL)) return;
  const uint32_t eb = a.b_edge[k], el = a.cl_edge[l];
  // busiest-window counts, reduced over windows by K2w (k_peak.cu)
  const unsigned long long ps = a.colmax_pk[eb], ph = a.colmax_pk[el], pl = a.pairmax_pk[k * a.n_cl + l];
  c.peak_short = ps; c.peak_long = pl; c.peak_homo = ph;
  const uint32_t ws = a.n_cs ? a.cs_win[s] : a.b_win[k], wl = a.cl_win[l];
  const uint32_t gw = g * a.n_windows;
  const unsigned long long nseq_s = sh.nseq[gw + ws], nseq_l = sh.nseq[gw + wl];
  c.lambda_short = __dmul_rn(u2d(ps), a.inv_w_s);
  c.lambda_long = __dmul_rn(u2d(pl), a.inv_w_s);
  c.lambda_homo = __dmul_rn(u2d(ph), a.inv_w_s);
  const bool ok_s = pool_instances(c.lambda_short, sh.mu[gw + ws], sh.rmu[gw + ws], nseq_s, &c.inst_short);
  const bool ok_l = pool_instances(c.lambda_long, sh.mu[gw + wl], sh.rmu[gw + wl], nseq_l, &c.inst_long);
  const bool ok_h = pool_instances(c.lambda_homo, sh.mu[gw + wl], sh.rmu[gw + wl], nseq_l, &c.inst_homo);
  const bool ok_d = ok_s && ok_l;
  if (!ok_d) { c.inst_short = 0; c.inst_long = 0; }
  const unsigned long long gpi = a.deploy[((uint64_t)m * a.n_gpus + g) * 3 + 1];
  c.gpus_dual = gpi * (c.inst_short + c.inst_long);
  c.gpus_homo = gpi * c.inst_homo;
  const double price = a.price[g];
  if (ok_d) c.cost_dual = __dmul_rn(__dmul_rn(u2d(c.gpus_dual), price), a.hours);
  if (ok_h) c.cost_homo = __dmul_rn(__dmul_rn(u2d(c.gpus_homo), price), a.hours);
  if (ok_d && ok_h && c.gpus_homo > 0)
    c.savings = __ddiv_rn(__dsub_rn(u2d(c.gpus_homo), u2d(c.gpus_dual)), u2d(c.gpus_homo));
  c.flags = FP_CAND_VALID | (ok_d ? FP_CAND_FEASIBLE : 0u) | (ok_h ? FP_CAND_HOMO_FEASIBLE : 0u);
}

__global__ void __launch_bounds__(256) k3_peak(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red_c[32];
  __shared__ uint32_t red_i[32], red_v[32];
  __shared__ bool is_last;
  const uint32_t m = blockIdx.y;
  Shared sh;
  sh.cnt_le = nullptr;
  sh.mass_le = nullptr;
  sh.nseq = reinterpret_cast<unsigned long long *>(smem);
  sh.mu = reinterpret_cast<double *>(sh.nseq + (size_t)a.n_gpus * a.n_windows);
  sh.rmu = sh.mu + (size_t)a.n_gpus * a.n_windows;
  sh.rN = 0.0;
  for (uint32_t j = threadIdx.x; j < a.n_gpus * a.n_windows; j += blockDim.x) {
    sh.nseq[j] = a.cap_nseq[(uint64_t)m * a.n_gpus * a.n_windows + j];
    const double mu = a.mu[(uint64_t)m * a.n_gpus * a.n_windows + j];
    sh.mu[j] = mu;
    sh.rmu[j] = mrcp(mu);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // K2w's window maxima (PDL launch)
  __syncthreads();
  const uint64_t lo = (uint64_t)m * a.per_model, hi = lo + a.per_model;
  double bc = 0.0;
  uint32_t bi = 0xffffffffu, bv = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t idx = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < hi; idx += stride) {
    fp_peak_candidate c;
    evaluate_peak(a, sh, m, idx, c);
    if (a.results_pk) a.results_pk[idx] = c;
    if ((c.flags & FP_CAND_FEASIBLE) && (!bv || c.cost_dual < bc)) { bc = c.cost_dual; bi = c.index; bv = 1; }
  }
  warp_argmin(bc, bi, bv);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) { red_c[w] = bc; red_i[w] = bi; red_v[w] = bv; }
  __syncthreads();
  if (w == 0) {
    bc = lane < nw ? red_c[lane] : 0.0;
    bi = lane < nw ? red_i[lane] : 0xffffffffu;
    bv = lane < nw ? red_v[lane] : 0u;
    warp_argmin(bc, bi, bv);
    if (lane == 0) {
      BlockBest *bb = a.block_best_pk + (size_t)m * gridDim.x + blockIdx.x;
      bb->cost = bc; bb->index = bi; bb->valid = bv;
      __threadfence();
      is_last = atomicAdd(a.done_pk + m, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  bc = 0.0; bi = 0xffffffffu; bv = 0;
  for (uint32_t j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
    const volatile BlockBest *bb = a.block_best_pk + (size_t)m * gridDim.x + j;
    better(bc, bi, bv, bb->cost, bb->index, bb->valid);
  }
  warp_argmin(bc, bi, bv);
  if (lane == 0) { red_c[w] = bc; red_i[w] = bi; red_v[w] = bv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < nw; ++j) better(bc, bi, bv, red_c[j], red_i[j], red_v[j]);
    fp_peak_candidate c;
    if (bv) {
      evaluate_peak(a, sh, m, bi, c);
    } else {
      memset(&c, 0, sizeof c);
      c.index = 0xffffffffu;
      c.model = m;
      c.cost_dual = c.cost_homo = __longlong_as_double(0x7ff0000000000000ll);
    }
    a.best_pk[m] = c;
    a.done_pk[m] = 0;
  }
}

}  // namespace

cudaError_t launch_eval_peak(const EvalArgs &a, int grid_x, int block, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k3_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  return launch_pdl(k3_peak, dim3(grid_x, a.n_models), dim3(block), smem, s, a);
}

size_t eval_smem_bytes(const EvalArgs &a, int) {
  return (size_t)a.nbins * 16 + (size_t)a.n_gpus * a.n_windows * 24;
}

cudaError_t eval_prepare() {
  cudaError_t e = cudaFuncSetAttribute(k3_eval<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k3_eval<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

cudaError_t launch_capacity(const EvalArgs &a, unsigned long long *cap, cudaStream_t s) {
  const uint64_t n = (uint64_t)a.n_models * a.n_gpus * a.n_windows;
  k_capacity<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, cap);
  return cudaGetLastError();
}

namespace {
// after K1 (stream order): make this rank's accumulators visible system-wide,
// then publish the step's epoch (release) for the peers' K3 prologues
__global__ void k_p2p_signal(unsigned int *flag, unsigned int epoch) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}
}  // namespace

cudaError_t launch_p2p_signal(unsigned int *flag, unsigned int epoch, cudaStream_t s) {
  k_p2p_signal<<<1, 1, 0, s>>>(flag, epoch);
  return cudaGetLastError();
}

// K3 after K1 as a programmatic dependent launch: its blocks are scheduled as
// K1's blocks exit and wait (griddepcontrol.wait) only before the histogram
// reads, which hides the launch latency and the table loads (FP_NO_PDL=1: a
// plain launch)
cudaError_t launch_eval(const EvalArgs &a, int grid_x, int block, size_t smem, cudaStream_t s) {
  return launch_pdl(k3_eval<false>, dim3(grid_x, a.n_models), dim3(block), smem, s, a);
}

cudaError_t launch_eval3(const EvalArgs &a, int grid_x, int block, size_t smem, cudaStream_t s) {
  dim3 grid(grid_x, a.n_models);
  k3_eval<true><<<grid, block, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace fp
