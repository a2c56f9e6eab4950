// K2 + K3: prefix scan of the trace histogram, candidate-grid evaluation and
// per-model argmin.
//
// Every block stages what its model's candidates read -- the grid values and
// their edge / window indices, the capacity table N_seq[g][w] (Eq. 1-2,
// P:23-39, computed once per plan), mu[g][w] and its correctly rounded
// reciprocal, GPUs per instance and price -- in shared memory BEFORE waiting
// on the trace pass (programmatic dependent launch: these loads overlap K1's
// drain), then reads the |E|+1-bin histogram and scans it into cnt_le /
// mass_le (K2, P:589 alpha = F(B)). After that a candidate touches no global
// memory. Each candidate is sized with the Sec. 3 formulas in
// IEEE binary64 with explicit round-to-nearest intrinsics and no contraction
// (DESIGN R14; the library is also built with --fmad=false).
//
// Three launch shapes (plan-time choice):
//  * k3_cluster: the paper-size grids (<= 8 blocks x 256 threads x 4
//    candidates per model). One thread-block cluster per model; the blocks'
//    winners are reduced through distributed shared memory after one cluster
//    barrier -- no global atomics, fences or last-block protocol -- and rank 0
//    writes the winner's full record.
//  * k3_factored: large grids, argmin only. The instance counts factor over
//    the Cartesian grid: I_short depends on (g, C_S, B) only, I_long on
//    (g, C_L, B). A block owns (model, g, a tile of 32 B values, a chunk of
//    C_L values) x every C_S; it builds the two instance tables for its tile
//    in shared memory (the same IEEE operations as the per-candidate
//    evaluation, computed once) and then each candidate is one add, one
//    integer multiply, two DMULs and a compare. Winners meet through the
//    arrival protocol; the last block re-evaluates the winner in full.
//  * k3_grid: full records of large grids, and the three-pool grid (NEXT-2):
//    one candidate per thread, grid-stride, arrival protocol.
#include <cfloat>
#include <cmath>
#include <type_traits>
#include "internal.cuh"

namespace fp {

namespace {

constexpr double kInf = __builtin_huge_val();
constexpr unsigned long long kNoPool = 1ull << 62;   // factored tables: infeasible / invalid pool
constexpr unsigned long long kNoGpu = 1ull << 63;    // factored GPU-count tables: infeasible / invalid

// ---- shared-memory tables of one model ---------------------------------------
struct Tab {
  unsigned long long *cnt_le, *mass_le;   // [nbins] (after the scan)
  unsigned long long *nseq;               // [G][W]
  double *mu, *rmu;                       // [G][W]; rmu = RN(1/mu) or 0 (mdiv)
  unsigned long long *gpi;                // [G] GPUs per instance
  double *price;                          // [G]
  uint32_t *b, *cs, *cl;                  // grid values
  uint16_t *b_edge, *cl_edge, *b_win, *cs_win, *cl_win, *cs_edge;
  double rN;                              // RN(1/N) or 0
};

struct TabLayout {
  size_t cnt, mass, nseq, mu, rmu, gpi, price, b, cs, cl, be, ce, bw, sw, lw, se, bytes;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline TabLayout tab_layout(const EvalArgs &a, bool hist) {
  TabLayout L{};
  size_t o = 0;
  const size_t GW = (size_t)a.n_gpus * a.n_windows;
  L.cnt = o; o += hist ? al16((size_t)a.nbins * 8) : 0;
  L.mass = o; o += hist ? al16((size_t)a.nbins * 8) : 0;
  L.nseq = o; o += al16(GW * 8);
  L.mu = o; o += al16(GW * 8);
  L.rmu = o; o += al16(GW * 8);
  L.gpi = o; o += al16((size_t)a.n_gpus * 8);
  L.price = o; o += al16((size_t)a.n_gpus * 8);
  L.b = o; o += al16((size_t)a.n_b * 4);
  L.cs = o; o += al16((size_t)a.n_cs * 4);
  L.cl = o; o += al16((size_t)a.n_cl * 4);
  L.be = o; o += al16((size_t)a.n_b * 2);
  L.ce = o; o += al16((size_t)a.n_cl * 2);
  L.bw = o; o += al16((size_t)a.n_b * 2);
  L.sw = o; o += al16((size_t)a.n_cs * 2);
  L.lw = o; o += al16((size_t)a.n_cl * 2);
  L.se = o; o += al16((size_t)a.n_cs * 2);
  L.bytes = o;
  return L;
}

__device__ Tab tab_bind(const EvalArgs &a, unsigned char *smem, bool hist) {
  const TabLayout L = tab_layout(a, hist);
  Tab T;
  T.cnt_le = hist ? reinterpret_cast<unsigned long long *>(smem + L.cnt) : nullptr;
  T.mass_le = hist ? reinterpret_cast<unsigned long long *>(smem + L.mass) : nullptr;
  T.nseq = reinterpret_cast<unsigned long long *>(smem + L.nseq);
  T.mu = reinterpret_cast<double *>(smem + L.mu);
  T.rmu = reinterpret_cast<double *>(smem + L.rmu);
  T.gpi = reinterpret_cast<unsigned long long *>(smem + L.gpi);
  T.price = reinterpret_cast<double *>(smem + L.price);
  T.b = reinterpret_cast<uint32_t *>(smem + L.b);
  T.cs = reinterpret_cast<uint32_t *>(smem + L.cs);
  T.cl = reinterpret_cast<uint32_t *>(smem + L.cl);
  T.b_edge = reinterpret_cast<uint16_t *>(smem + L.be);
  T.cl_edge = reinterpret_cast<uint16_t *>(smem + L.ce);
  T.b_win = reinterpret_cast<uint16_t *>(smem + L.bw);
  T.cs_win = reinterpret_cast<uint16_t *>(smem + L.sw);
  T.cl_win = reinterpret_cast<uint16_t *>(smem + L.lw);
  T.cs_edge = reinterpret_cast<uint16_t *>(smem + L.se);
  T.rN = 0.0;
  return T;
}

// The plan's tables for model m (do not depend on the trace pass).
__device__ void load_plan_tables(const EvalArgs &a, const Tab &T, uint32_t m) {
  const uint32_t GW = a.n_gpus * a.n_windows;
  const uint64_t base = (uint64_t)m * GW;
  for (uint32_t j = threadIdx.x; j < GW; j += blockDim.x) {
    T.nseq[j] = a.cap_nseq[base + j];
    T.mu[j] = a.mu[base + j];
    T.rmu[j] = a.rmu[base + j];
  }
  for (uint32_t g = threadIdx.x; g < a.n_gpus; g += blockDim.x) {
    T.gpi[g] = a.deploy[((uint64_t)m * a.n_gpus + g) * 3 + 1];
    T.price[g] = a.price[g];
  }
  for (uint32_t j = threadIdx.x; j < a.n_b; j += blockDim.x) {
    T.b[j] = a.b[j];
    T.b_edge[j] = a.b_edge[j];
    T.b_win[j] = a.b_win[j];
  }
  for (uint32_t j = threadIdx.x; j < a.n_cs; j += blockDim.x) {
    T.cs[j] = a.cs[j];
    T.cs_win[j] = a.cs_win[j];
    T.cs_edge[j] = a.cs_edge[j];
  }
  for (uint32_t j = threadIdx.x; j < a.n_cl; j += blockDim.x) {
    T.cl[j] = a.cl[j];
    T.cl_edge[j] = a.cl_edge[j];
    T.cl_win[j] = a.cl_win[j];
  }
}

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
// savings / rho / predicted / occupancy divisions
template <bool FULL>
__device__ void evaluate(const EvalArgs &a, const Tab &T, uint32_t m, uint64_t idx, fp_candidate &c) {
  // decompose idx = (((m * G + g) * n_cl + l) * n_cs' + s) * n_b + k
  // 32-bit index math: the plan guarantees < 2^32 candidates
  uint32_t r = (uint32_t)idx, k, s, l, g;
  r = divmod(r, a.n_b, a.div_b, k);
  r = divmod(r, a.n_cs_eff, a.div_cs, s);
  r = divmod(r, a.n_cl, a.div_cl, l);
  divmod(r, a.n_gpus, a.div_g, g);
  uint32_t B = T.b[k], CL = T.cl[l];
  uint32_t CS = a.n_cs ? T.cs[s] : B;
  c.index = (uint32_t)idx; c.model = m; c.gpu = g;
  c.b_short = B; c.c_short = CS; c.c_long = CL; c.flags = 0; c._pad = 0;
  c.nseq_short = c.nseq_long = 0;
  c.n_short = c.n_long = c.n_reject = c.mass_short = c.mass_long = 0;
  c.inst_short = c.inst_long = c.inst_homo = c.gpus_dual = c.gpus_homo = 0;
  c.alpha = c.rho = c.predicted_savings = c.savings = 0.0;
  c.cost_dual = c.cost_homo = kInf;
  c.occupancy_short = c.occupancy_long = 0.0;
  if (!(B <= CS && CS <= CL)) return;  // invalid split

  const unsigned long long N = T.cnt_le[a.nbins - 1];
  const uint32_t eb = T.b_edge[k], el = T.cl_edge[l];
  const unsigned long long n_s = T.cnt_le[eb], n_sl = T.cnt_le[el];
  c.n_short = n_s;
  c.n_long = n_sl - n_s;
  c.n_reject = N - n_sl;
  c.mass_short = T.mass_le[eb];
  c.mass_long = T.mass_le[el] - T.mass_le[eb];

  const uint32_t ws = a.n_cs ? T.cs_win[s] : T.b_win[k];
  const uint32_t wl = T.cl_win[l];
  const uint32_t gw = g * a.n_windows;
  c.nseq_short = T.nseq[gw + ws];
  c.nseq_long = T.nseq[gw + wl];
  const double mu_s = T.mu[gw + ws], mu_l = T.mu[gw + wl];
  const double rmu_s = T.rmu[gw + ws], rmu_l = T.rmu[gw + wl];

  const double dN = u2d(N);
  c.alpha = mdiv(u2d(n_s), dN, T.rN);
  const double lam_s = __dmul_rn(c.alpha, a.rate);
  const double lam_l = __dmul_rn(mdiv(u2d(c.n_long), dN, T.rN), a.rate);
  const double lam_h = __dmul_rn(mdiv(u2d(n_sl), dN, T.rN), a.rate);

  const bool ok_s = pool_instances(lam_s, mu_s, rmu_s, c.nseq_short, &c.inst_short);
  const bool ok_l = pool_instances(lam_l, mu_l, rmu_l, c.nseq_long, &c.inst_long);
  const bool ok_h = pool_instances(lam_h, mu_l, rmu_l, c.nseq_long, &c.inst_homo);
  const bool ok_d = ok_s && ok_l;
  if (!ok_d) { c.inst_short = 0; c.inst_long = 0; }
  const unsigned long long gpi = T.gpi[g];
  c.gpus_dual = gpi * (c.inst_short + c.inst_long);
  c.gpus_homo = gpi * c.inst_homo;
  const double price = T.price[g];
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
__device__ void evaluate3(const EvalArgs &a, const Tab &T, uint32_t m, uint64_t idx, fp_pool3_candidate &c) {
  uint32_t r = (uint32_t)idx;
  const uint32_t p = r % a.n_pairs; r /= a.n_pairs;
  const uint32_t l = r % a.n_cl; r /= a.n_cl;
  const uint32_t g = r % a.n_gpus;
  const uint32_t pr = a.pairs[p], i = pr & 0xFFFFu, j = pr >> 16;
  const uint32_t B1 = T.b[i], B2 = T.b[j], CL = T.cl[l];
  c.index = (uint32_t)idx; c.model = m; c.gpu = g; c.b1 = B1; c.b2 = B2; c.c_long = CL;
  c.flags = 0; c._pad = 0;
  c.n1 = c.n2 = c.n3 = c.n_reject = 0;
  c.nseq1 = c.nseq2 = c.nseq3 = 0;
  c.inst1 = c.inst2 = c.inst3 = c.inst_homo = c.gpus = c.gpus_homo = 0;
  c.cost = c.cost_homo = kInf;
  c.savings = 0.0;
  if (!(B1 < B2 && B2 <= CL)) return;
  const unsigned long long N = T.cnt_le[a.nbins - 1];
  const unsigned long long c1 = T.cnt_le[T.b_edge[i]], c2 = T.cnt_le[T.b_edge[j]], c3 = T.cnt_le[T.cl_edge[l]];
  c.n1 = c1;
  c.n2 = c2 - c1;
  c.n3 = c3 - c2;
  c.n_reject = N - c3;
  const uint32_t gw = g * a.n_windows;
  const uint32_t w1 = gw + a.b_win3[i], w2 = gw + a.b_win3[j], w3 = gw + T.cl_win[l];
  c.nseq1 = T.nseq[w1];
  c.nseq2 = T.nseq[w2];
  c.nseq3 = T.nseq[w3];
  const double dN = u2d(N);
  const double lam1 = __dmul_rn(mdiv(u2d(c.n1), dN, T.rN), a.rate);
  const double lam2 = __dmul_rn(mdiv(u2d(c.n2), dN, T.rN), a.rate);
  const double lam3 = __dmul_rn(mdiv(u2d(c.n3), dN, T.rN), a.rate);
  const double lamh = __dmul_rn(mdiv(u2d(c3), dN, T.rN), a.rate);
  const bool ok1 = pool_instances(lam1, T.mu[w1], T.rmu[w1], c.nseq1, &c.inst1);
  const bool ok2 = pool_instances(lam2, T.mu[w2], T.rmu[w2], c.nseq2, &c.inst2);
  const bool ok3 = pool_instances(lam3, T.mu[w3], T.rmu[w3], c.nseq3, &c.inst3);
  const bool okh = pool_instances(lamh, T.mu[w3], T.rmu[w3], c.nseq3, &c.inst_homo);
  const bool ok = ok1 && ok2 && ok3;
  if (!ok) { c.inst1 = c.inst2 = c.inst3 = 0; }
  const unsigned long long gpi = T.gpi[g];
  c.gpus = gpi * (c.inst1 + c.inst2 + c.inst3);
  c.gpus_homo = gpi * c.inst_homo;
  const double price = T.price[g];
  if (ok) c.cost = __dmul_rn(__dmul_rn(u2d(c.gpus), price), a.hours);
  if (okh) c.cost_homo = __dmul_rn(__dmul_rn(u2d(c.gpus_homo), price), a.hours);
  if (ok && okh && c.gpus_homo > 0)
    c.savings = __ddiv_rn(__dsub_rn(u2d(c.gpus_homo), u2d(c.gpus)), u2d(c.gpus_homo));
  c.flags = FP_CAND_VALID | (ok ? FP_CAND_FEASIBLE : 0u) | (okh ? FP_CAND_HOMO_FEASIBLE : 0u);
}

template <bool POOL3> struct RecOf { using T = fp_candidate; };
template <> struct RecOf<true> { using T = fp_pool3_candidate; };

template <bool FULL = true>
__device__ __forceinline__ void eval_any(const EvalArgs &a, const Tab &T, uint32_t m, uint64_t idx,
                                         fp_candidate &c, double &cost) {
  evaluate<FULL>(a, T, m, idx, c);
  cost = c.cost_dual;
}
template <bool FULL = true>
__device__ __forceinline__ void eval_any(const EvalArgs &a, const Tab &T, uint32_t m, uint64_t idx,
                                         fp_pool3_candidate &c, double &cost) {
  evaluate3(a, T, m, idx, c);
  cost = c.cost;
}

// (cost, index) lexicographic min; non-candidates carry valid = 0.
__device__ __forceinline__ void better(double &c0, uint32_t &i0, uint32_t &v0, double c1, uint32_t i1,
                                       uint32_t v1) {
  bool take = v1 && (!v0 || c1 < c0 || (c1 == c0 && i1 < i0));
  if (take) { c0 = c1; i0 = i1; v0 = v1; }
}

// (cost, index) argmin of a warp by three 32-bit min reductions (REDUX):
// costs are >= +0 (GPUs x price x hours, price >= 0, hours > 0) or +inf, and
// the IEEE bit patterns of non-negative doubles order like their values, so
// (cost bits, index) compares lexicographically as (hi word, lo word, index).
// Non-candidates (v = 0) carry the all-ones key. Every lane gets the result.
__device__ __forceinline__ void warp_argmin_key(double &c, uint32_t &i, uint32_t &v) {
  const unsigned long long bits = v ? (unsigned long long)__double_as_longlong(c) : ~0ull;
  const uint32_t hi = (uint32_t)(bits >> 32), lo = (uint32_t)bits, ix = v ? i : 0xffffffffu;
  const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
  const uint32_t mi = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? ix : 0xffffffffu);
  v = __reduce_or_sync(0xffffffffu, (v && hi == mh && lo == ml && ix == mi) ? 1u : 0u);
  c = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
  i = mi;
}

// block-wide (cost, index) argmin; the result is valid in warp 0 (every lane)
__device__ void block_argmin(double &bc, uint32_t &bi, uint32_t &bv, double *red_c, uint32_t *red_i,
                             uint32_t *red_v) {
  warp_argmin_key(bc, bi, bv);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) { red_c[w] = bc; red_i[w] = bi; red_v[w] = bv; }
  __syncthreads();
  if (w == 0) {
    bc = lane < nw ? red_c[lane] : 0.0;
    bi = lane < nw ? red_i[lane] : 0xffffffffu;
    bv = lane < nw ? red_v[lane] : 0u;
    warp_argmin_key(bc, bi, bv);
  }
}

// Block-wide inclusive scan of data[0..n) in shared memory.
__device__ void block_scan_inclusive(unsigned long long *data, uint32_t n, unsigned long long *warp_tot) {
  // each thread owns a contiguous run of ceil(n / blockDim) elements
  const uint32_t T = blockDim.x, t = threadIdx.x;
  const uint32_t per = (n + T - 1) / T;
  const uint32_t lo = min(n, t * per), hi = min(n, lo + per);
  unsigned long long run = 0;
  for (uint32_t j = lo; j < hi; ++j) run += data[j];
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
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// diagnostic phase stamps of block (0, 0), thread 0 (EvalArgs::phase_ts, env FP_K3_PHASES)
__device__ __forceinline__ void phase(const EvalArgs &a, int i) {
  if (a.phase_ts && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) a.phase_ts[i] = globaltimer();
}

// Prologue shared by every K3 shape: the plan tables (before the PDL wait),
// the histogram of this sweep, its scan and RN(1/N). `first` marks the one
// block that publishes the summed histogram and clears the other parity's
// accumulator copies (last read by the previous sweep, which completed
// before this sweep's trace pass started: the trace pass is a plain launch).
__device__ void prologue(const EvalArgs &a, Tab &T, uint32_t m, bool first, unsigned long long *warp_tot) {
  phase(a, 0);
  // the next kernel (K4p / K4b / K4v, or the speculative full trace pass) may be
  // scheduled now: each of them waits (griddepcontrol.wait) before it reads
  // anything this kernel writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  load_plan_tables(a, T, m);
  if (first && a.zero_copies) {
    for (size_t i = threadIdx.x; i < a.zero_elems; i += blockDim.x) a.zero_copies[i] = 0ull;
  }
  phase(a, 1);
  // the trace pass's histogram is complete and visible after this (no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // FP_FLAG_SPECULATE: the sample's accumulators, for the next step's sample
  // pass. Only past the wait: this K3 may start while the full trace pass
  // still waits for the sample's K3, which reads them
  if (first && a.zero_copies2) {
    for (size_t i = threadIdx.x; i < a.zero_elems; i += blockDim.x) a.zero_copies2[i] = 0ull;
  }
  phase(a, 2);
  if (a.p2p_world) {
    // peer-memory exchange (FP_FLAG_P2P): wait until every rank has published
    // this step's folded histogram (its K1 done, fenced system-wide), then
    // read all ranks' histograms directly -- the cross-rank sum fused into
    // this prologue. The wait is bounded: a rank that never publishes sets
    // the plan's error word (FP_ERR_NCCL at the next synchronising call).
    if (threadIdx.x < a.p2p_world) {
      const unsigned int *f = a.peer_flag[threadIdx.x];
      const unsigned long long t0 = globaltimer();
      unsigned int v;
      for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int)(v - a.p2p_epoch) >= 0) break;
        if (globaltimer() - t0 > a.p2p_timeout_ns) {
          atomicOr(a.err_word, 1u + (threadIdx.x << 8));
          break;
        }
        __nanosleep(128);
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < a.nbins; j += blockDim.x) {
      unsigned long long cnt = 0, mass = 0;
      for (uint32_t r = 0; r < a.p2p_world; ++r) {
        const unsigned long long *h = a.peer_hist[r] + a.p2p_off;
        cnt += __ldcv(h + j);
        mass += __ldcv(h + a.nbins + j);
      }
      T.cnt_le[j] = cnt;
      T.mass_le[j] = mass;
    }
  } else if (a.hist_copies == 16) {
    for (uint32_t j = threadIdx.x; j < a.nbins; j += blockDim.x) {
      // all 32 loads in flight at once (one L2 round trip, not sixteen)
      unsigned long long vc[16], vm[16], cnt = 0, mass = 0;
#pragma unroll
      for (uint32_t c = 0; c < 16; ++c) {
        vc[c] = a.hist_cnt[(size_t)c * 2 * a.nbins + j];
        vm[c] = a.hist_mass[(size_t)c * 2 * a.nbins + j];
      }
#pragma unroll
      for (uint32_t c = 0; c < 16; ++c) { cnt += vc[c]; mass += vm[c]; }
      T.cnt_le[j] = cnt;
      T.mass_le[j] = mass;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < a.nbins; j += blockDim.x) {
      unsigned long long cnt = 0, mass = 0;
      for (uint32_t c = 0; c < a.hist_copies; ++c) {
        cnt += a.hist_cnt[(size_t)c * 2 * a.nbins + j];
        mass += a.hist_mass[(size_t)c * 2 * a.nbins + j];
      }
      T.cnt_le[j] = cnt;
      T.mass_le[j] = mass;
    }
  }
  if (first && a.hist_out) {
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < a.nbins; j += blockDim.x) {
      a.hist_out[j] = T.cnt_le[j];
      a.hist_out[a.nbins + j] = T.mass_le[j];
    }
  }
  __syncthreads();
  phase(a, 3);
  if (a.nbins <= 256) {
    // one warp scans both arrays (<= 8 contiguous bins per lane): no block barriers
    if (threadIdx.x < 32) {
      const uint32_t lane = threadIdx.x, per = (a.nbins + 31) / 32;
      const uint32_t lo = min(a.nbins, lane * per), hi = min(a.nbins, lo + per);
      unsigned long long rc = 0, rm = 0;
      for (uint32_t j = lo; j < hi; ++j) { rc += T.cnt_le[j]; rm += T.mass_le[j]; }
      unsigned long long xc = rc, xm = rm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long yc = __shfl_up_sync(0xffffffffu, xc, o);
        const unsigned long long ym = __shfl_up_sync(0xffffffffu, xm, o);
        if (lane >= (uint32_t)o) { xc += yc; xm += ym; }
      }
      unsigned long long oc = xc - rc, om = xm - rm;
      for (uint32_t j = lo; j < hi; ++j) {
        oc += T.cnt_le[j]; T.cnt_le[j] = oc;
        om += T.mass_le[j]; T.mass_le[j] = om;
      }
      // N = the last lane's inclusive count; RN(1/N) formed once, shared below
      const unsigned long long N = __shfl_sync(0xffffffffu, xc, 31);
      if (lane == 0) warp_tot[0] = (unsigned long long)__double_as_longlong(mrcp(u2d(N)));
    }
  } else {
    block_scan_inclusive(T.cnt_le, a.nbins, warp_tot);
    __syncthreads();
    block_scan_inclusive(T.mass_le, a.nbins, warp_tot);
    __syncthreads();
    if (threadIdx.x == 0) warp_tot[0] = (unsigned long long)__double_as_longlong(mrcp(u2d(T.cnt_le[a.nbins - 1])));
  }
  __syncthreads();
  T.rN = __longlong_as_double((long long)warp_tot[0]);
  __syncthreads();                       // warp_tot is reused by the caller
  phase(a, 4);
}

// The empty record of a model without a feasible candidate.
__device__ void no_winner(fp_candidate &c, uint32_t m) {
  memset(&c, 0, sizeof c);
  c.index = 0xffffffffu;
  c.model = m;
  c.cost_dual = c.cost_homo = kInf;
}

// sweep_and_route: the routed split's edge indices #{e in E : e < v} for its
// B, C_S, C_L -- the positions of those values in E (they are edges), read
// from the plan's index tables -- and whether it is feasible.
__device__ void emit_route(const EvalArgs &a, const Tab &T, uint32_t bi, uint32_t bv) {
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (bv) {
    uint32_t r = bi, k, s, l;
    r = divmod(r, a.n_b, a.div_b, k);
    r = divmod(r, a.n_cs_eff, a.div_cs, s);
    divmod(r, a.n_cl, a.div_cl, l);
    v = make_uint4(T.b_edge[k], a.n_cs ? T.cs_edge[s] : T.b_edge[k], T.cl_edge[l], 1u);
  }
  *reinterpret_cast<uint4 *>(a.route_out) = v;
}

// The winner's record, evaluated in full by one thread (grid-stride shapes).
__device__ void emit_winner(const EvalArgs &a, const Tab &T, uint32_t m, uint32_t bi, uint32_t bv) {
  fp_candidate c;
  if (bv) evaluate<true>(a, T, m, bi, c);
  else no_winner(c, m);
  a.best_out[m] = c;
  if (a.route_out && m == a.route_model) emit_route(a, T, bi, bv);
}

// ---- cluster-scope helpers (PTX) ------------------------------------------------
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t dsmem_addr(const void *p, uint32_t rank) {
  uint32_t local = (uint32_t)__cvta_generic_to_shared(p), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  return remote;
}
__device__ __forceinline__ double ld_dsmem_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_dsmem_u64(uint32_t addr) {
  unsigned long long v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}

// ---- latency shape: one cluster of gridDim.x blocks per model -------------------
// Every thread evaluates its (<= 4) candidates in full and keeps its best
// record in its shared-memory slot; the blocks' winners meet in rank 0 through
// DSMEM after one cluster barrier, and rank 0 copies the winning record out of
// its owner's slot (the owner follows from the index: no re-evaluation).
template <bool RESULTS>
__global__ void __launch_bounds__(256) k3_cluster(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long warp_tot[32];
  __shared__ double red_c[32];
  __shared__ uint32_t red_i[32], red_v[32];
  __shared__ double win_c;
  __shared__ uint32_t win_i, win_v;
  const uint32_t m = blockIdx.y, rank = blockIdx.x;   // cluster (gridDim.x, 1, 1): rank = blockIdx.x
  Tab T = tab_bind(a, smem, true);
  fp_candidate *slot = reinterpret_cast<fp_candidate *>(smem + tab_layout(a, true).bytes);
  prologue(a, T, m, rank == 0 && m == 0, warp_tot);

  const uint64_t m_lo = (uint64_t)m * a.per_model, m_hi = m_lo + a.per_model;
  const uint64_t lo = max(m_lo, a.cand_first), hi = min(m_hi, a.cand_first + a.cand_count);
  double bc = 0.0;
  uint32_t bi = 0xffffffffu, bv = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t idx = lo + (uint64_t)rank * blockDim.x + threadIdx.x; idx < hi; idx += stride) {
    fp_candidate c;
    evaluate<true>(a, T, m, idx, c);
    if (RESULTS) a.results[idx - a.cand_first] = c;
    // indices increase along the loop, so strict '<' keeps the lowest index on ties
    if ((c.flags & FP_CAND_FEASIBLE) && (!bv || c.cost_dual < bc)) {
      bc = c.cost_dual; bi = c.index; bv = 1;
      slot[threadIdx.x] = c;
    }
  }
  phase(a, 5);
  block_argmin(bc, bi, bv, red_c, red_i, red_v);
  if (threadIdx.x == 0) { win_c = bc; win_i = bi; win_v = bv; }
  phase(a, 6);
  // every block's winner (and its record) is in its shared memory: one cluster barrier
  cluster_arrive();
  cluster_wait();
  phase(a, 7);
  if (rank != 0) {
    // keep this block's shared memory alive until rank 0 has read it
    cluster_arrive();
    cluster_wait();
    return;
  }
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    double c = 0.0;
    uint32_t i = 0xffffffffu, v = 0;
    if (lane < gridDim.x) {
      c = ld_dsmem_f64(dsmem_addr(&win_c, lane));
      i = ld_dsmem_u32(dsmem_addr(&win_i, lane));
      v = ld_dsmem_u32(dsmem_addr(&win_v, lane));
    }
    warp_argmin_key(c, i, v);
    phase(a, 8);
    // the record: owner block and thread from the loop's index mapping
    constexpr uint32_t kWords = sizeof(fp_candidate) / 8;
    if (v) {
      const uint64_t off = (uint64_t)i - lo;
      const uint32_t r = (uint32_t)(off % stride), owner = r / blockDim.x, t = r % blockDim.x;
      if (lane < kWords) {
        const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&slot[t]) + lane;
        reinterpret_cast<unsigned long long *>(a.best_out + m)[lane] = ld_dsmem_u64(dsmem_addr(src, owner));
      }
    } else if (lane == 0) {
      fp_candidate e;
      no_winner(e, m);
      a.best_out[m] = e;
    }
    if (lane == 0 && a.route_out && m == a.route_model) emit_route(a, T, i, v);
  }
  phase(a, 9);
  cluster_arrive();                     // the other blocks may exit now
  cluster_wait();
}

// ---- arrival protocol of the grid-stride shapes ---------------------------------------
// Block winner -> block_best[m][blockIdx.x]; the last block of model m to
// arrive reduces them. Returns true in the last block (its thread 0 holds the
// model's winner).
__device__ bool arrive_last(BlockBest *bbase, unsigned int *done, uint32_t m, double &bc, uint32_t &bi,
                            uint32_t &bv, double *red_c, uint32_t *red_i, uint32_t *red_v) {
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    BlockBest *bb = bbase + (size_t)m * gridDim.x + blockIdx.x;
    bb->cost = bc; bb->index = bi; bb->valid = bv;
    if (gridDim.x == 1) {
      is_last = true;                 // one block per model: no arrival protocol
    } else {
      __threadfence();
      unsigned int prev = atomicAdd(done + m, 1u);
      is_last = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!is_last) return false;
  if (gridDim.x > 1) __threadfence();
  bc = 0.0; bi = 0xffffffffu; bv = 0;
  for (uint32_t j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
    const volatile BlockBest *bb = bbase + (size_t)m * gridDim.x + j;
    better(bc, bi, bv, bb->cost, bb->index, bb->valid);
  }
  __syncthreads();
  block_argmin(bc, bi, bv, red_c, red_i, red_v);
  if (threadIdx.x == 0) done[m] = 0;     // self-reset for the next launch / graph replay
  return true;
}

// ---- grid-stride shape: full records of large grids, and the three-pool grid ----------
template <bool POOL3>
__global__ void __launch_bounds__(256, 3) k3_grid(EvalArgs a) {
  using Rec = typename RecOf<POOL3>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long warp_tot[32];
  __shared__ double red_c[32];
  __shared__ uint32_t red_i[32], red_v[32];
  const uint32_t m = blockIdx.y;
  Tab T = tab_bind(a, smem, true);
  prologue(a, T, m, blockIdx.x == 0 && m == 0, warp_tot);

  const uint64_t per = POOL3 ? a.per_model3 : a.per_model;
  const uint64_t m_lo = (uint64_t)m * per, m_hi = m_lo + per;
  // the three-pool grid is evaluated whole on every rank (replicated)
  const uint64_t lo = POOL3 ? m_lo : max(m_lo, a.cand_first);
  const uint64_t hi = POOL3 ? m_hi : min(m_hi, a.cand_first + a.cand_count);
  double bc = 0.0;
  uint32_t bi = 0xffffffffu, bv = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool want = POOL3 ? a.results3 != nullptr : a.results != nullptr;
  if (want) {
    for (uint64_t idx = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < hi; idx += stride) {
      Rec c;
      double cost;
      eval_any<true>(a, T, m, idx, c, cost);
      if (POOL3) reinterpret_cast<Rec *>(a.results3)[idx] = c;
      else reinterpret_cast<Rec *>(a.results)[idx - a.cand_first] = c;
      if ((c.flags & FP_CAND_FEASIBLE) && (!bv || cost < bc)) { bc = cost; bi = c.index; bv = 1; }
    }
  } else {
    for (uint64_t idx = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < hi; idx += stride) {
      Rec c;
      double cost;
      eval_any<false>(a, T, m, idx, c, cost);
      if ((c.flags & FP_CAND_FEASIBLE) && (!bv || cost < bc)) { bc = cost; bi = c.index; bv = 1; }
    }
  }
  block_argmin(bc, bi, bv, red_c, red_i, red_v);
  if (!arrive_last(POOL3 ? a.block_best3 : a.block_best, POOL3 ? a.done3 : a.done, m, bc, bi, bv, red_c,
                   red_i, red_v))
    return;
  if constexpr (POOL3) {
    if (threadIdx.x == 0) {
      Rec c;
      double cost;
      if (bv) {
        eval_any(a, T, m, bi, c, cost);
      } else {
        memset(&c, 0, sizeof c);
        c.index = 0xffffffffu;
        c.model = m;
        c.cost = c.cost_homo = kInf;
      }
      a.best3[m] = c;
    }
  } else {
    if (threadIdx.x == 0) emit_winner(a, T, m, bi, bv);
  }
}

// ---- factored shape: large grids, argmin only ------------------------------------------
// blockIdx.x = (g * n_lc + lc) * n_kt + kt: B tile kt (32 values, one per
// lane), C_L chunk lc (a.fac_lc values), GPU g; every C_S. Shared tables:
//   Is[s][32] = I_short(g, C_S[s], B[k])   (kNoPool: infeasible or B > C_S)
//   Il[lc][32] = I_long(g, C_L[l], B[k])   (kNoPool: infeasible)
// built with the per-candidate evaluation's operations (identical values).
constexpr int kMaxLC = 64;                 // EvalArgs::fac_lc <= kMaxLC

__device__ __forceinline__ unsigned long long short_instances(const EvalArgs &a, const Tab &T, uint32_t g, uint32_t s,
                                                              uint32_t k) {
  const uint32_t B = T.b[k];
  const uint32_t CS = a.n_cs ? T.cs[s] : B;
  if (!(B <= CS)) return kNoPool;
  const uint32_t w = g * a.n_windows + (a.n_cs ? T.cs_win[s] : T.b_win[k]);
  const double alpha = mdiv(u2d(T.cnt_le[T.b_edge[k]]), u2d(T.cnt_le[a.nbins - 1]), T.rN);
  uint64_t inst;
  return pool_instances(__dmul_rn(alpha, a.rate), T.mu[w], T.rmu[w], T.nseq[w], &inst) ? inst : kNoPool;
}

__device__ __forceinline__ unsigned long long long_instances(const EvalArgs &a, const Tab &T, uint32_t g, uint32_t l,
                                                             uint32_t k) {
  const uint32_t w = g * a.n_windows + T.cl_win[l];
  const unsigned long long n_long = T.cnt_le[T.cl_edge[l]] - T.cnt_le[T.b_edge[k]];
  const double lam = __dmul_rn(mdiv(u2d(n_long), u2d(T.cnt_le[a.nbins - 1]), T.rN), a.rate);
  uint64_t inst;
  return pool_instances(lam, T.mu[w], T.rmu[w], T.nseq[w], &inst) ? inst : kNoPool;
}

__global__ void __launch_bounds__(256, 2) k3_factored(EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long warp_tot[32];
  __shared__ double red_c[32];
  __shared__ uint32_t red_i[32], red_v[32];
  const uint32_t m = blockIdx.y;
  Tab T = tab_bind(a, smem, true);
  unsigned long long *Is = reinterpret_cast<unsigned long long *>(smem + tab_layout(a, true).bytes);
  unsigned long long *Il = Is + (size_t)a.n_cs_eff * 32;
  prologue(a, T, m, blockIdx.x == 0 && m == 0, warp_tot);

  const uint32_t LC = a.fac_lc;
  const uint32_t n_kt = (a.n_b + 31) / 32, n_lc = (a.n_cl + LC - 1) / LC;
  const uint32_t kt = blockIdx.x % n_kt, lc = (blockIdx.x / n_kt) % n_lc, g = blockIdx.x / (n_kt * n_lc);
  const uint32_t l0 = lc * LC, nl = min(LC, a.n_cl - l0);
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t k = kt * 32 + lane;
  const bool kin = k < a.n_b;
  const unsigned long long gpi = T.gpi[g];
  // the GPU-count tables of this tile: gpi x I_short, gpi x I_long, bit 63 set
  // when the pool is infeasible (or B > C_S). gpi x I <= 2^9 x 2^53, so a
  // valid entry never has bit 63; gpi (I_s + I_l) = gpi I_s + gpi I_l mod 2^64
  // as in the per-candidate evaluation
  __shared__ uint32_t gmax_s, gmax_l, gmax_big, cs_unsorted, s_hi[kMaxLC];
  if (threadIdx.x == 0) { gmax_s = 0u; gmax_l = 0u; gmax_big = 0u; cs_unsorted = 0u; }
  __syncthreads();
  unsigned long long ms = 0ull, ml = 0ull;       // largest feasible table entries
  for (uint32_t e = threadIdx.x; e < a.n_cs_eff * 32; e += blockDim.x) {
    const uint32_t kk = kt * 32 + (e & 31);
    const unsigned long long v = kk < a.n_b ? short_instances(a, T, g, e >> 5, kk) : kNoPool;
    Is[e] = v == kNoPool ? kNoGpu : gpi * v;
    if (v != kNoPool) ms = max(ms, gpi * v);
  }
  for (uint32_t e = threadIdx.x; e < nl * 32; e += blockDim.x) {
    const uint32_t kk = kt * 32 + (e & 31);
    const unsigned long long v = kk < a.n_b ? long_instances(a, T, g, l0 + (e >> 5), kk) : kNoPool;
    Il[e] = v == kNoPool ? kNoGpu : gpi * v;
    if (v != kNoPool) ml = max(ml, gpi * v);
  }
  // independent C_S grid: the C_S values <= C_L of chunk entry li are a prefix
  // [0, s_hi[li]) when the grid is ascending (checked here)
  if (a.n_cs) {
    for (uint32_t s = threadIdx.x; s + 1 < a.n_cs; s += blockDim.x)
      if (T.cs[s] > T.cs[s + 1]) cs_unsorted = 1u;
    for (uint32_t li = threadIdx.x; li < nl; li += blockDim.x) {
      uint32_t c = 0;
      while (c < a.n_cs && T.cs[c] <= T.cl[l0 + li]) ++c;
      s_hi[li] = c;
    }
  }
  // block maxima in u32 (an upper bound is all the test below needs); an entry
  // of 2^32 or more disables the integer argmin for the block
  {
    const uint32_t s32 = __reduce_max_sync(0xffffffffu, (uint32_t)min(ms, 0xffffffffull));
    const uint32_t l32 = __reduce_max_sync(0xffffffffu, (uint32_t)min(ml, 0xffffffffull));
    const bool big = __any_sync(0xffffffffu, (ms | ml) >> 32);
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&gmax_s, s32);
      atomicMax(&gmax_l, l32);
      if (big) gmax_big = 1u;
    }
  }
  __syncthreads();

  const uint64_t m_lo = (uint64_t)m * a.per_model;
  const uint64_t lo = max(m_lo, a.cand_first), hi = min(m_lo + a.per_model, a.cand_first + a.cand_count);
  const double price = T.price[g], hours = a.hours;
  const uint32_t B = kin ? T.b[k] : 0xffffffffu;
  // flat index = idx0 + q n_b, q = li n_cs' + s; for a fixed lane (k) the
  // loops below visit q in increasing order, so strict '<' keeps the lowest index
  const uint32_t ncs = a.n_cs_eff;
  const uint64_t idx0 = m_lo + ((uint64_t)g * a.n_cl + l0) * ncs * a.n_b + k;
  const uint64_t tile_lo = idx0 - lane, tile_hi = tile_lo + ((uint64_t)nl * ncs - 1) * a.n_b + 31;
  const bool whole = tile_lo >= lo && tile_hi < hi;      // no per-candidate slice check
  double bc = 0.0;
  uint32_t bq = 0, bv = 0;
  auto scan = [&](auto check) {
    for (uint32_t li = w; li < nl; li += nw) {
      const unsigned long long gl = Il[li * 32 + lane];
      if (gl >> 63) continue;
      const uint32_t CL = T.cl[l0 + li], qb = li * ncs;
#pragma unroll 4
      for (uint32_t s = 0; s < ncs; ++s) {
        const unsigned long long gs = Is[s * 32 + lane];
        const uint32_t CS = a.n_cs ? T.cs[s] : B;
        bool ok = !(gs >> 63) && CS <= CL;
        if (decltype(check)::value) {
          const uint64_t idx = idx0 + (uint64_t)(qb + s) * a.n_b;
          ok = ok && idx >= lo && idx < hi;
        }
        if (ok) {
          const double cost = __dmul_rn(__dmul_rn(u2d(gs + gl), price), hours);
          if (!bv || cost < bc) { bc = cost; bq = qb + s; bv = 1; }
        }
      }
    }
  };
  // Integer argmin. For this block's GPU the cost is RN(RN(G price) hours) of
  // the candidate's GPU count G = gpi (I_short + I_long), monotone in G; it is
  // STRICTLY monotone (distinct G -> distinct costs, so the (cost, index)
  // argmin is the (G, index) argmin) when the products stay far from fp64's
  // precision: price >= 1/32, hours >= 1, G price <= 2^40 and G price hours
  // <= 2^44 for every G of this block (bounded by the tables' largest feasible
  // entries) -- then RN(G2 p) - RN(G1 p) >= p - 2^-11 > 1/64 and the product
  // with hours keeps a gap > 2 ulp(2^44) = 1/128. Each candidate is then one
  // 64-bit add and compare on the integer pipes (an infeasible table entry
  // carries bit 63, so its sum never beats the initial 2^63); the winner's
  // cost is formed once, with the same operations as evaluate().
  const double gbound = u2d((unsigned long long)gmax_s + gmax_l);
  const bool int_argmin = !gmax_big && !(a.n_cs && cs_unsorted) && price >= 0.03125 && hours >= 1.0 &&
                          __dmul_rn(gbound, price) <= 1099511627776.0 &&
                          __dmul_rn(__dmul_rn(gbound, price), hours) <= 17592186044416.0;
  if (kin && whole && int_argmin) {
    unsigned long long bg = kNoGpu;
    for (uint32_t li = w; li < nl; li += nw) {
      const unsigned long long gl = Il[li * 32 + lane];
      if (gl >> 63) continue;
      const uint32_t qb = li * ncs;
      uint32_t s_end = ncs;
      if (a.n_cs) s_end = s_hi[li];
      else if (B > T.cl[l0 + li]) continue;        // C_S = B <= C_L
#pragma unroll 8
      for (uint32_t s = 0; s < s_end; ++s) {
        const unsigned long long G = Is[s * 32 + lane] + gl;
        if (G < bg) { bg = G; bq = qb + s; }
      }
    }
    if (bg < kNoGpu) { bv = 1; bc = __dmul_rn(__dmul_rn(u2d(bg), price), hours); }
  } else if (kin) {
    if (whole) scan(std::false_type{});
    else scan(std::true_type{});
  }
  uint32_t bi = bv ? (uint32_t)(idx0 + (uint64_t)bq * a.n_b) : 0xffffffffu;
  block_argmin(bc, bi, bv, red_c, red_i, red_v);
  if (!arrive_last(a.block_best, a.done, m, bc, bi, bv, red_c, red_i, red_v)) return;
  if (threadIdx.x == 0) emit_winner(a, T, m, bi, bv);
}

// N_seq (Eq. 2) and RN(1/mu) for every (model, GPU, window): plan data only, computed once
__global__ void k_capacity(EvalArgs a, unsigned long long *cap, double *rmu) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (uint64_t)a.n_models * a.n_gpus * a.n_windows) return;
  const uint32_t w = (uint32_t)(j % a.n_windows), g = (uint32_t)(j / a.n_windows % a.n_gpus);
  const uint32_t m = (uint32_t)(j / ((uint64_t)a.n_windows * a.n_gpus));
  const unsigned long long *dp = a.deploy + ((uint64_t)m * a.n_gpus + g) * 3;
  cap[j] = max_seqs(kv_budget(a.gpu_u64 + 4 * g, dp[2]), (uint32_t)dp[0], a.model_arch + 4 * m, a.windows[w]);
  rmu[j] = mrcp(a.mu[j]);
}

// NEXT-4: peak-window sizing. Same grid and index decomposition
// as evaluate(); the routing counts of a pool become its busiest window's
// counts (max over windows of the cumulative per-window histogram), the rates
// peak * (1e9 / window_ns), and each pool is sized with the Sec. 3 formula in
// the oracle's operation order (or_sweep_peak).
__device__ void evaluate_peak(const EvalArgs &a, const Tab &T, uint32_t m, uint64_t idx, fp_peak_candidate &c) {
  uint32_t r = (uint32_t)idx, k, s, l, g;
  r = divmod(r, a.n_b, a.div_b, k);
  r = divmod(r, a.n_cs_eff, a.div_cs, s);
  r = divmod(r, a.n_cl, a.div_cl, l);
  divmod(r, a.n_gpus, a.div_g, g);
  const uint32_t B = T.b[k], CL = T.cl[l], CS = a.n_cs ? T.cs[s] : B;
  c.index = (uint32_t)idx; c.model = m; c.gpu = g; c.b_short = B; c.c_short = CS; c.c_long = CL;
  c.flags = 0; c._pad = 0;
  c.peak_short = c.peak_long = c.peak_homo = 0;
  c.inst_short = c.inst_long = c.inst_homo = c.gpus_dual = c.gpus_homo = 0;
  c.lambda_short = c.lambda_long = c.lambda_homo = 0.0;
  c.cost_dual = c.cost_homo = kInf;
  c.savings = 0.0;
  if (!(B <= CS && CS <= CL)) return;
  const uint32_t eb = T.b_edge[k], el = T.cl_edge[l];
  // busiest-window counts, reduced over windows by K2w (k_peak.cu)
  const unsigned long long ps = a.colmax_pk[eb], ph = a.colmax_pk[el], pl = a.pairmax_pk[k * a.n_cl + l];
  c.peak_short = ps; c.peak_long = pl; c.peak_homo = ph;
  const uint32_t ws = a.n_cs ? T.cs_win[s] : T.b_win[k], wl = T.cl_win[l];
  const uint32_t gw = g * a.n_windows;
  const unsigned long long nseq_s = T.nseq[gw + ws], nseq_l = T.nseq[gw + wl];
  c.lambda_short = __dmul_rn(u2d(ps), a.inv_w_s);
  c.lambda_long = __dmul_rn(u2d(pl), a.inv_w_s);
  c.lambda_homo = __dmul_rn(u2d(ph), a.inv_w_s);
  const bool ok_s = pool_instances(c.lambda_short, T.mu[gw + ws], T.rmu[gw + ws], nseq_s, &c.inst_short);
  const bool ok_l = pool_instances(c.lambda_long, T.mu[gw + wl], T.rmu[gw + wl], nseq_l, &c.inst_long);
  const bool ok_h = pool_instances(c.lambda_homo, T.mu[gw + wl], T.rmu[gw + wl], nseq_l, &c.inst_homo);
  const bool ok_d = ok_s && ok_l;
  if (!ok_d) { c.inst_short = 0; c.inst_long = 0; }
  const unsigned long long gpi = T.gpi[g];
  c.gpus_dual = gpi * (c.inst_short + c.inst_long);
  c.gpus_homo = gpi * c.inst_homo;
  const double price = T.price[g];
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
  const uint32_t m = blockIdx.y;
  const Tab T = tab_bind(a, smem, false);
  load_plan_tables(a, T, m);
  asm volatile("griddepcontrol.wait;" ::: "memory");   // K2w's window maxima (PDL launch)
  __syncthreads();
  const uint64_t lo = (uint64_t)m * a.per_model, hi = lo + a.per_model;
  double bc = 0.0;
  uint32_t bi = 0xffffffffu, bv = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t idx = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < hi; idx += stride) {
    fp_peak_candidate c;
    evaluate_peak(a, T, m, idx, c);
    if (a.results_pk) a.results_pk[idx] = c;
    if ((c.flags & FP_CAND_FEASIBLE) && (!bv || c.cost_dual < bc)) { bc = c.cost_dual; bi = c.index; bv = 1; }
  }
  block_argmin(bc, bi, bv, red_c, red_i, red_v);
  if (!arrive_last(a.block_best_pk, a.done_pk, m, bc, bi, bv, red_c, red_i, red_v)) return;
  if (threadIdx.x == 0) {
    fp_peak_candidate c;
    if (bv) {
      evaluate_peak(a, T, m, bi, c);
    } else {
      memset(&c, 0, sizeof c);
      c.index = 0xffffffffu;
      c.model = m;
      c.cost_dual = c.cost_homo = kInf;
    }
    a.best_pk[m] = c;
  }
}

// after K1 (stream order): sum the trace pass's accumulator copies into one
// [2][nbins] histogram (out), for the cross-rank exchange. With flag != NULL
// (FP_FLAG_P2P) make it visible system-wide and publish the step's epoch
// (release) for the peers' K3 prologues.
__global__ void k_fold(const unsigned long long *copies, uint32_t n_copies, uint32_t nbins, unsigned long long *out,
                       unsigned int *flag, unsigned int epoch) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // K1's accumulators (PDL launch)
  for (uint32_t j = threadIdx.x; j < 2 * nbins; j += blockDim.x) {
    const uint32_t h = j / nbins, b = j - h * nbins;
    unsigned long long v = 0;
    for (uint32_t c = 0; c < n_copies; ++c) v += copies[((size_t)c * 2 + h) * nbins + b];
    out[j] = v;
  }
  if (flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    }
  }
}

}  // namespace

// ---- host side --------------------------------------------------------------------------
size_t eval_smem_bytes(const EvalArgs &a, int) { return tab_layout(a, true).bytes; }
size_t eval_factored_smem_bytes(const EvalArgs &a) {
  return tab_layout(a, true).bytes + ((size_t)a.n_cs_eff + a.fac_lc) * 32 * 8;
}
size_t eval_peak_smem_bytes(const EvalArgs &a) { return tab_layout(a, false).bytes; }
uint32_t eval_factored_blocks_per_model(const EvalArgs &a) {
  return a.n_gpus * ((a.n_cl + a.fac_lc - 1) / a.fac_lc) * ((a.n_b + 31) / 32);
}

cudaError_t eval_prepare() {
  const int big = 200 * 1024;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k3_grid<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big))) return e;
  if ((e = cudaFuncSetAttribute(k3_grid<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big))) return e;
  if ((e = cudaFuncSetAttribute(k3_cluster<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big))) return e;
  if ((e = cudaFuncSetAttribute(k3_cluster<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big))) return e;
  if ((e = cudaFuncSetAttribute(k3_factored, cudaFuncAttributeMaxDynamicSharedMemorySize, big))) return e;
  return cudaFuncSetAttribute(k3_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

cudaError_t launch_capacity(const EvalArgs &a, unsigned long long *cap, double *rmu, cudaStream_t s) {
  const uint64_t n = (uint64_t)a.n_models * a.n_gpus * a.n_windows;
  k_capacity<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, cap, rmu);
  return cudaGetLastError();
}

cudaError_t launch_fold(const unsigned long long *copies, uint32_t n_copies, uint32_t nbins, unsigned long long *out,
                        unsigned int *flag, unsigned int epoch, cudaStream_t s) {
  return launch_pdl(k_fold, dim3(1), dim3(256), 0, s, copies, n_copies, nbins, out, flag, epoch);
}

// K3 after K1 as a programmatic dependent launch: its blocks are scheduled as
// K1's blocks exit and wait (griddepcontrol.wait) only before the histogram
// reads, which hides the launch latency and the table loads (FP_NO_PDL=1: a
// plain launch).
cudaError_t launch_eval(const EvalArgs &a, const EvalLaunch &L, cudaStream_t s) {
  switch (L.shape) {
    case kK3Cluster: {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(L.grid_x, a.n_models);
      cfg.blockDim = dim3(L.block);
      cfg.dynamicSmemBytes = L.smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = L.grid_x;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      return a.results ? cudaLaunchKernelEx(&cfg, k3_cluster<true>, a) : cudaLaunchKernelEx(&cfg, k3_cluster<false>, a);
    }
    case kK3Factored:
      return launch_pdl(k3_factored, dim3(L.grid_x, a.n_models), dim3(L.block), L.smem, s, a);
    default:
      return launch_pdl(k3_grid<false>, dim3(L.grid_x, a.n_models), dim3(L.block), L.smem, s, a);
  }
}

cudaError_t launch_eval3(const EvalArgs &a, int grid_x, int block, size_t smem, cudaStream_t s) {
  k3_grid<true><<<dim3(grid_x, a.n_models), block, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_eval_peak(const EvalArgs &a, int grid_x, int block, cudaStream_t s) {
  return launch_pdl(k3_peak, dim3(grid_x, a.n_models), dim3(block), eval_peak_smem_bytes(a), s, a);
}

// the largest cluster the device can co-schedule for k3_cluster with this
// shared memory and block size (<= 8, portable)
int eval_max_cluster(int block, size_t smem) {
  for (int c = 8; c >= 1; c >>= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c, 1);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k3_cluster<false>, &cfg) == cudaSuccess && n > 0) return c;
    cudaGetLastError();
  }
  return 1;
}

}  // namespace fp
