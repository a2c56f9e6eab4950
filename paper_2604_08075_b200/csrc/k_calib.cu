// NEXT-3: calibration replay on the GPU -- Alg. 1 OnResponse with
// Eq. `ema` over a feedback stream in arrival order:
//   c_obs = |r| / usage.prompt_tokens
//   c_k   <- beta c_k + (1 - beta) c_obs
//   s_k   <- beta s_k + (1 - beta) |c_obs - c_k(before)|          (R26)
// Both recurrences are affine in their state, x -> a x + b, and affine maps
// compose associatively: (a2, b2) o (a1, b1) = (a2 a1, a2 b1 + b2); n
// observations of one category compose to a = beta^n. The stream is cut into
// one contiguous segment per thread, 256 consecutive segments per block:
//   C1  each thread composes, per category, the c_hat maps of its segment; a
//       block scan turns them into within-block exclusive prefixes and one
//       block total
//   C2  one block per category scans the block totals (exclusive prefixes;
//       the grand total applied to c_0 is the final c_hat)
//   C3  each thread replays its segment from its start state (block prefix,
//       then within-block prefix, applied to c_0) -- exactly the sequential
//       update -- which yields every c_hat(before) and so the sigma maps; at
//       the snap_at-th observation of a category it records c_hat and the
//       sigma map composed so far; block scan of the sigma maps as in C1
//   C2  again for the sigma block totals; C4 applies the snapshot's sigma map
//       (from its block's start) to the sigma state at that block's start
// Category state lives in registers (select chains) for n_cats <= 4 and in
// shared memory [k][thread] above that.
// Segments are contiguous per thread, but the columns are read coalesced: in
// each round a block stages the next 16 records of all 256 of its segments
// into shared memory (64-B pieces, 16-B loads, a warp covering 8 segments),
// swizzled so that each thread then reads its own 16 records with
// conflict-free 16-B shared loads; the global loads of round r+1 are issued
// before round r is consumed. Records past a segment's end are staged with
// prompt_tokens = 0, which the update skips.
// The composition reassociates the fp64 sums, so results agree with the
// sequential oracle to rounding (tests: <= 1e-12 relative), not bit for bit.
#include <algorithm>
#include <cmath>
#include "internal.cuh"

namespace fp {

namespace {

constexpr int kCalBlock = 256;
constexpr int kRound = 8;                  // records per segment per round

__device__ __forceinline__ uint64_t umin(uint64_t x, uint64_t y) { return x < y ? x : y; }

// ---- affine maps and their block scan ------------------------------------------
struct Aff {
  double a, b;
  unsigned long long n;
};

__device__ __forceinline__ Aff aff_id() { return Aff{1.0, 0.0, 0ull}; }

// e first, then l
__device__ __forceinline__ Aff compose(const Aff &e, const Aff &l) {
  return Aff{__dmul_rn(l.a, e.a), __fma_rn(l.a, e.b, l.b), e.n + l.n};
}

__device__ __forceinline__ Aff shfl_up(const Aff &x, int o) {
  return Aff{__shfl_up_sync(0xffffffffu, x.a, o), __shfl_up_sync(0xffffffffu, x.b, o),
             __shfl_up_sync(0xffffffffu, x.n, o)};
}

__device__ __forceinline__ Aff warp_inclusive(Aff inc, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Aff y = shfl_up(inc, o);
    if (lane >= o) inc = compose(y, inc);
  }
  return inc;
}

// exclusive prefix of x over the block's threads in order, and the block total;
// sw: shared scratch of 32 maps. Every thread of the block must call it.
__device__ __forceinline__ void block_scan(const Aff &x, Aff &excl, Aff &total, Aff *sw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const Aff inc = warp_inclusive(x, lane);
  if (lane == 31) sw[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    Aff w = lane < nw ? sw[lane] : aff_id();
    w = warp_inclusive(w, lane);
    if (lane < nw) sw[lane] = w;
  }
  __syncthreads();
  Aff ex = shfl_up(inc, 1);
  if (lane == 0) ex = aff_id();
  excl = warp ? compose(sw[warp - 1], ex) : ex;
  total = sw[nw - 1];
  __syncthreads();
}

__device__ __forceinline__ double apply(const Aff &m, double x) { return __fma_rn(m.a, x, m.b); }

// ---- per-category state: registers (NC <= 4) or shared memory ----------------
template <int NC, bool REG>
struct Vec;

template <int NC>
struct Vec<NC, true> {
  double v[NC];
  __device__ __forceinline__ void bind(double *) {}
  __device__ __forceinline__ double get(uint32_t k) const {
    double r = v[0];
#pragma unroll
    for (int j = 1; j < NC; ++j) r = k == (uint32_t)j ? v[j] : r;
    return r;
  }
  __device__ __forceinline__ void set(uint32_t k, double x) {
#pragma unroll
    for (int j = 0; j < NC; ++j) v[j] = k == (uint32_t)j ? x : v[j];
  }
  // v[k] = beta v[k] + x as NC predicated DFMAs (no select chains: a double
  // select is two FSELs per category, more issue slots than the DFMAs)
  __device__ __forceinline__ void ema(uint32_t k, double beta, double x) {
#pragma unroll
    for (int j = 0; j < NC; ++j)
      asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\t@p fma.rn.f64 %0, %3, %0, %4;\n\t}"
          : "+d"(v[j]) : "r"(k), "r"((uint32_t)j), "d"(beta), "d"(x));
  }
};

template <int NC>
struct Vec<NC, false> {
  double *p;
  __device__ __forceinline__ void bind(double *q) { p = q; }
  __device__ __forceinline__ double get(uint32_t k) const { return p[k * kCalBlock + threadIdx.x]; }
  __device__ __forceinline__ void set(uint32_t k, double x) { p[k * kCalBlock + threadIdx.x] = x; }
  __device__ __forceinline__ void ema(uint32_t k, double beta, double x) { set(k, __fma_rn(beta, get(k), x)); }
};

template <int NC, bool REG>
struct UVec;

// NC <= 4 counters of < 2^16 (seg <= 65,520) packed in one u64: one shift-add per update
template <int NC>
struct UVec<NC, true> {
  static_assert(NC <= 4, "packed counters hold 4 categories");
  unsigned long long v;
  __device__ __forceinline__ void bind(uint32_t *) { v = 0ull; }
  __device__ __forceinline__ uint32_t get(uint32_t k) const { return (uint32_t)(v >> (16 * k)) & 0xffffu; }
  __device__ __forceinline__ void inc(uint32_t k) { v += 1ull << (16 * k); }
  __device__ __forceinline__ void set(uint32_t k, uint32_t x) {
    v = (v & ~(0xffffull << (16 * k))) | ((unsigned long long)(x & 0xffffu) << (16 * k));
  }
  // field k equal in both
  __device__ __forceinline__ bool eq(uint32_t k, const UVec &o) const { return !(((v ^ o.v) >> (16 * k)) & 0xffffu); }
};

template <int NC>
struct UVec<NC, false> {
  uint32_t *p;
  __device__ __forceinline__ void bind(uint32_t *q) { p = q; }
  __device__ __forceinline__ uint32_t get(uint32_t k) const { return p[k * kCalBlock + threadIdx.x]; }
  __device__ __forceinline__ void inc(uint32_t k) { p[k * kCalBlock + threadIdx.x] += 1u; }
  __device__ __forceinline__ void set(uint32_t k, uint32_t x) { p[k * kCalBlock + threadIdx.x] = x; }
  __device__ __forceinline__ bool eq(uint32_t k, const UVec &o) const { return get(k) == o.get(k); }
};

// ---- coalesced staging of per-thread segments ---------------------------------
// Rounds of kRound = 8 records per segment, 256 segments per block, double-
// buffered: while round r is consumed, round r + 1 is copied global -> shared
// by cp.async (no registers held, unlike a register prefetch, which kept the
// kernels at 80 registers and 3 blocks per SM). bytes / tokens [segment][8]
// u32 with the two 16-B groups swizzled by (segment >> 2) & 1 (each thread
// then reads its own records conflict-free), categories [segment][8] u8.
struct StageSmem {
  uint32_t *b, *t, *c;
};

constexpr size_t kStageBytes = (size_t)kCalBlock * kRound * 4 * 2 + (size_t)kCalBlock * kRound;
constexpr size_t kScanBytes = 32 * sizeof(Aff);
constexpr int kParts = kRound / 4;           // 16-B groups per segment per round
static_assert(kRound == 8, "the swizzle below is for two 16-B groups");

__device__ __forceinline__ uint32_t swz(uint32_t seg, uint32_t group) {
  return seg * kRound + ((group ^ ((seg >> 2) & 1u)) << 2);
}

__device__ __forceinline__ StageSmem stage_at(unsigned char *smem, uint32_t i) {
  StageSmem st;
  st.b = reinterpret_cast<uint32_t *>(smem + i * kStageBytes);
  st.t = st.b + kCalBlock * kRound;
  st.c = st.t + kCalBlock * kRound;
  return st;
}

__device__ __forceinline__ void cp_async(void *dst, const void *src, int bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

// full blocks (every segment complete, 16-B aligned columns): round r by
// cp.async; each warp stages its own 32 segments, so a round needs only
// __syncwarp, not a block barrier
__device__ __forceinline__ void issue_round(const CalibArgs &a, uint64_t t0, uint64_t r, const StageSmem &st) {
#pragma unroll
  for (int i = 0; i < kParts; ++i) {
    const uint32_t q = (threadIdx.x & 31u) + 32u * i, seg = (threadIdx.x & ~31u) + q / kParts, part = q % kParts;
    const uint64_t g = (t0 + seg) * a.seg + r * kRound + part * 4;
    cp_async(st.b + swz(seg, part), a.bytes + g, 16);
    cp_async(st.t + swz(seg, part), a.tokens + g, 16);
  }
  cp_async(st.c + threadIdx.x * (kRound / 4), a.cat + (t0 + threadIdx.x) * a.seg + r * kRound, 8);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ uint32_t load1(const uint32_t *p, uint64_t g, uint64_t end) {
  return g < end ? p[g] : 0u;
}

// partial blocks: round r synchronously, element by element (records past a
// segment's end are staged with prompt_tokens = 0, which the update skips)
__device__ __forceinline__ void stage_sync(const CalibArgs &a, uint64_t t0, uint64_t r, const StageSmem &st) {
#pragma unroll
  for (int i = 0; i < kParts; ++i) {
    const uint32_t q = threadIdx.x + kCalBlock * i, seg = q / kParts, part = q % kParts;
    const uint64_t base = (t0 + seg) * a.seg, end = umin(a.n, base + a.seg);
    const uint64_t g = base + r * kRound + part * 4;
    uint4 vb, vt;
    vb.x = load1(a.bytes, g, end); vb.y = load1(a.bytes, g + 1, end);
    vb.z = load1(a.bytes, g + 2, end); vb.w = load1(a.bytes, g + 3, end);
    vt.x = load1(a.tokens, g, end); vt.y = load1(a.tokens, g + 1, end);
    vt.z = load1(a.tokens, g + 2, end); vt.w = load1(a.tokens, g + 3, end);
    *reinterpret_cast<uint4 *>(st.b + swz(seg, part)) = vb;
    *reinterpret_cast<uint4 *>(st.t + swz(seg, part)) = vt;
  }
  const uint64_t base = (t0 + threadIdx.x) * a.seg, end = umin(a.n, base + a.seg);
  const uint64_t g = base + r * kRound;
  uint32_t w0 = 0u, w1 = 0u;
#pragma unroll
  for (int j = 0; j < kRound; ++j) {
    const uint32_t v = g + j < end ? (uint32_t)a.cat[g + j] << (8 * (j & 3)) : 0u;
    if (j < 4) w0 |= v; else w1 |= v;
  }
  *reinterpret_cast<uint2 *>(st.c + threadIdx.x * (kRound / 4)) = make_uint2(w0, w1);
}

__device__ __forceinline__ uint32_t get(const uint4 &v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

// exact u32 -> f64 on the FP64 pipe (2^52 + x is exact), instead of the
// conversion unit that the reciprocal seed also needs
__device__ __forceinline__ double u2d(uint32_t x) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)x), 4503599627370496.0);
}

// c_obs = |r| / tokens without the IEEE division's slow-path branch: the
// hardware f64 reciprocal estimate refined by two Newton steps (relative
// error <= 2^-20 -> 2^-40 -> below fp64 rounding), then one multiply: within
// 2 ulp of the correctly rounded quotient, which the replay's reassociated
// sums absorb (1e-12).
__device__ __forceinline__ double ratio(uint32_t num, uint32_t den) {
  const double d = u2d(den);
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = __fma_rn(y, __fma_rn(-d, y, 1.0), y);
  y = __fma_rn(y, __fma_rn(-d, y, 1.0), y);
  return __dmul_rn(u2d(num), y);
}

// PRED: body(c_obs, k) for every staged record, k = n_cats for dropped feedback
// (the bodies below then update a scratch slot: no branch, no select of
// the whole update); otherwise body is called for valid records only.
template <bool PRED, typename Body>
__device__ __forceinline__ void consume(const StageSmem &st, uint32_t last, Body &body) {
  const uint2 cc = *reinterpret_cast<const uint2 *>(st.c + threadIdx.x * (kRound / 4));
#pragma unroll
  for (int gi = 0; gi < kParts; ++gi) {
    const uint4 vb = *reinterpret_cast<const uint4 *>(st.b + swz(threadIdx.x, gi));
    const uint4 vt = *reinterpret_cast<const uint4 *>(st.t + swz(threadIdx.x, gi));
    const uint32_t cw = gi == 0 ? cc.x : cc.y;
    double o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = ratio(get(vb, e), get(vt, e) | (get(vt, e) == 0u));
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t cat = (cw >> (8 * e)) & 0xffu;
      if (PRED) body(o[e], get(vt, e) != 0u ? (cat < last ? cat : last) : last + 1u);
      else if (get(vt, e) != 0u) body(o[e], cat < last ? cat : last);   // S:240 drop; R23
    }
  }
}

// Runs body(c_obs, category) over this thread's segment in order (valid records only).
// Stage buffers 0 and 1 at smem + {0, kStageBytes}.
template <bool PRED = false, typename Body>
__device__ __forceinline__ void for_segment(const CalibArgs &a, unsigned char *smem, Body body) {
  const uint64_t t0 = (uint64_t)blockIdx.x * kCalBlock;
  const uint64_t rounds = (a.seg + kRound - 1) / kRound;
  const uint32_t last = a.n_cats - 1;
  const bool full = a.vec_bt && a.vec_c && (t0 + kCalBlock) * a.seg <= a.n;
  if (full) {
    issue_round(a, t0, 0, stage_at(smem, 0));
    for (uint64_t r = 0; r < rounds; ++r) {
      if (r + 1 < rounds) issue_round(a, t0, r + 1, stage_at(smem, (uint32_t)(r + 1) & 1u));
      else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
      consume<PRED>(stage_at(smem, (uint32_t)r & 1u), last, body);
      __syncwarp();                    // buffer r & 1 is refilled at round r + 2
    }
  } else {
    const StageSmem st = stage_at(smem, 0);
    for (uint64_t r = 0; r < rounds; ++r) {
      __syncthreads();                 // previous round consumed
      stage_sync(a, t0, r, st);
      __syncthreads();
      consume<PRED>(st, last, body);
    }
  }
}

// beta^n by squaring (the maps' multiplicative part: one factor per observation)
__device__ __forceinline__ double pow_n(double beta, uint32_t n) {
  double r = 1.0, b = beta;
  while (n) {
    if (n & 1u) r = __dmul_rn(r, b);
    b = __dmul_rn(b, b);
    n >>= 1;
  }
  return r;
}

// ---- NC <= 4 fast paths: scaled recurrences ---------------------------------------
// The recurrences run on state scaled by 1 / w (w = 1 - beta), one FMA per update:
//   C1  b~ <- beta b~ + c_obs                   (the map's offset = w b~)
//   C3  c~ <- beta c~ + c_obs                   (c_hat = w c~)
//       s~ <- beta s~ + |c_obs - c_hat(before)|,  c_obs - c_hat = fma(-w, c~, c_obs)   (R26)
// -- the oracle's sums with each term rounded once more by the final scaling,
// within the replay's reassociation tolerance (1e-12 relative). Category state
// is indexed where a register select chain would cost more issue slots:
// ptxas turns a predicated DFMA into an unconditional DFMA + two FSELs per
// category, so C1's b~ lives in shared memory rows [k][thread] (one LDS.64 +
// STS.64 per record, no select) with the counters packed in one u64; C3 keeps
// c~ in registers (read and written through select chains) and s~ in shared
// memory. (Both states in shared memory -- 64- or 128-bit rows -- measured
// slower: the MIO queue saturates, profiles/r02/r02_next3_variants.md.)

struct Smem {
  Aff *scan;
  double *d0, *d1;      // [NC][kCalBlock]: d0 shared-memory state only, d1 always (sigma maps)
  uint32_t *u0, *u1;
};

__device__ __forceinline__ Smem smem_layout(unsigned char *smem, uint32_t nc, bool reg) {
  Smem s;
  s.scan = reinterpret_cast<Aff *>(smem + 2 * kStageBytes);
  s.d0 = reinterpret_cast<double *>(smem + 2 * kStageBytes + kScanBytes);
  s.d1 = s.d0 + (reg ? 0 : nc * kCalBlock);
  s.u0 = reinterpret_cast<uint32_t *>(s.d1 + nc * kCalBlock);
  s.u1 = s.u0 + (reg ? 0 : nc * kCalBlock);
  return s;
}

// C1: per-thread c_hat maps -> within-block exclusive prefixes + block totals
template <int NC, bool REG>
__global__ void __launch_bounds__(kCalBlock, 4) c1_maps(CalibArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem sm = smem_layout(smem, NC, REG);
  Vec<NC, REG> b;
  UVec<NC, REG> n;
  b.bind(sm.d0);
  n.bind(sm.u0);
  for (uint32_t k = 0; k < NC; ++k) { b.set(k, 0.0); n.set(k, 0u); }
  const double beta = a.beta, w = __dsub_rn(1.0, a.beta);
  if constexpr (REG) {
    // scaled b~ indexed in shared memory (d1 rows [k][thread]; row n_cats
    // takes dropped feedback): one LDS.64 + STS.64 per record instead of NC
    // DFMAs and 2 NC FSELs; the NC 16-bit counters packed in one u64
    // (shl.b64 by 16 k >= 64 adds nothing: dropped feedback)
    double *bk = sm.d1 + threadIdx.x;
    for (uint32_t j = 0; j <= a.n_cats; ++j) bk[j * kCalBlock] = 0.0;
    unsigned long long cnt = 0ull;
    for_segment<true>(a, smem, [&](double c, uint32_t k) {
      double *p = bk + k * kCalBlock;
      *p = __fma_rn(beta, *p, c);
      unsigned long long inc;
      asm("shl.b64 %0, %1, %2;" : "=l"(inc) : "l"(1ull), "r"(16u * k));
      cnt += inc;
    });
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      b.set(j, j < (int)a.n_cats ? __dmul_rn(w, bk[j * kCalBlock]) : 0.0);
      n.set(j, (uint32_t)(cnt >> (16 * j)) & 0xffffu);
    }
  } else {
    for_segment(a, smem, [&](double c, uint32_t k) {
      b.ema(k, beta, __dmul_rn(w, c));
      n.inc(k);
    });
  }
  const uint64_t t = (uint64_t)blockIdx.x * kCalBlock + threadIdx.x;
  for (uint32_t k = 0; k < a.n_cats; ++k) {
    const uint32_t nk = n.get(k);
    Aff ex, tot;
    block_scan(Aff{pow_n(beta, nk), b.get(k), nk}, ex, tot, sm.scan);
    a.thrA[k * a.threads + t] = ex.a;
    a.thrB[k * a.threads + t] = ex.b;
    a.thrN[k * a.threads + t] = (uint32_t)ex.n;
    a.thrC[k * a.threads + t] = nk;
    if (threadIdx.x == 0) {
      a.blkA[k * a.blocks + blockIdx.x] = tot.a;
      a.blkB[k * a.blocks + blockIdx.x] = tot.b;
      a.blkN[k * a.blocks + blockIdx.x] = tot.n;
    }
  }
}

// C2: exclusive scan of the block totals of one category (block = category);
// which = 0: c_hat maps (final c_hat, counts), 1: sigma maps (final sigma)
__global__ void __launch_bounds__(1024) c2_scan(CalibArgs a, int which) {
  __shared__ Aff sw[32];
  const uint32_t k = blockIdx.x;
  double *A = (which ? a.sblkA : a.blkA) + (uint64_t)k * a.blocks;
  double *B = (which ? a.sblkB : a.blkB) + (uint64_t)k * a.blocks;
  unsigned long long *N = a.blkN + (uint64_t)k * a.blocks;
  Aff carry = aff_id();
  for (uint64_t base = 0; base < a.blocks; base += blockDim.x) {
    const uint64_t j = base + threadIdx.x;
    const bool in = j < a.blocks;
    const Aff x = in ? Aff{A[j], B[j], which ? 0ull : N[j]} : aff_id();
    Aff ex, tot;
    block_scan(x, ex, tot, sw);
    const Aff pre = compose(carry, ex);
    if (in) {
      A[j] = pre.a;
      B[j] = pre.b;
      if (!which) N[j] = pre.n;
    }
    carry = compose(carry, tot);
  }
  if (threadIdx.x == 0) {
    if (which == 0) {
      a.totA[k] = apply(carry, a.c0[k]);
      a.totN[k] = carry.n;
      a.mapA[k] = carry.a; a.mapB[k] = carry.b; a.mapN[k] = carry.n;
    } else {
      a.totSA[k] = apply(carry, a.s0[k]);
      a.smapA[k] = carry.a; a.smapB[k] = carry.b;
    }
  }
}

// C3: replay each segment from its c_hat start state; sigma maps; snapshots
template <int NC, bool REG>
__global__ void __launch_bounds__(kCalBlock, 4) c3_replay(CalibArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem sm = smem_layout(smem, NC, REG);
  Vec<NC, REG> c;
  Vec<NC, false> sb;              // shared memory: frees the select chains for c
  UVec<NC, REG> n, target;
  c.bind(sm.d0);
  sb.bind(sm.d1);
  n.bind(sm.u0);
  target.bind(sm.u1);
  const uint64_t t = (uint64_t)blockIdx.x * kCalBlock + threadIdx.x;
  for (uint32_t k = 0; k < NC; ++k) {
    double ck = 0.0;
    uint32_t tk = 0u;
    if (k < a.n_cats) {
      const Aff blk{a.blkA[k * a.blocks + blockIdx.x], a.blkB[k * a.blocks + blockIdx.x],
                    a.blkN[k * a.blocks + blockIdx.x]};
      const Aff thr{a.thrA[k * a.threads + t], a.thrB[k * a.threads + t], a.thrN[k * a.threads + t]};
      const Aff pre = compose(blk, thr);
      ck = apply(pre, a.c0[k]);
      // observations of category k before this segment; the snapshot fires at seen == target
      const unsigned long long before = pre.n + a.snap_off[k];
      tk = (a.snap_at > before && a.snap_at - before <= a.seg) ? (uint32_t)(a.snap_at - before) : 0u;
    }
    c.set(k, ck);
    sb.set(k, 0.0);
    n.set(k, 0u);
    target.set(k, tk);
  }
  const double beta = a.beta, w = __dsub_rn(1.0, a.beta);
  uint32_t snapped = 0u;          // bit k: this thread holds category k's snapshot
  // Only the blocks holding a snapshot count observations per record; the
  // others take each segment's counts from C1 (thrC) and skip the counters
  bool mine = false;
  for (uint32_t k = 0; k < a.n_cats; ++k) mine |= target.get(k) != 0u;
  if (__syncthreads_or(mine)) {
    for_segment(a, smem, [&](double o, uint32_t k) {
      const double prev = c.get(k);
      const double cn = __fma_rn(beta, prev, __dmul_rn(w, o));
      c.set(k, cn);
      const double sn = __fma_rn(beta, sb.get(k), __dmul_rn(w, fabs(__dsub_rn(o, prev))));
      sb.set(k, sn);
      n.inc(k);
      if (n.eq(k, target)) {
        a.snap_c[k] = cn;
        a.snap_sa[k] = pow_n(beta, target.get(k));
        a.snap_sb[k] = sn;
        snapped |= 1u << k;
      }
    });
  } else {
    if constexpr (REG) {
      // scaled c~ in registers (select chains), scaled s~ in shared memory
      // (row n_cats <= NC takes dropped feedback)
      sb.set(a.n_cats, 0.0);
      const double neg_w = -w;
      Vec<NC, true> cs;
#pragma unroll
      for (int j = 0; j < NC; ++j) cs.v[j] = __ddiv_rn(c.get(j), w);
      for_segment<true>(a, smem, [&](double o, uint32_t k) {
        const double prev = cs.get(k);
        const double d = __fma_rn(neg_w, prev, o);
        cs.set(k, __fma_rn(beta, prev, o));
        sb.set(k, __fma_rn(beta, sb.get(k), fabs(d)));
      });
      for (uint32_t k = 0; k < a.n_cats; ++k) sb.set(k, __dmul_rn(w, sb.get(k)));
    } else {
      for_segment(a, smem, [&](double o, uint32_t k) {
        const double prev = c.get(k);
        c.set(k, __fma_rn(beta, prev, __dmul_rn(w, o)));
        sb.set(k, __fma_rn(beta, sb.get(k), __dmul_rn(w, fabs(__dsub_rn(o, prev)))));
      });
    }
    for (uint32_t k = 0; k < a.n_cats; ++k) n.set(k, a.thrC[k * a.threads + t]);
  }
  for (uint32_t k = 0; k < a.n_cats; ++k) {
    const uint32_t nk = n.get(k);
    Aff ex, tot;
    block_scan(Aff{pow_n(beta, nk), sb.get(k), nk}, ex, tot, sm.scan);
    if (threadIdx.x == 0) {
      a.sblkA[k * a.blocks + blockIdx.x] = tot.a;
      a.sblkB[k * a.blocks + blockIdx.x] = tot.b;
    }
    if (snapped & (1u << k)) {      // snapshot map from the block's start
      const Aff part{a.snap_sa[k], a.snap_sb[k], 0ull};
      const Aff m = compose(ex, part);
      a.snap_sa[k] = m.a;
      a.snap_sb[k] = m.b;
      a.snap_block[k] = blockIdx.x;
    }
  }
}

// C4: sigma snapshot = (map from its block's start) applied to sigma at that start
__global__ void c4_snap(CalibArgs a) {
  const uint32_t k = threadIdx.x;
  if (k >= a.n_cats || a.snap_block[k] == ~0ull) return;
  const uint64_t j = a.snap_block[k];
  const double s_start = __fma_rn(a.sblkA[k * a.blocks + j], a.s0[k], a.sblkB[k * a.blocks + j]);
  a.snap_s[k] = __fma_rn(a.snap_sa[k], s_start, a.snap_sb[k]);
}


// ============================================================================
// One rank, n_cats <= 4: the streaming replay (c_stream) -- every record is
// read from HBM once and its c_obs computed once.
//
// A persistent grid of G co-resident CTAs (cooperative launch) walks the
// stream in chunks of G pieces of 3,584 records; CTA c owns piece c of every
// chunk. Iteration i of a CTA runs phase A on chunk i, then phase C on chunk
// i - 2, whose piece is still in the CTA's shared memory (a ring of three):
// the lag of two leaves a whole iteration for chunk i - 2's scan to land.
//   A  each warp loads a region of 448 records (coalesced 128-B column loads),
//      ranks every valid record inside its category with three ballots
//      (valid, category bit 0, bit 1), and stores c_obs in category order --
//      each category's run starting on a 16-slot boundary, so lane l's 16
//      slots hold one category only. Each lane composes the c_hat maps of its
//      slots (Horner, one FMA per observation: no per-record category
//      dispatch); a segmented warp scan (lanes of one category are adjacent)
//      gives every lane its exclusive map in the region and the region
//      aggregates; 4 threads compose the 8 regions into the piece aggregate.
//      The CTA that finishes chunk i last (atomic count) scans the chunk's G
//      piece aggregates, takes the chunk's start state from chunk i - 1's
//      scanner (flag), and publishes every piece's start state and the next
//      chunk's (flag) -- the only cross-CTA step on the path, once per chunk.
//   C  waits for its chunk's flag, then every lane replays its slots from the
//      exact start state (piece start, region map, lane map): c_hat(before)
//      for each observation and so the sigma maps (R26), the snap_at-th
//      observation's state; a segmented warp scan and 4 threads compose the
//      piece's sigma map (global, [piece][k]).
// c_stream_final composes the sigma piece maps in stream order and writes the
// final state and the snapshots.
// Reassociation: within 1e-12 of the sequential oracle like the kernels above.
// Opt-in (FP_CALIB_STREAM=1): it reads exactly 9 B/record from HBM (ncu), but
// each iteration is a chain of latencies -- the column loads (~2 us), the
// fence and chunk counter, the scanner's hand-off -- that two CTAs per SM
// (the shared-memory ring of three pieces allows no more) cannot hide: A 6.0,
// C 2.2, waiting 10.7 us per iteration, 17.5 ms per 1e9 records against the
// two-pass kernels' 4.7 ms (FP_CALIB_PROFILE=1 prints the phase stamps;
// profiles/r02/next3_stream_profile.log).
// ============================================================================
constexpr int kSW = 8;                         // warps per CTA
constexpr int kSThreads = kSW * 32;
constexpr int kSWords = 14;                    // 32-record words per warp region
constexpr int kSRegion = kSWords * 32;         // 448 records
constexpr int kSSlots = 512;                   // sorted slots per region: 16 per lane (<= 448 + 4 x 15 used)
constexpr int kSLag = 2;                       // iteration i: phase A of chunk i, phase C of chunk i - kSLag
constexpr int kSRing = kSLag + 1;              // pieces held in shared memory
constexpr int kSBeta = kSRegion + 1;           // beta^j, 0 <= j <= 448 (compositions inside a region)
constexpr uint32_t kIdle = 7u;                 // lane category of an empty lane
constexpr uint32_t kFinBlocks = 148;           // c_stream_final blocks per category (<= 256)

struct SLayout {
  static constexpr size_t sorted = 0;                                             // double [ring][w][512]
  static constexpr size_t lane_b = sorted + (size_t)kSRing * kSW * kSSlots * 8;   // double [ring][w][32]
  static constexpr size_t lane_m = lane_b + (size_t)kSRing * kSW * 32 * 8;        // u32 [ring][w][32]
  static constexpr size_t rex = lane_m + (size_t)kSRing * kSW * 32 * 4;           // Aff [ring][w][4]
  static constexpr size_t bpow = rex + (size_t)kSRing * kSW * 4 * sizeof(Aff);    // double [513]
  static constexpr size_t bytes = bpow + (size_t)kSBeta * 8;
};

__device__ __forceinline__ Aff ld_aff(const Aff *p) {
  return Aff{__ldcg(&p->a), __ldcg(&p->b), __ldcg(&p->n)};
}
__device__ __forceinline__ void st_release(unsigned int *p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const unsigned int *p) {
  unsigned int f;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(p) : "memory");
    if (f) return;
    __nanosleep(32);
  }
}

// physical slot of sorted slot s: lane chunk l = s / 16 owns 8 16-B units,
// swizzled by l & 7 so that lanes reading their own unit u hit distinct banks
__device__ __forceinline__ uint32_t sslot(uint32_t s) {
  const uint32_t l = s >> 4;
  return (l << 4) | ((((s & 15u) >> 1) ^ (l & 7u)) << 1) | (s & 1u);
}
__device__ __forceinline__ uint32_t r16(uint32_t x) { return (x + 15u) & ~15u; }
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// FP_CALIB_PROFILE: phase stamps -- [chunk][0..3] scanner, [n_chunks + i][0..7] CTA 0's iteration i
#define CS_STAMP(row, col)                                                   \
  do {                                                                       \
    if (a.prof && threadIdx.x == 0) a.prof[(uint64_t)(row) * 8 + (col)] = gtime(); \
  } while (0)

// compose within a region: a from the beta^n table (n <= 512)
__device__ __forceinline__ Aff compose_t(const Aff &e, const Aff &l, const double *bpow) {
  const unsigned long long n = e.n + l.n;
  return Aff{bpow[n], __fma_rn(l.a, e.b, l.b), n};
}

// lanes sorted by category (kIdle last): inclusive segmented scan of the lane maps
__device__ __forceinline__ Aff seg_scan(Aff x, uint32_t kl, uint32_t lane, const double *bpow) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Aff y = shfl_up(x, o);
    const uint32_t yk = __shfl_up_sync(0xffffffffu, kl, o);
    if (lane >= (uint32_t)o && yk == kl) x = compose_t(y, x, bpow);
  }
  return x;
}

// the lane's own category run: [start, start + 16) of category kl with cnt observations
__device__ __forceinline__ void lane_run(uint32_t lane, const uint32_t st[5], const uint32_t cnt4[4], uint32_t &kl,
                                         uint32_t &cnt) {
  const uint32_t ls = lane * 16u;
  kl = kIdle;
  cnt = 0u;
#pragma unroll
  for (uint32_t k = 0; k < 4; ++k)
    if (ls >= st[k] && ls < st[k + 1]) { kl = k; cnt = min(16u, cnt4[k] - (ls - st[k])); }
}

__device__ __forceinline__ void phase_a(const CalibStreamArgs &a, unsigned char *smem, uint32_t i, int &scanner) {
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5, ring = i % kSRing, c = blockIdx.x;
  const double *bpow = reinterpret_cast<const double *>(smem + SLayout::bpow);
  double *srt = reinterpret_cast<double *>(smem + SLayout::sorted) + (ring * kSW + w) * kSSlots;
  Aff *rex = reinterpret_cast<Aff *>(smem + SLayout::rex) + ring * kSW * 4;
  const double beta = a.beta, wgt = __dsub_rn(1.0, a.beta);
  const uint64_t rb = ((uint64_t)i * a.G + c) * (uint64_t)(kSW * kSRegion) + (uint64_t)w * kSRegion;
  const uint32_t last = a.n_cats - 1u;
  uint32_t vb[kSWords], vt[kSWords], info[kSWords];
#pragma unroll
  for (int j = 0; j < kSWords; ++j) {
    const uint64_t r = rb + 32u * j + lane;
    const bool in = r < a.n;
    vb[j] = in ? __ldcs(a.bytes + r) : 0u;
    vt[j] = in ? __ldcs(a.tokens + r) : 0u;
    info[j] = in ? (uint32_t)__ldcs(a.cat + r) : 0u;
  }
  // rank of each valid record inside its category (stream order): three ballots per word
  uint32_t run[4] = {0u, 0u, 0u, 0u};
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kSWords; ++j) {
    const bool valid = vt[j] != 0u;                              // zero-token feedback is dropped
    const uint32_t k = info[j] < last ? info[j] : last;          // R23
    const uint32_t v = __ballot_sync(0xffffffffu, valid);
    const uint32_t b0 = __ballot_sync(0xffffffffu, valid && (k & 1u));
    const uint32_t b1 = __ballot_sync(0xffffffffu, valid && (k & 2u));
    const uint32_t m0 = v & ~(b0 | b1), m1 = b0 & ~b1, m2 = b1 & ~b0, m3 = b0 & b1;
    const uint32_t mine = (k & 2u) ? ((k & 1u) ? m3 : m2) : ((k & 1u) ? m1 : m0);
    const uint32_t base = (k & 2u) ? ((k & 1u) ? run[3] : run[2]) : ((k & 1u) ? run[1] : run[0]);
    info[j] = valid ? ((base + __popc(mine & lt)) | (k << 10) | 0x1000u) : 0u;
    run[0] += __popc(m0); run[1] += __popc(m1); run[2] += __popc(m2); run[3] += __popc(m3);
  }
  uint32_t st[5];
  st[0] = 0u;
#pragma unroll
  for (int k = 0; k < 4; ++k) st[k + 1] = st[k] + r16(run[k]);
#pragma unroll
  for (int j = 0; j < kSWords; ++j) {
    const double o = ratio(vb[j], vt[j] | (vt[j] == 0u));
    if (info[j] & 0x1000u) {
      const uint32_t k = (info[j] >> 10) & 3u;
      srt[sslot((info[j] & 0x3ffu) + st[k])] = o;
    }
  }
  __syncwarp();
  uint32_t kl, cnt;
  lane_run(lane, st, run, kl, cnt);
  const double *lc = srt + lane * 16u;
  double bt = 0.0;
  if (cnt == 16u) {
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u) {
      const double2 q = *reinterpret_cast<const double2 *>(lc + ((u ^ (lane & 7u)) << 1));
      bt = __fma_rn(beta, bt, q.x);
      bt = __fma_rn(beta, bt, q.y);
    }
  } else {
    for (uint32_t e = 0; e < cnt; ++e) bt = __fma_rn(beta, bt, lc[(((e >> 1) ^ (lane & 7u)) << 1) | (e & 1u)]);
  }
  const Aff inc = seg_scan(Aff{bpow[cnt], __dmul_rn(wgt, bt), cnt}, kl, lane, bpow);
  Aff ex = shfl_up(inc, 1);
  const uint32_t kprev = __shfl_up_sync(0xffffffffu, kl, 1);
  if (lane == 0u || kprev != kl) ex = aff_id();
  reinterpret_cast<double *>(smem + SLayout::lane_b)[(ring * kSW + w) * 32 + lane] = ex.b;
  reinterpret_cast<uint32_t *>(smem + SLayout::lane_m)[(ring * kSW + w) * 32 + lane] =
      (uint32_t)ex.n | (cnt << 10) | (kl << 16);
  // region aggregates: the last lane of each category run (identity for empty categories)
  const uint32_t knext = __shfl_down_sync(0xffffffffu, kl, 1);
  if (lane < 4u) {
    const uint32_t rl = lane == 0u ? run[0] : lane == 1u ? run[1] : lane == 2u ? run[2] : run[3];
    if (rl == 0u) rex[w * 4 + lane] = aff_id();
  }
  if (kl != kIdle && (lane == 31u || knext != kl)) rex[w * 4 + kl] = inc;
  __syncthreads();
  if (threadIdx.x < 4u) {                          // regions -> exclusive maps in the piece, piece aggregate
    const uint32_t k = threadIdx.x;
    Aff acc = aff_id();
    for (int r = 0; r < kSW; ++r) {
      const Aff g = rex[r * 4 + k];
      rex[r * 4 + k] = acc;
      acc = compose(acc, g);
    }
    static_cast<Aff *>(a.cagg)[((uint64_t)i * a.G + c) * 4 + k] = acc;
    __threadfence();
  }
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(a.done + i, 1u) == a.G - 1u;
  __syncthreads();
  scanner = s_last;
}

// exclusive scan of four maps per thread (one per category) over the block:
// one set of barriers for all four
__device__ __forceinline__ void block_scan4(const Aff (&x)[4], Aff (&ex)[4], Aff (&tot)[4], Aff (*sw)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  Aff inc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) inc[k] = warp_inclusive(x[k], lane);
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < 4; ++k) sw[warp][k] = inc[k];
  }
  __syncthreads();
  if (warp < 4) {                                   // warp k scans category k's warp totals
    Aff v = lane < nw ? sw[lane][warp] : aff_id();
    v = warp_inclusive(v, lane);
    if (lane < nw) sw[lane][warp] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Aff e = shfl_up(inc[k], 1);
    if (lane == 0) e = aff_id();
    ex[k] = warp ? compose(sw[warp - 1][k], e) : e;
    tot[k] = sw[nw - 1][k];
  }
  __syncthreads();
}

// the last CTA of chunk i: piece start states of chunk i, start state of chunk i + 1
__device__ __noinline__ void scan_chunk(const CalibStreamArgs &a, uint32_t i) {
  __shared__ Aff s_red[kSW][4];
  __shared__ double s_c[4];
  __shared__ unsigned long long s_n[4];
  CS_STAMP(i, 0);
  __threadfence();
  const Aff *ag = static_cast<const Aff *>(a.cagg) + (uint64_t)i * a.G * 4;
  const uint32_t p0 = 2u * threadIdx.x, p1 = p0 + 1u;
  Aff x0[4], x1[4], x[4], e0[4], tot[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    x0[k] = p0 < a.G ? ld_aff(ag + p0 * 4 + k) : aff_id();
    x1[k] = p1 < a.G ? ld_aff(ag + p1 * 4 + k) : aff_id();
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = compose(x0[k], x1[k]);
  block_scan4(x, e0, tot, s_red);
  CS_STAMP(i, 1);
  if (threadIdx.x < 4u) {
    const uint32_t k = threadIdx.x;
    if (i) wait_flag(a.ready + i);
    s_c[k] = i ? __ldcg(a.cstart_c + (uint64_t)i * 4 + k) : a.c0[k];
    s_n[k] = i ? __ldcg(a.cstart_n + (uint64_t)i * 4 + k) : 0ull;
  }
  __syncthreads();
  CS_STAMP(i, 2);
  const uint64_t q = (uint64_t)i * a.G;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const Aff e1 = compose(e0[k], x0[k]);
    if (p0 < a.G) { a.pstate_c[(q + p0) * 4 + k] = apply(e0[k], s_c[k]); a.pstate_n[(q + p0) * 4 + k] = s_n[k] + e0[k].n; }
    if (p1 < a.G) { a.pstate_c[(q + p1) * 4 + k] = apply(e1, s_c[k]); a.pstate_n[(q + p1) * 4 + k] = s_n[k] + e1.n; }
  }
  if (threadIdx.x < 4u) {
    const uint32_t k = threadIdx.x;
    const Aff t = k == 0u ? tot[0] : k == 1u ? tot[1] : k == 2u ? tot[2] : tot[3];
    a.cstart_c[(uint64_t)(i + 1) * 4 + k] = apply(t, s_c[k]);
    a.cstart_n[(uint64_t)(i + 1) * 4 + k] = s_n[k] + t.n;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(a.ready + i + 1, 1u);
  CS_STAMP(i, 3);
}

__device__ __forceinline__ void phase_c(const CalibStreamArgs &a, unsigned char *smem, uint32_t i) {
  __shared__ double s_pc[4];
  __shared__ unsigned long long s_pn[4];
  __shared__ Aff s_sreg[kSW][4];                  // region sigma aggregates
  __shared__ Aff s_snap[4];                       // sigma map region start -> snapshot
  __shared__ double s_snapc[4];
  __shared__ int s_snapw[4];
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5, ring = i % kSRing, c = blockIdx.x;
  const double *bpow = reinterpret_cast<const double *>(smem + SLayout::bpow);
  const double *srt = reinterpret_cast<const double *>(smem + SLayout::sorted) + (ring * kSW + w) * kSSlots;
  const Aff *rex = reinterpret_cast<const Aff *>(smem + SLayout::rex) + ring * kSW * 4;
  const double beta = a.beta, wgt = __dsub_rn(1.0, a.beta), inv_w = __drcp_rn(wgt), neg_w = -wgt;
  const uint64_t piece = (uint64_t)i * a.G + c;
  if (a.prof && blockIdx.x == 0) CS_STAMP(a.n_chunks + i + kSLag, 3);
  if (threadIdx.x == 0) wait_flag(a.ready + i + 1);
  if (a.prof && blockIdx.x == 0) CS_STAMP(a.n_chunks + i + kSLag, 4);
  if (lane < 4u) s_sreg[w][lane] = aff_id();
  if (threadIdx.x < 4u) s_snapw[threadIdx.x] = -1;
  __syncthreads();
  if (threadIdx.x < 4u) {
    s_pc[threadIdx.x] = __ldcg(a.pstate_c + piece * 4 + threadIdx.x);
    s_pn[threadIdx.x] = __ldcg(a.pstate_n + piece * 4 + threadIdx.x);
  }
  __syncthreads();
  const uint32_t m = reinterpret_cast<const uint32_t *>(smem + SLayout::lane_m)[(ring * kSW + w) * 32 + lane];
  const double lb = reinterpret_cast<const double *>(smem + SLayout::lane_b)[(ring * kSW + w) * 32 + lane];
  const uint32_t kl = m >> 16, cnt = (m >> 10) & 31u, ne = m & 0x3ffu;
  const uint32_t kk = kl & 3u;
  const Aff rg = rex[w * 4 + kk];
  const double start = apply(Aff{bpow[ne], lb, ne}, apply(rg, s_pc[kk]));   // c_hat at the lane's first slot
  const unsigned long long before = s_pn[kk] + rg.n + ne;                    // observations of kl before it
  const double *lc = srt + lane * 16u;
  double cs = __dmul_rn(start, inv_w), ss = 0.0;                             // scaled state (1 / w)
  if (cnt == 16u) {
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u) {
      const double2 q = *reinterpret_cast<const double2 *>(lc + ((u ^ (lane & 7u)) << 1));
      double d = __fma_rn(neg_w, cs, q.x);
      cs = __fma_rn(beta, cs, q.x);
      ss = __fma_rn(beta, ss, fabs(d));
      d = __fma_rn(neg_w, cs, q.y);
      cs = __fma_rn(beta, cs, q.y);
      ss = __fma_rn(beta, ss, fabs(d));
    }
  } else {
    for (uint32_t e = 0; e < cnt; ++e) {
      const double o = lc[(((e >> 1) ^ (lane & 7u)) << 1) | (e & 1u)];
      const double d = __fma_rn(neg_w, cs, o);
      cs = __fma_rn(beta, cs, o);
      ss = __fma_rn(beta, ss, fabs(d));
    }
  }
  // the snap_at-th observation of category kl in this lane: replay up to it (once per category)
  const bool snap = cnt != 0u && a.snap_at > before && a.snap_at - before <= cnt;
  Aff m1 = aff_id();
  double csnap = 0.0;
  if (snap) {
    const uint32_t t = (uint32_t)(a.snap_at - before);
    double c2 = __dmul_rn(start, inv_w), s2 = 0.0;
    for (uint32_t e = 0; e < t; ++e) {
      const double o = lc[(((e >> 1) ^ (lane & 7u)) << 1) | (e & 1u)];
      const double d = __fma_rn(neg_w, c2, o);
      c2 = __fma_rn(beta, c2, o);
      s2 = __fma_rn(beta, s2, fabs(d));
    }
    csnap = __dmul_rn(wgt, c2);
    m1 = Aff{bpow[t], __dmul_rn(wgt, s2), t};
  }
  const Aff inc = seg_scan(Aff{bpow[cnt], __dmul_rn(wgt, ss), cnt}, kl, lane, bpow);
  Aff ex = shfl_up(inc, 1);
  const uint32_t kprev = __shfl_up_sync(0xffffffffu, kl, 1);
  if (lane == 0u || kprev != kl) ex = aff_id();
  const uint32_t knext = __shfl_down_sync(0xffffffffu, kl, 1);
  if (kl != kIdle && (lane == 31u || knext != kl)) s_sreg[w][kl] = inc;
  if (snap) {
    s_snap[kl] = compose(ex, m1);
    s_snapc[kl] = csnap;
    s_snapw[kl] = (int)w;
  }
  __syncthreads();
  if (threadIdx.x < 4u) {                            // piece sigma map; snapshot map from the piece start
    const uint32_t k = threadIdx.x;
    Aff acc = aff_id();
    for (int r = 0; r < kSW; ++r) {
      if (r == s_snapw[k]) {
        const Aff sm = compose(acc, s_snap[k]);
        a.snap_piece[k] = piece;
        a.snap_v[k * 4 + 0] = sm.a;
        a.snap_v[k * 4 + 1] = sm.b;
        a.snap_v[k * 4 + 2] = s_snapc[k];
      }
      acc = compose(acc, s_sreg[r][k]);
    }
    a.sig_a[piece * 4 + k] = acc.a;
    a.sig_b[piece * 4 + k] = acc.b;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSThreads, 2) c_stream(CalibStreamArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  double *bpow = reinterpret_cast<double *>(smem + SLayout::bpow);
  for (int j = threadIdx.x; j < kSBeta; j += kSThreads) bpow[j] = pow_n(a.beta, (uint32_t)j);
  __syncthreads();
  for (uint32_t i = 0; i < a.n_chunks + kSLag; ++i) {
    const bool p0 = a.prof && blockIdx.x == 0;
    if (p0) CS_STAMP(a.n_chunks + i, 0);
    if (i < a.n_chunks) {
      int scanner = 0;
      phase_a(a, smem, i, scanner);
      if (p0) CS_STAMP(a.n_chunks + i, 1);
      if (scanner) scan_chunk(a, i);
      if (p0) CS_STAMP(a.n_chunks + i, 2);
    }
    if (i >= (uint32_t)kSLag) phase_c(a, smem, i - kSLag);
    if (p0) CS_STAMP(a.n_chunks + i, 5);
  }
}

// sigma piece maps composed in stream order: block (b, k) composes a
// contiguous range of pieces of category k; the last block of category k
// composes the ranges, applies them to s0 and resolves the snapshot
__global__ void __launch_bounds__(256) c_stream_final(CalibStreamArgs a) {
  __shared__ Aff s_red[32];
  __shared__ int s_last;
  const uint32_t k = blockIdx.y, nb = gridDim.x, b = blockIdx.x, t = threadIdx.x;
  const uint64_t P = (uint64_t)a.n_chunks * a.G;
  const uint64_t blo = P * b / nb, bn = P * (b + 1) / nb - blo;
  const uint64_t lo = blo + bn * t / blockDim.x, hi = blo + bn * (t + 1) / blockDim.x;
  const uint64_t sp = a.snap_piece[k];
  Aff run = aff_id(), pre = aff_id();
  bool mine = false;
  for (uint64_t p = lo; p < hi; ++p) {
    if (p == sp) { pre = run; mine = true; }
    run = compose(run, Aff{a.sig_a[p * 4 + k], a.sig_b[p * 4 + k], 0ull});
  }
  Aff ex, tot;
  block_scan(run, ex, tot, s_red);
  Aff *part = static_cast<Aff *>(a.fin_part) + (uint64_t)k * nb;
  if (mine) {                                        // sigma map: this block's first piece -> snapshot piece
    static_cast<Aff *>(a.fin_pre)[k] = compose(ex, pre);
    a.fin_snapb[k] = b;
  }
  if (t == 0) part[b] = tot;
  __threadfence();
  __syncthreads();
  if (t == 0) s_last = atomicAdd(a.fin_done + k, 1u) == nb - 1u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const Aff x = t < nb ? ld_aff(part + t) : aff_id();
  block_scan(x, ex, tot, s_red);
  if (sp != ~0ull && t == __ldcg(a.fin_snapb + k)) {
    const double sb = apply(compose(ex, ld_aff(static_cast<const Aff *>(a.fin_pre) + k)), a.s0[k]);
    a.out[48 + k] = a.snap_v[k * 4 + 2];
    a.out[64 + k] = apply(Aff{a.snap_v[k * 4 + 0], a.snap_v[k * 4 + 1], 0ull}, sb);
  }
  if (t == 0) {
    a.out[k] = a.cstart_c[(uint64_t)a.n_chunks * 4 + k];
    a.out[16 + k] = apply(tot, a.s0[k]);
    reinterpret_cast<unsigned long long *>(a.out)[32 + k] = a.cstart_n[(uint64_t)a.n_chunks * 4 + k];
  }
}

}  // namespace

size_t calib_stream_smem() { return SLayout::bytes; }
uint32_t calib_stream_fin_blocks() { return kFinBlocks; }
uint32_t calib_stream_piece() { return (uint32_t)(kSW * kSRegion); }

int calib_stream_blocks_per_sm() {
  if (cudaFuncSetAttribute(c_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SLayout::bytes) != cudaSuccess)
    return 0;
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, c_stream, kSThreads, SLayout::bytes) != cudaSuccess) return 0;
  return b;
}

cudaError_t launch_calib_stream(const CalibStreamArgs &a, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(c_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SLayout::bytes);
  if (e != cudaSuccess) return e;
  CalibStreamArgs args = a;
  void *params[] = {&args};
  // every CTA must be resident: phase C waits on flags that other CTAs' phase A publishes
  e = cudaLaunchCooperativeKernel((const void *)c_stream, dim3(a.G), dim3(kSThreads), params, SLayout::bytes, s);
  if (e != cudaSuccess) return e;
  c_stream_final<<<dim3(kFinBlocks, a.n_cats), 256, 0, s>>>(a);
  return cudaGetLastError();
}

namespace {

size_t calib_smem(uint32_t nc, bool reg) {
  // reg: d1 = [nc + 1][256] (row nc: C3's scratch row for dropped feedback)
  return 2 * kStageBytes + kScanBytes + (size_t)(nc + (reg ? 1 : 0)) * kCalBlock * 8 +
         (reg ? 0 : (size_t)nc * kCalBlock * (8 + 4 * 2));
}

template <int NC, bool REG>
cudaError_t set_attrs() {
  const size_t smem = calib_smem(NC, REG);
  cudaError_t e = cudaFuncSetAttribute(c1_maps<NC, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(c3_replay<NC, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int NC, bool REG>
int blocks_per_sm() {
  if (set_attrs<NC, REG>() != cudaSuccess) return 0;
  const size_t smem = calib_smem(NC, REG);
  int b1 = 0, b3 = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, c1_maps<NC, REG>, kCalBlock, smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b3, c3_replay<NC, REG>, kCalBlock, smem) != cudaSuccess)
    return 0;
  return b1 < b3 ? b1 : b3;
}

template <int NC, bool REG>
cudaError_t launch_maps(const CalibArgs &a, cudaStream_t s) {
  cudaError_t e = set_attrs<NC, REG>();
  if (e != cudaSuccess) return e;
  c1_maps<NC, REG><<<(unsigned)a.blocks, kCalBlock, calib_smem(NC, REG), s>>>(a);
  c2_scan<<<a.n_cats, 1024, 0, s>>>(a, 0);
  return cudaGetLastError();
}

template <int NC, bool REG>
cudaError_t launch_replay(const CalibArgs &a, cudaStream_t s) {
  c3_replay<NC, REG><<<(unsigned)a.blocks, kCalBlock, calib_smem(NC, REG), s>>>(a);
  c2_scan<<<a.n_cats, 1024, 0, s>>>(a, 1);
  return cudaGetLastError();
}

}  // namespace

size_t calib_scratch_bytes(uint64_t blocks, uint32_t n_cats) {
  // thrA, thrB (double), thrN, thrC (u32) per (category, thread); blkA, blkB,
  // sblkA, sblkB (double), blkN (u64) per (category, block)
  return (size_t)blocks * n_cats * ((size_t)kCalBlock * (8 * 2 + 4 * 2) + 8 * 5);
}

int calib_blocks_per_sm(uint32_t n_cats) {
  return n_cats <= 4 ? blocks_per_sm<4, true>() : blocks_per_sm<16, false>();
}

cudaError_t launch_calib_maps(const CalibArgs &a, cudaStream_t s) {
  return a.n_cats <= 4 ? launch_maps<4, true>(a, s) : launch_maps<16, false>(a, s);
}

cudaError_t launch_calib_replay(const CalibArgs &a, cudaStream_t s) {
  return a.n_cats <= 4 ? launch_replay<4, true>(a, s) : launch_replay<16, false>(a, s);
}

cudaError_t launch_calib_snap(const CalibArgs &a, cudaStream_t s) {
  c4_snap<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_calibrate(CalibArgs a, cudaStream_t s) {
  cudaError_t e = launch_calib_maps(a, s);
  if (e == cudaSuccess) e = launch_calib_replay(a, s);
  if (e == cudaSuccess) e = launch_calib_snap(a, s);
  return e;
}

}  // namespace fp
