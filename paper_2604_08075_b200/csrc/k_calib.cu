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
// One rank, single pass: every record is read from HBM once.
//
// The stream is cut into tiles of 4,096 records taken in order by a ticket.
// A block stages its tile in shared memory as c_obs (fp64; dropped feedback
// has no category) and lists, per category, the positions of its
// observations in tile order (ballot masks, popcount ranks): a category's
// observations are then read through that list without per-record category
// dispatch. The block's 256 threads form per-category worker groups in
// proportion to the category counts (balanced for any mix); worker j of
// category k owns the j-th slice of k's list.
//   pass A  each worker composes the c_hat maps (Eq. `ema`) of its slice; a
//           scan inside each group gives every worker its exclusive map and
//           the tile's per-category aggregate
//   look-back (decoupled single-pass scan over tiles; block-wide: 256
//           predecessors per round) -> the tile's exact exclusive prefix
//   pass B  each worker replays its slice from its exact start state (tile
//           prefix, then group prefix, applied to c_0) -- the sequential
//           update -- which yields c_hat(before) for every observation and so
//           the sigma maps (R26); the snapshot at the snap_at-th observation;
//           group scan and a second look-back for sigma
// The last tile writes the final state. Reassociation: within 1e-12 of the
// sequential oracle, like the multi-rank kernels above.
// ============================================================================
constexpr uint32_t kTileRecs = 4096;
constexpr uint32_t kTileWords = kTileRecs / 32;
constexpr uint32_t kTileThreads = 256;
constexpr uint32_t kTileWarps = kTileThreads / 32;

template <int NC>
struct TileLayout {
  static constexpr size_t o = 0;                                          // double [4096]
  static constexpr size_t mask = o + kTileRecs * 8;                       // u32 [NC][128]
  static constexpr size_t wpre = mask + (size_t)NC * kTileWords * 4;      // u32 [NC][129]
  static constexpr size_t pos = wpre + (size_t)NC * (kTileWords + 1) * 4; // u16 [4096]
  static constexpr size_t cat = pos + kTileRecs * 2;                      // u8 [4096] (0xFF: dropped)
  static constexpr size_t wmap = (cat + kTileRecs + 15) & ~size_t(15);    // Aff [256]
  static constexpr size_t bytes = wmap + kTileThreads * sizeof(Aff);
};

__device__ __forceinline__ void st_release(unsigned int *p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ Aff ld_aff(const Aff *p) {
  return Aff{__ldcg(&p->a), __ldcg(&p->b), __ldcg(&p->n)};
}

// Per-category exclusive scan of the worker maps wm[g0 .. g0 + P) of each
// group (one warp per group); the group total -> tot[k].
__device__ void group_scan(Aff *wm, const uint32_t *gstart, uint32_t n_cats, Aff *tot) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t k = warp; k < n_cats; k += kTileWarps) {
    const uint32_t g0 = gstart[k], P = gstart[k + 1] - g0;
    const uint32_t q = (P + 31) / 32, lo = min(P, lane * q), hi = min(P, lo + q);
    Aff run = aff_id();
    for (uint32_t i = lo; i < hi; ++i) run = compose(run, wm[g0 + i]);
    const Aff inc = warp_inclusive(run, lane);
    Aff cur = shfl_up(inc, 1);
    if (lane == 0) cur = aff_id();
    for (uint32_t i = lo; i < hi; ++i) {
      const Aff x = wm[g0 + i];
      wm[g0 + i] = cur;
      cur = compose(cur, x);
    }
    if (lane == 31) tot[k] = inc;
  }
}

template <int NC>
struct TileSm {                           // static shared state of one tile
  Aff tot[NC], excl[NC], sexcl[NC], part[NC];
  Aff red[NC][kTileWarps];                // look-back: per-warp partial compositions
  double snapv[NC];
  uint32_t gstart[NC + 1], cbase[NC + 1], snap_w[NC];
  uint32_t tile, last[2];
};

struct TileBuf {
  double *o;
  uint32_t *mask, *wpre;
  uint16_t *pos;
  uint8_t *cat;
  Aff *wm;
};

template <int NC>
__device__ __forceinline__ TileBuf tile_buf(unsigned char *smem) {
  using L = TileLayout<NC>;
  return TileBuf{reinterpret_cast<double *>(smem + L::o), reinterpret_cast<uint32_t *>(smem + L::mask),
                 reinterpret_cast<uint32_t *>(smem + L::wpre), reinterpret_cast<uint16_t *>(smem + L::pos),
                 reinterpret_cast<uint8_t *>(smem + L::cat), reinterpret_cast<Aff *>(smem + L::wmap)};
}

// Stage tile `tile`: c_obs and categories, masks, per-category word prefixes,
// worker groups, per-category position lists. Returns this thread's slice
// [r0, r1) of category kw's list (kw == n_cats: no work).
template <int NC>
__device__ void stage_tile(const CalibTileArgs &a, const TileBuf &X, TileSm<NC> &S, uint32_t tile, uint32_t &kw,
                           uint32_t &r0, uint32_t &r1) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nc = a.n_cats, last_cat = nc - 1;
  const uint64_t base = (uint64_t)tile * kTileRecs;
  // warp w stages words 16 w .. 16 w + 15 (coalesced 128-B column loads per word)
#pragma unroll 1
  for (uint32_t i0 = 0; i0 < 16; i0 += 4) {
    uint32_t vb[4], vt[4], vc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = base + (uint64_t)(warp * 16 + i0 + u) * 32 + lane;
      const bool in = i < a.n;
      vb[u] = in ? __ldcs(a.bytes + i) : 0u;
      vt[u] = in ? __ldcs(a.tokens + i) : 0u;
      vc[u] = in ? (uint32_t)__ldcs(a.cat + i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t word = warp * 16 + i0 + u, r = word * 32 + lane;
      const bool valid = vt[u] != 0u;                           // zero-token feedback is dropped
      const uint32_t k = vc[u] < last_cat ? vc[u] : last_cat;   // R23
      X.o[r] = ratio(vb[u], vt[u] | (vt[u] == 0u));
      X.cat[r] = valid ? (uint8_t)k : (uint8_t)0xFF;
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        if (j < (int)nc) {
          const unsigned mk = __ballot_sync(0xffffffffu, valid && k == (uint32_t)j);
          if (lane == (uint32_t)j) X.mask[j * kTileWords + word] = mk;
        }
      }
    }
  }
  __syncthreads();
  // per category: exclusive prefix of the observation counts over words
  for (uint32_t k = warp; k < nc; k += kTileWarps) {
    const uint32_t *mk = X.mask + k * kTileWords;
    uint32_t c[4], run = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) { c[u] = __popc(mk[lane * 4 + u]); run += c[u]; }
    uint32_t inc = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= (uint32_t)off) inc += y;
    }
    uint32_t ex = inc - run;
    uint32_t *wp = X.wpre + k * (kTileWords + 1);
#pragma unroll
    for (int u = 0; u < 4; ++u) { wp[lane * 4 + u] = ex; ex += c[u]; }
    if (lane == 31) wp[kTileWords] = inc;
  }
  __syncthreads();
  // list offsets and worker groups in proportion to the category counts
  if (threadIdx.x == 0) {
    uint32_t total = 0, nonempty = 0, big = 0, bigc = 0;
    for (uint32_t k = 0; k < nc; ++k) {
      const uint32_t ck = X.wpre[k * (kTileWords + 1) + kTileWords];
      S.cbase[k] = total;
      total += ck;
      nonempty += ck ? 1u : 0u;
      if (ck > bigc) { big = k; bigc = ck; }
    }
    S.cbase[nc] = total;
    uint32_t used = 0;
    for (uint32_t k = 0; k < nc; ++k) {
      const uint32_t ck = X.wpre[k * (kTileWords + 1) + kTileWords];
      used += ck ? 1u + (uint32_t)((uint64_t)ck * (kTileThreads - nonempty) / total) : 0u;
    }
    const uint32_t extra = total ? kTileThreads - used : 0u;
    uint32_t g0 = 0;
    for (uint32_t k = 0; k < nc; ++k) {
      const uint32_t ck = X.wpre[k * (kTileWords + 1) + kTileWords];
      S.gstart[k] = g0;
      g0 += (ck ? 1u + (uint32_t)((uint64_t)ck * (kTileThreads - nonempty) / total) : 0u) + (k == big ? extra : 0u);
    }
    S.gstart[nc] = g0;
  }
  __syncthreads();
  // position lists: record r of category k -> pos[cbase[k] + rank of r in k]
#pragma unroll 4
  for (uint32_t i = 0; i < 16; ++i) {
    const uint32_t word = warp * 16 + i, r = word * 32 + lane;
    const uint32_t k = X.cat[r];
    if (k != 0xFFu) {
      const uint32_t below = X.mask[k * kTileWords + word] & ((1u << lane) - 1u);
      X.pos[S.cbase[k] + X.wpre[k * (kTileWords + 1) + word] + __popc(below)] = (uint16_t)r;
    }
  }
  kw = 0;
  while (kw < nc && S.gstart[kw + 1] <= threadIdx.x) ++kw;
  r0 = r1 = 0;
  if (kw < nc) {
    const uint32_t P = S.gstart[kw + 1] - S.gstart[kw], j = threadIdx.x - S.gstart[kw];
    const uint32_t ck = S.cbase[kw + 1] - S.cbase[kw];
    r0 = S.cbase[kw] + ck * j / P;
    r1 = S.cbase[kw] + ck * (j + 1) / P;
  }
  __syncthreads();
}

// Decoupled look-back over the whole block (one predecessor per thread, 256
// per round): publish this tile's aggregates (flag 1), compose the
// predecessors' aggregates / inclusive prefixes into the exclusive prefix
// excl[k], publish the inclusive prefix (flag 2). A round covers 256 tiles,
// so the walk back to the nearest inclusive prefix stays about one round deep
// at the stream's tile rate. Flags are polled relaxed (no L1 invalidation per
// poll); one fence after they are seen orders the map reads.
// desc: [tile][2 (aggregate, inclusive)][NC] maps.
template <int NC>
__device__ void look_back_block(uint32_t tile, uint32_t n_cats, unsigned int *flags, Aff *desc, const Aff *agg,
                                Aff *excl, TileSm<NC> &S) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Aff *mine = desc + (size_t)tile * 2 * NC;
  if (threadIdx.x < n_cats) {
    mine[threadIdx.x] = agg[threadIdx.x];
    if (tile == 0) mine[NC + threadIdx.x] = agg[threadIdx.x];
    excl[threadIdx.x] = aff_id();
  }
  if (threadIdx.x == 0) { S.last[0] = 0xffffffffu; S.last[1] = 0u; }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(flags + tile, tile == 0 ? 2u : 1u);
  if (tile == 0) return;
  int64_t top = (int64_t)tile - 1;
  for (;;) {
    const int64_t p = top - (int64_t)threadIdx.x;
    unsigned int f = 0;
    if (p >= 0) {
      for (;;) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(flags + p) : "memory");
        if (f) break;
        __nanosleep(20);
      }
    }
    __threadfence();                     // acquire: the maps published before the flag
    // the nearest predecessor with an inclusive prefix (lowest thread), else the oldest valid one
    const unsigned inc_w = __ballot_sync(0xffffffffu, p >= 0 && f == 2u);
    const unsigned val_w = __ballot_sync(0xffffffffu, p >= 0);
    if (lane == 0 && inc_w) atomicMin(&S.last[0], warp * 32 + (uint32_t)__ffs(inc_w) - 1);
    if (lane == 0 && val_w) atomicMax(&S.last[1], warp * 32 + 31 - (uint32_t)__clz(val_w));
    __syncthreads();
    const bool found = S.last[0] != 0xffffffffu;
    const uint32_t last = found ? S.last[0] : S.last[1];
    // every category at once: warp-ordered reductions, then one thread per category
    for (uint32_t k = 0; k < n_cats; ++k) {
      Aff x = aff_id();
      if (threadIdx.x <= last)
        x = ld_aff(desc + ((size_t)p * 2 + ((threadIdx.x == last && f == 2u) ? 1 : 0)) * NC + k);
      // older predecessors (higher threads) are applied first
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const Aff y = Aff{__shfl_down_sync(0xffffffffu, x.a, o), __shfl_down_sync(0xffffffffu, x.b, o),
                          __shfl_down_sync(0xffffffffu, x.n, o)};
        if ((lane & (2 * o - 1)) == 0) x = compose(y, x);
      }
      if (lane == 0) S.red[k][warp] = x;
    }
    __syncthreads();
    if (threadIdx.x < n_cats) {
      const uint32_t k = threadIdx.x;
      Aff acc = S.red[k][kTileWarps - 1];
      for (int w = (int)kTileWarps - 2; w >= 0; --w) acc = compose(acc, S.red[k][w]);
      excl[k] = compose(acc, excl[k]);
    }
    if (found) break;
    __syncthreads();
    if (threadIdx.x == 0) { S.last[0] = 0xffffffffu; S.last[1] = 0u; }
    __syncthreads();
    top -= (int64_t)kTileThreads;
  }
  __syncwarp();
  if (threadIdx.x < n_cats) mine[NC + threadIdx.x] = compose(excl[threadIdx.x], agg[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(flags + tile, 2u);
}

template <int NC>
__global__ void __launch_bounds__(kTileThreads, NC <= 4 ? 4 : 3) c_single(CalibTileArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ TileSm<NC> S;
  const TileBuf X = tile_buf<NC>(smem);
  const uint32_t nc = a.n_cats;
  if (threadIdx.x == 0) S.tile = atomicAdd(a.ticket, 1u);
  if (threadIdx.x < NC) S.snap_w[threadIdx.x] = 0xffffffffu;
  __syncthreads();
  const uint32_t tile = S.tile;
  Aff *cdesc = static_cast<Aff *>(a.cdesc), *sdesc = static_cast<Aff *>(a.sdesc);
  const double beta = a.beta, wgt = __dsub_rn(1.0, a.beta);
  uint32_t kw, r0, r1;
  stage_tile<NC>(a, X, S, tile, kw, r0, r1);
  // ---- pass A: c_hat maps ----
  {
    double b = 0.0;
    for (uint32_t r = r0; r < r1; ++r) b = __fma_rn(beta, b, __dmul_rn(wgt, X.o[X.pos[r]]));
    X.wm[threadIdx.x] = Aff{pow_n(beta, r1 - r0), b, (unsigned long long)(r1 - r0)};
  }
  __syncthreads();
  group_scan(X.wm, S.gstart, nc, S.tot);
  __syncthreads();
  look_back_block<NC>(tile, nc, a.cflag, cdesc, S.tot, S.excl, S);
  __syncthreads();
  // ---- pass B: replay from the exact start state; sigma maps; snapshot ----
  double sb = 0.0;
  if (r1 > r0) {
    const Aff p0 = compose(S.excl[kw], X.wm[threadIdx.x]);
    double cv = apply(p0, a.c0[kw]);
    const unsigned long long before = p0.n;
    const uint64_t target = (a.snap_at > before && a.snap_at - before <= r1 - r0) ? a.snap_at - before : 0ull;
    for (uint32_t r = r0; r < r1; ++r) {
      const double x = X.o[X.pos[r]];
      const double prev = cv;
      cv = __fma_rn(beta, prev, __dmul_rn(wgt, x));
      sb = __fma_rn(beta, sb, __dmul_rn(wgt, fabs(__dsub_rn(x, prev))));
      if (r - r0 + 1 == target) {
        S.snapv[kw] = cv;
        S.part[kw] = Aff{pow_n(beta, (uint32_t)target), sb, 0ull};
        S.snap_w[kw] = threadIdx.x;
      }
    }
  }
  __syncthreads();                                   // every worker has read its c map
  X.wm[threadIdx.x] = Aff{pow_n(beta, r1 - r0), sb, 0ull};
  __syncthreads();
  group_scan(X.wm, S.gstart, nc, S.tot);
  __syncthreads();
  look_back_block<NC>(tile, nc, a.sflag, sdesc, S.tot, S.sexcl, S);
  __syncthreads();
  if (threadIdx.x < nc) {
    const uint32_t k = threadIdx.x;
    if (S.snap_w[k] != 0xffffffffu) {                // the snap_at-th observation of category k is here
      const Aff m = compose(S.sexcl[k], compose(X.wm[S.snap_w[k]], S.part[k]));
      a.out[48 + k] = S.snapv[k];
      a.out[64 + k] = apply(m, a.s0[k]);
    }
    if (tile == a.n_tiles - 1) {                     // the last tile: the final state
      const Aff ci = ld_aff(cdesc + ((size_t)tile * 2 + 1) * NC + k);
      const Aff si = compose(S.sexcl[k], S.tot[k]);
      a.out[k] = apply(ci, a.c0[k]);
      a.out[16 + k] = apply(si, a.s0[k]);
      reinterpret_cast<unsigned long long *>(a.out)[32 + k] = ci.n;
    }
  }
}

template <int NC>
cudaError_t launch_single(const CalibTileArgs &a, cudaStream_t s) {
  const size_t smem = TileLayout<NC>::bytes;
  cudaError_t e = cudaFuncSetAttribute(c_single<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  c_single<NC><<<(unsigned)a.n_tiles, kTileThreads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

uint64_t calib_tiles(uint64_t n) { return (n + kTileRecs - 1) / kTileRecs; }

cudaError_t launch_calib_tile(const CalibTileArgs &a, int, cudaStream_t s) {
  return a.n_cats <= 4 ? launch_single<4>(a, s) : launch_single<16>(a, s);
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
