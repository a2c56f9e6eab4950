// K1: the trace pass of sweep_thresholds (K4, route_batch, is in k_route.cu).
//
// K1 streams the u32 L_total column once (128-bit loads, one contiguous
// tile of blockDim x 64 B per block per step, 4 loads in flight per thread)
// and routes every request against EVERY candidate at once: its bin
//     b(L) = #{e in E : e < L}          (E = sortuniq(B u C_L), "<=")
// is read from a fine-cell LUT in shared memory (cell = ceil(min(L, e_max+1)
// / 2^s); every edge is a multiple of 2^s, so the LUT is exact), and the
// request adds 1 to cnt[b] and L to mass[b]. A request in bin b is short for
// every candidate with B >= e_b, long for B < L <= C_L and rejected for
// L > C_L, so the scan of this histogram (K3 prologue) gives every
// candidate's routing outcome of Alg. 1 with bit-exact counts.
//
// Histogram layout: R replicas x (|E|+1) bins of u32 counters in shared
// memory; with R = 32 every lane owns a replica ("lane-private"), so the 32
// atomics of one warp instruction hit 32 distinct banks whatever the length
// distribution (no same-address serialisation on skewed traces). Mass uses
// u32 slots flushed into a u64 per-bin accumulator before they can overflow
// (64-bit shared atomics are a CAS loop on sm_100a: ATOMS.CAST.SPIN.64). The
// bin above the last edge also receives its L (so the hot loop has no
// branch); that slot may wrap and is never published -- no candidate uses
// the mass of requests above every edge. When e_max is too large for the
// u32 flush bound the mass is split into 16-bit halves.
//
// The kernel is issue-bound unless the per-request instruction count is
// small (ncu r01: 21 instr/request -> 82% issue-active at 5.5 TB/s), so the
// hot loop is: VIMNMX, IADD, SHF (cell), LDS.U8 (bin), LEA (slot), ATOMS x2.
#include <algorithm>
#include <cstdio>
#include "estimate.cuh"
#include "internal.cuh"

namespace fp {

namespace {

constexpr int kUnroll = 4;   // uint4 loads in flight per thread per step

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

struct K1Ctx {
  const unsigned char *lut;  // LUT bytes (or the edge list in binary-search mode)
  unsigned char *hist;       // R = 32: [nbins][W][32] u32 (W = 1 cnt, 2 cnt|mass, 3 cnt|lo|hi)
                             // R = 1:  [nbins][W] u32
  unsigned long long *acc;   // [nbins] u64 mass accumulator
  uint32_t clampv;           // e_max + 1
  uint32_t round;            // 2^s - 1
  uint32_t shift;            // s
  uint32_t n_edges;
  uint32_t lane4;            // lane * 4 (R = 32) or 0
};

template <int R, bool SPLIT, bool MASS>
struct Layout {
  static constexpr uint32_t W = MASS ? (SPLIT ? 3u : 2u) : 1u;   // u32 words per slot kind
  static constexpr uint32_t kStride = (R == 32) ? 128u : 4u;     // bytes between kinds
  static_assert(kStride == 128u || kStride == 4u, "");
  static constexpr uint32_t kBinShift = (R == 32) ? (W == 1 ? 7 : W == 2 ? 8 : 0) : (W == 1 ? 2 : W == 2 ? 3 : 0);
  __device__ static __forceinline__ uint32_t bin_off(uint32_t b) {
    if constexpr (kBinShift) return b << kBinShift;
    else return b * (W * kStride);
  }
};

// bin = #{e in E : e < L}
template <int LUTW>
__device__ __forceinline__ uint32_t bin_of(const K1Ctx &c, uint32_t L) {
  if constexpr (LUTW == 1 || LUTW == 2) {
    // plan guarantees e_max + 2^s <= 2^32 - 1, so this cannot overflow
    const uint32_t cell = (min(L, c.clampv) + c.round) >> c.shift;
    if constexpr (LUTW == 1) return (uint32_t)c.lut[cell];
    else return (uint32_t)reinterpret_cast<const uint16_t *>(c.lut)[cell];
  } else {
    // binary search (large or irregular edge sets): lower_bound of L in E
    const uint32_t *edges = reinterpret_cast<const uint32_t *>(c.lut);
    uint32_t lo = 0, n = c.n_edges;
    while (n > 0) {
      uint32_t half = n >> 1;
      if (edges[lo + half] < L) { lo += half + 1; n -= half + 1; } else { n = half; }
    }
    return lo;
  }
}

template <int LUTW, int R, bool SPLIT, bool MASS>
__device__ __forceinline__ uint32_t add_one(const K1Ctx &c, uint32_t L) {
  using Ly = Layout<R, SPLIT, MASS>;
  const uint32_t b = bin_of<LUTW>(c, L);
  unsigned char *slot = c.hist + Ly::bin_off(b) + c.lane4;
  atomicAdd(reinterpret_cast<uint32_t *>(slot), 1u);
  if constexpr (MASS) {
    if constexpr (SPLIT) {
      atomicAdd(reinterpret_cast<uint32_t *>(slot + Ly::kStride), L & 0xFFFFu);
      atomicAdd(reinterpret_cast<uint32_t *>(slot + 2 * Ly::kStride), L >> 16);
    } else {
      atomicAdd(reinterpret_cast<uint32_t *>(slot + Ly::kStride), L);
    }
  }
  return b;
}

// speculative routing: Alg. 1's decision byte from a bin for the split's edge
// indices (pool + 4 stage, k_route.cu dec_byte), SWAR for bins < 128: adding
// 0x7F - j sets a byte's top bit iff the byte is > j
struct DecK {
  uint32_t kB, kCS, kCL;
};
__device__ __forceinline__ DecK dec_k(uint32_t iB, uint32_t iCS, uint32_t iCL) {
  auto r = [](uint32_t j) { return (0x7Fu - (j < 0x7Fu ? j : 0x7Fu)) * 0x01010101u; };
  return DecK{r(iB), r(iCS), r(iCL)};
}
__device__ __forceinline__ uint32_t dec_word(uint32_t w, const DecK &k) {
  const uint32_t gB = (w + k.kB) & 0x80808080u, gS = (w + k.kCS) & 0x80808080u, gL = (w + k.kCL) & 0x80808080u;
  return (gB >> 7) + (gS >> 5) + (gL >> 7) * 9u;
}

// the same decision byte from L_total itself, for edge sets whose bins do not
// fit the SWAR compare (u16 LUT: |E| >= 256): bin > j <=> e_j < L (E is sorted
// and unique), so d = [L > B] + 4 [L > C_S] + 9 [L > C_L] with the split's
// edge values -- dec_word's byte exactly
struct DecL {
  uint32_t vB, vCS, vCL;
};
__device__ __forceinline__ uint32_t dec_l1(uint32_t L, const DecL &k) {
  return (L > k.vB ? 1u : 0u) + (L > k.vCS ? 4u : 0u) + (L > k.vCL ? 9u : 0u);
}
__device__ __forceinline__ uint32_t dec_l4(const uint4 &v, const DecL &k) {
  return dec_l1(v.x, k) | (dec_l1(v.y, k) << 8) | (dec_l1(v.z, k) << 16) | (dec_l1(v.w, k) << 24);
}

// the byte a request's bin is stored as: the bin itself when |E| < 256 (u8
// LUT), else min(bin, 255) -- 255 then stands for "bin >= 255" (the routing
// pass reads L_total back for such requests only when the routed split has an
// edge index >= 255)
template <int LUTW>
__device__ __forceinline__ uint32_t bin_byte(uint32_t b) { return LUTW == 1 ? b : min(b, 255u); }

// returns the four bins packed in bytes (bin_byte)
template <int LUTW, int R, bool SPLIT, bool MASS>
__device__ __forceinline__ uint32_t add_four(const K1Ctx &c, const uint4 &v) {
  const uint32_t b0 = bin_byte<LUTW>(add_one<LUTW, R, SPLIT, MASS>(c, v.x));
  const uint32_t b1 = bin_byte<LUTW>(add_one<LUTW, R, SPLIT, MASS>(c, v.y));
  const uint32_t b2 = bin_byte<LUTW>(add_one<LUTW, R, SPLIT, MASS>(c, v.z));
  const uint32_t b3 = bin_byte<LUTW>(add_one<LUTW, R, SPLIT, MASS>(c, v.w));
  return b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
}

template <int R, bool SPLIT>
__device__ __forceinline__ void flush_mass(const K1Ctx &c, uint32_t nbins) {
  using Ly = Layout<R, SPLIT, true>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if constexpr (R == 32) {
    for (uint32_t j = warp; j < nbins; j += nw) {
      uint32_t *lo = reinterpret_cast<uint32_t *>(c.hist + Ly::bin_off(j) + Ly::kStride) + lane;
      unsigned long long v = *lo;
      *lo = 0;
      if constexpr (SPLIT) {
        uint32_t *hi = lo + 32;
        v += (unsigned long long)*hi << 16;
        *hi = 0;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) c.acc[j] += v;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < nbins; j += blockDim.x) {
      uint32_t *lo = reinterpret_cast<uint32_t *>(c.hist + Ly::bin_off(j) + Ly::kStride);
      unsigned long long v = *lo;
      *lo = 0;
      if constexpr (SPLIT) {
        v += (unsigned long long)lo[1] << 16;
        lo[1] = 0;
      }
      c.acc[j] += v;
    }
  }
}

// ---- element sources -------------------------------------------------------------
// Plain: the caller's L_total column. Raw (NEXT-1): body bytes, max_output and
// category columns; L_total is estimated in the kernel with Eq. `budget`
// from the per-category conservative ratio c* of Eq.
// `conservative`, computed once per block into shared memory.
struct SrcPlain {
  const uint32_t *len;
  __device__ __forceinline__ uint4 load4(const uint4 *p4, uint64_t i) const { return ldg_stream(p4 + i); }
  __device__ __forceinline__ uint32_t load1(uint64_t i) const { return len[i]; }
};

struct SrcRaw {
  const uint32_t *body, *mo;
  const uint8_t *cat;
  const double2 *tab;    // shared memory [256]: {1/c*, c*} per category byte
  uint64_t base;         // element offset of uint4 index 0 (the aligned head)
  __device__ __forceinline__ uint4 load4(const uint4 *, uint64_t i) const {
    const uint64_t e = base + 4 * i;
    const uint4 b = ldg_stream(reinterpret_cast<const uint4 *>(body + e));
    const uint4 m = ldg_stream(reinterpret_cast<const uint4 *>(mo + e));
    const uint32_t k = __ldg(reinterpret_cast<const unsigned int *>(cat + e));
    return make_uint4(estimate_l_total(b.x, m.x, k & 0xFFu, tab), estimate_l_total(b.y, m.y, (k >> 8) & 0xFFu, tab),
                      estimate_l_total(b.z, m.z, (k >> 16) & 0xFFu, tab), estimate_l_total(b.w, m.w, k >> 24, tab));
  }
  __device__ __forceinline__ uint32_t load1(uint64_t i) const { return estimate_l_total(body[i], mo[i], cat[i], tab); }
};

// The 6-bit packing of a thread's step (4 words w_u of 4 byte-bins each,
// every bin < 64), SIMD within the words -- no per-bin extraction:
//   lo (u64) = (w0 & 0x0F..) | (w1 & 0x0F..) << 4  |  ((w2 & 0x0F..) | (w3 & 0x0F..) << 4) << 32
//   hi (u32) = sum_u ((w_u >> 4) & 0x03030303) << 2u
// i.e. byte e of each half of lo holds the low nibbles of bins (u, e) and
// (u + 1, e), byte e of hi the high 2-bit parts of bins (0..3, e). ALU only
// (no shuffles: the hot loop's shared-memory atomics already load the MIO pipe).
__device__ __forceinline__ void pack_step(const uint32_t (&w)[4], unsigned long long &lo, uint32_t &hi) {
  const uint32_t l01 = (w[0] & 0x0F0F0F0Fu) | ((w[1] & 0x0F0F0F0Fu) << 4);
  const uint32_t l23 = (w[2] & 0x0F0F0F0Fu) | ((w[3] & 0x0F0F0F0Fu) << 4);
  lo = (unsigned long long)l01 | ((unsigned long long)l23 << 32);
  hi = ((w[0] >> 4) & 0x03030303u) | (((w[1] >> 4) & 0x03030303u) << 2) | (((w[2] >> 4) & 0x03030303u) << 4) |
       (((w[3] >> 4) & 0x03030303u) << 6);
}

__device__ __forceinline__ void store_chunk(const TraceArgs &a, uint64_t c, unsigned long long lo, uint32_t hi) {
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(a.bins_out + 8 * c), "l"(lo) : "memory");
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(a.bins_hi + 4 * c), "r"(hi) : "memory");
}

// BINS: also write each request's bin (u8; |E| < 256) to a.bins_out, where
// (a.bins_out + element index) is 4-B aligned for every uint4 of the body;
// BINS && PACK: the 6-bit chunks of a.bins_out / a.bins_hi (|E| < 64).
template <int LUTW, int R, bool SPLIT, bool MASS, bool RAW, bool BINS, bool PACK = false>
__global__ void __launch_bounds__(512, (RAW || BINS) ? 3 : 1) k1_trace(TraceArgs a) {
  // raw: 3 columns per request (36 B per uint4 step in flight), 2 steps per
  // thread at 3 x 512 threads/SM keep ~110 KB/SM in flight within 42 registers
  constexpr int U = RAW ? 2 : kUnroll;
  // a programmatic dependent (K3, or the fold kernel) may be scheduled right
  // away into the room this grid leaves on each SM: it loads the plan's tables
  // and then waits (griddepcontrol.wait) for this grid to complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t nbins = a.n_edges + 1;
  uint32_t lut_bytes = (LUTW == 0) ? a.n_edges * 4 : a.lut_cells * LUTW;
  lut_bytes = (lut_bytes + 15u) & ~15u;
  K1Ctx c;
  c.lut = smem;
  c.acc = reinterpret_cast<unsigned long long *>(smem + lut_bytes);
  // RAW: [256] {1/c*, c*}, 16-B aligned for one LDS.128 per request. Offsets
  // are integer arithmetic on `smem` so the compiler keeps the shared state
  // space (a pointer rounded through uintptr_t becomes generic: ATOM.E/LD.E)
  const uint32_t cst_off = RAW ? ((lut_bytes + nbins * 8u + 15u) & ~15u) : lut_bytes + nbins * 8u;
  double2 *cstar = reinterpret_cast<double2 *>(smem + cst_off);
  c.hist = smem + cst_off + (RAW ? 16u * kCatTable : 0u);
  c.clampv = a.max_edge + 1u;
  c.round = (1u << a.shift) - 1u;
  c.shift = a.shift;
  c.n_edges = a.n_edges;
  c.lane4 = (R == 32) ? (threadIdx.x & 31u) * 4u : 0u;

  // stage the LUT (or the edge list), the routing ratios, and clear the histogram
  {
    const uint32_t *src = (LUTW == 0) ? a.edges : reinterpret_cast<const uint32_t *>(a.lut);
    uint32_t *dst = reinterpret_cast<uint32_t *>(smem);
    // the device tables are padded to 16 B inside the plan's table blob
    for (uint32_t i = threadIdx.x; i < lut_bytes / 4; i += blockDim.x) dst[i] = src[i];
    for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) c.acc[i] = 0ull;
    if (RAW) setup_cstar(a.calib, a.n_cats, a.gamma, a.c_floor, cstar);
    const uint32_t words = nbins * R * (MASS ? (SPLIT ? 3u : 2u) : 1u);
    uint32_t *h = reinterpret_cast<uint32_t *>(c.hist);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) h[i] = 0u;
  }
  __syncthreads();

  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t me = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t since_flush = 0;
  auto maybe_flush = [&](uint32_t period) {
    if (MASS && ++since_flush == period) {
      since_flush = 0;
      __syncthreads();
      flush_mass<R, SPLIT>(c, nbins);
      __syncthreads();
    }
  };

  // element source; RAW without a common 16-B phase of the columns -> scalar rounds
  SrcPlain sp{a.len};
  SrcRaw sr{a.body, a.maxout, a.cat, cstar, 0};
  const uintptr_t anchor = RAW ? reinterpret_cast<uintptr_t>(a.body) : reinterpret_cast<uintptr_t>(a.len);
  const uint32_t mis = (uint32_t)((anchor & 15u) >> 2);
  const uint64_t head = (RAW && !a.raw_vec) ? a.n : (mis ? umin64(a.n, 4u - mis) : 0u);
  const uint64_t n4 = (a.n - head) >> 2;                       // uint4 count of the body
  const uint64_t tail_first = head + (n4 << 2);
  sr.base = head;
  auto load1 = [&](uint64_t i) -> uint32_t { return RAW ? sr.load1(i) : sp.load1(i); };

  if (RAW && !a.raw_vec) {
    // scalar rounds over the whole trace (uniform trip count: flush-safe)
    const uint64_t rounds = (a.n + S - 1) / S;
    for (uint64_t r = 0; r < rounds; ++r) {
      const uint64_t i = r * S + me;
      if (i < a.n) add_one<LUTW, R, SPLIT, MASS>(c, load1(i));
      maybe_flush(a.flush_iters * 4u * kUnroll);
    }
  } else {
    // speculative routing: the split to write decisions for (after the
    // predecessor -- the sample's K3 -- has completed)
    bool store = true;
    DecK dk{0u, 0u, 0u};
    DecL dl{0u, 0u, 0u};
    // decisions by SWAR on the bin bytes (u8 LUT; the host speculates there
    // only for |E| < 127) or, for the u16 LUT's clamped bins, from L_total
    constexpr bool swar = LUTW == 1;
    // a programmatic-dependent launch (the sample pass after the previous
    // step's verify): nothing of the predecessor's is read before this wait
    if (a.pdl && !a.dec_route) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (BINS && !PACK && a.dec_route) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      uint4 rt;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(rt.x), "=r"(rt.y), "=r"(rt.z), "=r"(rt.w) : "l"(a.dec_route));
      store = rt.w != 0u;
      dk = dec_k(rt.x, rt.y, rt.z);
      if (!swar && store) dl = DecL{__ldg(a.edges + rt.x), __ldg(a.edges + rt.y), __ldg(a.edges + rt.z)};
    }
    const bool decm = BINS && !PACK && a.dec_route;
    uint32_t *bins4 = (BINS && !PACK) ? reinterpret_cast<uint32_t *>(a.bins_out + head) : nullptr;
    auto dec1 = [&](uint32_t b, uint32_t L) { return swar ? dec_word(b, dk) : dec_l1(L, dl); };
    if (a.step_stride == 1u && blockIdx.x == 0 && threadIdx.x < head) {
      const uint32_t L = load1(threadIdx.x);
      const uint32_t b = add_one<LUTW, R, SPLIT, MASS>(c, L);
      if (BINS && store)
        (PACK ? a.bins_side : a.bins_out)[threadIdx.x] = (uint8_t)(decm ? dec1(b, L) : bin_byte<LUTW>(b));
    }
    if (a.step_stride == 1u && blockIdx.x == gridDim.x - 1 && threadIdx.x < a.n - tail_first) {
      const uint32_t L = load1(tail_first + threadIdx.x);
      const uint32_t b = add_one<LUTW, R, SPLIT, MASS>(c, L);
      if (BINS && store) {
        if (PACK) a.bins_side[4 + threadIdx.x] = (uint8_t)b;
        else a.bins_out[tail_first + threadIdx.x] = (uint8_t)(decm ? dec1(b, L) : bin_byte<LUTW>(b));
      }
    }
    auto dec4 = [&](uint32_t w, const uint4 &v) { return swar ? dec_word(w, dk) : dec_l4(v, dl); };
    const uint4 *body = reinterpret_cast<const uint4 *>(a.len + head);
    // grid-stride stripes: at every step the whole grid reads kUnroll contiguous
    // stripes of gridDim x blockDim x 16 B (measured 7.2 TB/s read-only vs
    // 6.6 TB/s for per-block contiguous tiles; profiles/r01_microbench_*).
    // The step count is uniform over the grid so the flush barrier is safe.
    const uint64_t step4 = S * U;
    const uint64_t full_steps = n4 / step4;
    const uint64_t nsteps = (n4 + step4 - 1) / step4;
    for (uint64_t k = 0; k < nsteps; k += a.step_stride) {
      const uint64_t base = k * step4 + me;
      if (k < full_steps) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = RAW ? sr.load4(body, base + u * S) : sp.load4(body, base + u * S);
        uint32_t pw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t w = add_four<LUTW, R, SPLIT, MASS>(c, v[u]);
          if (BINS && PACK) pw[u & 3] = w;
          else if (BINS && store)
            asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(bins4 + base + u * S), "r"(decm ? dec4(w, v[u]) : w)
                         : "memory");
        }
        if (BINS && PACK) {
          unsigned long long plo;
          uint32_t phi;
          pack_step(pw, plo, phi);
          store_chunk(a, k * S + me, plo, phi);
        }
      } else {
        uint32_t pw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t j = base + u * S;
          if (j < n4) {
            const uint4 vj = RAW ? sr.load4(body, j) : sp.load4(body, j);
            const uint32_t w = add_four<LUTW, R, SPLIT, MASS>(c, vj);
            if (BINS && PACK) pw[u & 3] = w;
            else if (BINS && store) bins4[j] = decm ? dec4(w, vj) : w;
          }
        }
        if (BINS && PACK) {
          unsigned long long plo;
          uint32_t phi;
          pack_step(pw, plo, phi);
          store_chunk(a, k * S + me, plo, phi);
        }
      }
      maybe_flush(a.flush_iters);
    }
  }
  __syncthreads();
  if (MASS) {
    flush_mass<R, SPLIT>(c, nbins);
    __syncthreads();
  }
  // fold replicas and publish this block's histogram (mass of the last bin,
  // above every edge, is not part of the result)
  using Ly = Layout<R, SPLIT, MASS>;
  // this block's copy of the global accumulators: with one copy, 444 blocks x
  // 2 |E| same-address u64 atomics serialise at a few L2 slices (~35 ns per
  // block on C2; the C2 step's K1 fell from 33 to 23 us with 148 blocks)
  // (the block index is re-read here by a volatile asm, which the compiler
  // cannot hoist above the main loop's volatile loads: computed up front, the
  // copy address stayed live through the loop and cost a spill and ~7% on the
  // raw-column trace pass)
  uint32_t bx;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(bx));
  unsigned long long *g_cnt = a.g_cnt + (size_t)(bx & (a.hist_copies - 1u)) * 2 * nbins;
  unsigned long long *g_mass = g_cnt + nbins;
  if constexpr (R == 32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t j = warp; j < nbins; j += nw) {
      unsigned long long v = reinterpret_cast<const uint32_t *>(c.hist + Ly::bin_off(j))[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) {
        if (v) atomicAdd(g_cnt + j, v);
        if (MASS && j < a.n_edges && c.acc[j]) atomicAdd(g_mass + j, c.acc[j]);
      }
    }
  } else {
    for (uint32_t j = threadIdx.x; j < nbins; j += blockDim.x) {
      const uint32_t v = *reinterpret_cast<const uint32_t *>(c.hist + Ly::bin_off(j));
      if (v) atomicAdd(g_cnt + j, (unsigned long long)v);
      if (MASS && j < a.n_edges && c.acc[j]) atomicAdd(g_mass + j, c.acc[j]);
    }
  }
}

// ---- variant selection ----------------------------------------------------------
struct Variant {
  bool raw;      // estimate L_total from raw columns (NEXT-1)
  bool bins;     // also write per-request bins (u8)
  bool pack;     // ... 6-bit packed (|E| < 64)
  int lutw;      // 1, 2 (LUT bytes per cell) or 0 (binary search)
  int R;         // 32 lane-private replicas or 1
  bool split;    // 16-bit mass halves
  bool mass;
};

uint32_t adds_per_iter(int R, int block) { return R == 32 ? (uint32_t)(block / 32) * 4 * kUnroll : (uint32_t)block * 4 * kUnroll; }

size_t smem_for(const TraceArgs &a, const Variant &v) {
  const uint32_t nbins = a.n_edges + 1;
  size_t lut = v.lutw == 0 ? (size_t)a.n_edges * 4 : (size_t)a.lut_cells * v.lutw;
  lut = (lut + 15) & ~size_t(15);
  const uint32_t words = v.mass ? (v.split ? 3u : 2u) : 1u;
  return lut + (size_t)nbins * 8 + (v.raw ? (size_t)kCatTable * 16 + 8 : 0) + (size_t)nbins * v.R * words * 4;
}

Variant choose(const TraceArgs &a, int block) {
  Variant v;
  v.raw = a.body != nullptr;
  v.bins = a.bins_out != nullptr;
  v.pack = v.bins && a.bins_pack;
  v.lutw = a.lut_cells ? (a.lut_u8 ? 1 : 2) : 0;
  v.mass = a.want_mass != 0;
  v.R = 32;
  // split when a u32 slot could overflow in fewer than 16 steps
  v.split = false;
  if (v.mass) {
    unsigned long long per = (unsigned long long)adds_per_iter(32, block) * a.max_edge;
    v.split = per * 16ull > 0xFFFFFFFFull;
  }
  if (smem_for(a, v) > 100 * 1024) {
    v.R = 1;
    if (v.mass) v.split = (unsigned long long)adds_per_iter(1, block) * a.max_edge * 4ull > 0xFFFFFFFFull;
  }
  return v;
}

uint32_t flush_iters_for(const TraceArgs &a, const Variant &v, int block) {
  if (!v.mass) return 1;
  const unsigned long long per_add = v.split ? 0xFFFFull : (unsigned long long)a.max_edge;
  const unsigned long long per_iter = (unsigned long long)adds_per_iter(v.R, block) * per_add;
  unsigned long long it = per_iter ? 0xFFFFFFFFull / per_iter : 1ull << 30;
  if (it < 1) it = 1;
  if (it > (1ull << 30)) it = 1ull << 30;
  return (uint32_t)it;
}

template <int LUTW, int R, bool SPLIT, bool MASS, bool RAW, bool BINS = false, bool PACK = false>
void *kernel_ptr() { return reinterpret_cast<void *>(&k1_trace<LUTW, R, SPLIT, MASS, RAW, BINS, PACK>); }

template <bool RAW>
void *pick_kernel_src(const Variant &v) {
#define FP_K(L)                                                                  \
  if (v.lutw == L) {                                                             \
    if (!v.mass) return v.R == 32 ? kernel_ptr<L, 32, false, false, RAW>() : kernel_ptr<L, 1, false, false, RAW>(); \
    if (v.R == 32) return v.split ? kernel_ptr<L, 32, true, true, RAW>() : kernel_ptr<L, 32, false, true, RAW>();   \
    return v.split ? kernel_ptr<L, 1, true, true, RAW>() : kernel_ptr<L, 1, false, true, RAW>();                    \
  }
  FP_K(0)
  FP_K(1)
  FP_K(2)
#undef FP_K
  return nullptr;
}

// the bin-writing variants exist for the plain LUT paths: u8 LUT (|E| < 256;
// 6-bit packed when |E| < 64) and u16 LUT (clamped bytes, bin_byte)
template <int L, bool PACK>
void *pick_kernel_bins_w(const Variant &v) {
  if (!v.mass)
    return v.R == 32 ? kernel_ptr<L, 32, false, false, false, true, PACK>() : kernel_ptr<L, 1, false, false, false, true, PACK>();
  if (v.R == 32)
    return v.split ? kernel_ptr<L, 32, true, true, false, true, PACK>() : kernel_ptr<L, 32, false, true, false, true, PACK>();
  return v.split ? kernel_ptr<L, 1, true, true, false, true, PACK>() : kernel_ptr<L, 1, false, true, false, true, PACK>();
}

template <bool PACK>
void *pick_kernel_bins(const Variant &v) {
  if (v.raw) {
    // raw columns + byte bins / decision bytes (sweep_and_route_raw's
    // speculative pass): u8 LUT, vector-aligned columns only (raw_vec)
    if (PACK || v.lutw != 1) return nullptr;
    if (!v.mass)
      return v.R == 32 ? kernel_ptr<1, 32, false, false, true, true>() : kernel_ptr<1, 1, false, false, true, true>();
    if (v.R == 32) return v.split ? kernel_ptr<1, 32, true, true, true, true>() : kernel_ptr<1, 32, false, true, true, true>();
    return v.split ? kernel_ptr<1, 1, true, true, true, true>() : kernel_ptr<1, 1, false, true, true, true>();
  }
  if (v.lutw == 1) return pick_kernel_bins_w<1, PACK>(v);
  if (v.lutw == 2 && !PACK) return pick_kernel_bins_w<2, false>(v);
  return nullptr;
}

void *pick_kernel(const Variant &v) {
  if (v.bins) return v.pack ? pick_kernel_bins<true>(v) : pick_kernel_bins<false>(v);
  return v.raw ? pick_kernel_src<true>(v) : pick_kernel_src<false>(v);
}

}  // namespace

size_t trace_smem_bytes(const TraceArgs &a, int block) { return smem_for(a, choose(a, block)); }

int trace_grid(const TraceArgs &a, int grid, int block) {
  const Variant v = choose(a, block);
  if (!(v.raw || v.bins)) return grid;
  void *k = pick_kernel(v);
  const size_t smem = smem_for(a, v);
  if (!k || cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return grid;
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, smem) != cudaSuccess) return grid;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::min(grid, std::max(1, per_sm) * sms);
}

cudaError_t trace_occupancy(const TraceArgs &a, int block, size_t smem, int *per_sm) {
  void *k = pick_kernel(choose(a, block));
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k, block, smem);
}

cudaError_t launch_trace(const TraceArgs &a0, int grid, int block, size_t smem, cudaStream_t s) {
  TraceArgs a = a0;
  const Variant v = choose(a, block);
  a.flush_iters = flush_iters_for(a, v, block);
  // u32 per-block counters: keep every block below 2^31 requests per launch
  const uint64_t cap = (uint64_t)grid * (1ull << 31);
  // the packed bin stream assumes one body per trace (a piece boundary would
  // put a body uint4 into the side bytes); cap is ~1e12 requests anyway
  if (a0.bins_out && a0.bins_pack && a0.n > cap) return cudaErrorInvalidValue;
  void *k = pick_kernel(v);
  if (!k) return cudaErrorInvalidValue;
  if (v.raw || v.bins) {
    // the raw variants carry the c* table: size and opt in per launch
    smem = smem_for(a, v);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // the grid is persistent: never more blocks than are resident at once
    // (the raw variant uses more registers than the plain one)
    int per_sm = 0, dev = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, smem);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = std::min(grid, std::max(1, per_sm) * sms);
  }
  for (uint64_t off = 0; off < a0.n; off += cap) {
    if (a0.len) a.len = a0.len + off;
    if (a0.bins_out && !a0.bins_pack) a.bins_out = a0.bins_out + off;   // (packed: one piece, checked above)
    if (a0.body) {
      a.body = a0.body + off;
      a.maxout = a0.maxout + off;
      a.cat = a0.cat + off;
      const uintptr_t b = reinterpret_cast<uintptr_t>(a.body), m = reinterpret_cast<uintptr_t>(a.maxout),
                      k = reinterpret_cast<uintptr_t>(a.cat);
      const uint64_t mis = (b & 15u) >> 2, head = mis ? 4 - mis : 0;
      // vector loads need the three columns in the same 16-B phase
      a.raw_vec = ((b & 3u) == 0) && ((m & 15u) == (b & 15u)) && (((k + head) & 3u) == 0);
      // the scalar raw rounds write no bins: the bin variant needs vector columns
      if (a.bins_out && !a.raw_vec) return cudaErrorInvalidValue;
    }
    a.n = std::min<uint64_t>(cap, a0.n - off);
    void *args[] = {&a};
    cudaError_t e;
    if (a0.pdl && off == 0 && pdl_enabled()) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(block);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      e = cudaLaunchKernelExC(&cfg, k, args);
    } else {
      e = cudaLaunchKernel(k, dim3(grid), dim3(block), args, smem, s);
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fp
