// K4: route_batch -- Alg. 1 for one (B, C_S, C_L) over a trace.
//
// With 1 <= B <= C_S <= C_L (validated by the host) and a = L > B,
// b = L > C_S, c = L > C_L (c => b => a) the outcome of Alg. 1 is
//   L <= B          -> short, step 2 (budget)        decision 0
//   B < L <= C_S    -> long,  step 2 (budget)        decision 1
//   C_S < L <= C_L  -> long,  step 1 (feasibility)   decision 1 | 1 << 2 = 5
//   L > C_L         -> rejected (R3)      decision 2 | 3 << 2 = 14
// i.e. decision = a + 4 b + 9 c, branch-free. (The final safety check of
// Alg. 1 can only fire after a spillover, which a static trace does not
// have; under B <= C_S its condition is never true.)
//
// Memory pattern: per-block tiles of 128-bit loads (coalesced: lane i reads
// the i-th 16 B of each warp's 512 B), and per uint4 one streaming
// 32-bit store of its 4 decision bytes (a warp stores 128 B contiguous).
// Counts live in registers (short = !a, served = !c), masses are summed per
// step in u32 (16 requests x L <= C_L < 2^28: exact) and then in u64; one
// warp/block reduction and 5 global atomics per block.
#include <algorithm>
#include "internal.cuh"

namespace fp {

namespace {

constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// One request: counters + decision byte, as predicated PTX (3 compares +
// 7 predicated ops; nvcc otherwise emits VIADD + predicated MOV pairs).
__device__ __forceinline__ uint32_t route_u32(uint32_t L, uint32_t B, uint32_t CS, uint32_t CL, uint32_t &ns,
                                              uint32_t &nsv, uint32_t &ms, uint32_t &msv) {
  uint32_t d;
  asm("{\n\t.reg .pred pa, pb, pc;\n\t"
      "setp.gt.u32 pa, %5, %6;\n\t"
      "setp.gt.u32 pb, %5, %7;\n\t"
      "setp.gt.u32 pc, %5, %8;\n\t"
      "selp.u32 %0, 1, 0, pa;\n\t"
      "@pb add.u32 %0, %0, 4;\n\t"
      "@pc add.u32 %0, %0, 9;\n\t"
      "@!pa add.u32 %1, %1, 1;\n\t"
      "@!pa add.u32 %3, %3, %5;\n\t"
      "@!pc add.u32 %2, %2, 1;\n\t"
      "@!pc add.u32 %4, %4, %5;\n\t"
      "}"
      : "=r"(d), "+r"(ns), "+r"(nsv), "+r"(ms), "+r"(msv)
      : "r"(L), "r"(B), "r"(CS), "r"(CL));
  return d;
}

struct Acc {
  uint32_t ns = 0, nsv = 0, n = 0;          // short, served (<= C_L), routed by this thread
  unsigned long long ms = 0, msv = 0;       // mass short, mass served
};

// generic (u64 mass) single request
__device__ __forceinline__ uint32_t route_u64(uint32_t L, uint32_t B, uint32_t CS, uint32_t CL, Acc &a) {
  const bool pa = L > B, pb = L > CS, pc = L > CL;
  if (!pa) { ++a.ns; a.ms += L; }
  if (!pc) { ++a.nsv; a.msv += L; }
  ++a.n;
  return (pa ? 1u : 0u) + (pb ? 4u : 0u) + (pc ? 9u : 0u);
}

template <bool SMALL>
__device__ __forceinline__ uint32_t route4(const uint4 &v, uint32_t B, uint32_t CS, uint32_t CL, Acc &a,
                                           uint32_t &gms, uint32_t &gmsv) {
  if constexpr (SMALL) {
    const uint32_t d0 = route_u32(v.x, B, CS, CL, a.ns, a.nsv, gms, gmsv);
    const uint32_t d1 = route_u32(v.y, B, CS, CL, a.ns, a.nsv, gms, gmsv);
    const uint32_t d2 = route_u32(v.z, B, CS, CL, a.ns, a.nsv, gms, gmsv);
    const uint32_t d3 = route_u32(v.w, B, CS, CL, a.ns, a.nsv, gms, gmsv);
    a.n += 4;
    return d0 | (d1 << 8) | (d2 << 16) | (d3 << 24);
  } else {
    const uint32_t d0 = route_u64(v.x, B, CS, CL, a);
    const uint32_t d1 = route_u64(v.y, B, CS, CL, a);
    const uint32_t d2 = route_u64(v.z, B, CS, CL, a);
    const uint32_t d3 = route_u64(v.w, B, CS, CL, a);
    return d0 | (d1 << 8) | (d2 << 16) | (d3 << 24);
  }
}

template <bool DEC, bool DVEC>
__device__ __forceinline__ void store4(uint8_t *dec, uint32_t w) {
  if constexpr (DEC) {
    if constexpr (DVEC) {
      // streaming store (evict-first): 6.9 vs 6.4 TB/s for this 4:1 mix
      // (profiles/r01_microbench_route_variants.txt)
      asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(dec), "r"(w) : "memory");
    } else {
      dec[0] = (uint8_t)w; dec[1] = (uint8_t)(w >> 8); dec[2] = (uint8_t)(w >> 16); dec[3] = (uint8_t)(w >> 24);
    }
  }
}

// DEC: write decisions; SMALL: C_L < 2^28 (u32 tile masses); DVEC: the
// decision address of every uint4 of the body is 4-byte aligned.
template <bool DEC, bool SMALL, bool DVEC>
__global__ void __launch_bounds__(512, 2) k4_route(RouteArgs a) {
  const uint32_t B = a.b, CS = a.cs, CL = a.cl;
  Acc acc;
  const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(a.len) & 15u) >> 2);
  const uint64_t head = mis ? (a.n < 4u - mis ? a.n : 4u - mis) : 0u;
  const uint64_t n4 = (a.n - head) >> 2;
  const uint64_t tail_first = head + (n4 << 2);
  if (blockIdx.x == 0 && threadIdx.x < head) {
    const uint32_t d = route_u64(a.len[threadIdx.x], B, CS, CL, acc);
    if (DEC) a.decision[threadIdx.x] = (uint8_t)d;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < a.n - tail_first) {
    const uint64_t i = tail_first + threadIdx.x;
    const uint32_t d = route_u64(a.len[i], B, CS, CL, acc);
    if (DEC) a.decision[i] = (uint8_t)d;
  }
  const uint4 *body = reinterpret_cast<const uint4 *>(a.len + head);
  uint8_t *dbody = DEC ? a.decision + head : nullptr;
  // per-block contiguous tiles of blockDim x kUnroll uint4 (for this 4:1
  // read/write mix tiles beat grid-stride stripes: 0.89 vs 0.97 ms on C5,
  // profiles/r01_tune_launch_*.txt)
  const uint64_t tile4 = (uint64_t)blockDim.x * kUnroll;
  const uint64_t full_tiles = n4 / tile4;
  const uint64_t ntiles = (n4 + tile4 - 1) / tile4;
  // software pipeline: the next full tile's loads are in flight while this one
  // is routed (2 x 512 threads per SM at 63 registers: 0.83 -> 0.77 ms on C5)
  uint4 nx[kUnroll];
  if ((uint64_t)blockIdx.x < full_tiles) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) nx[u] = ldg_stream(body + blockIdx.x * tile4 + threadIdx.x + (uint64_t)u * blockDim.x);
  }
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * tile4 + threadIdx.x;
    uint32_t gms = 0, gmsv = 0;
    if (t < full_tiles) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = nx[u];
      const uint64_t tn = t + gridDim.x;
      if (tn < full_tiles) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) nx[u] = ldg_stream(body + tn * tile4 + threadIdx.x + (uint64_t)u * blockDim.x);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint32_t w = route4<SMALL>(v[u], B, CS, CL, acc, gms, gmsv);
        store4<DEC, DVEC>(dbody + 4 * (base + (uint64_t)u * blockDim.x), w);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t i = base + (uint64_t)u * blockDim.x;
        if (i < n4) {
          const uint32_t w = route4<SMALL>(ldg_stream(body + i), B, CS, CL, acc, gms, gmsv);
          store4<DEC, DVEC>(dbody + 4 * i, w);
        }
      }
    }
    if constexpr (SMALL) {
      acc.ms += gms;
      acc.msv += gmsv;
    }
  }
  // reduce: warp shuffles, then one atomic per block per counter
  unsigned long long v[5] = {acc.ns, (unsigned long long)acc.nsv - acc.ns, (unsigned long long)acc.n - acc.nsv,
                             acc.ms, acc.msv - acc.ms};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  __shared__ unsigned long long red[5][16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) red[k][w] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    unsigned long long t = 0;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) t += red[threadIdx.x][j];
    if (t) atomicAdd(a.g_counts + threadIdx.x, t);
  }
}

}  // namespace

// Resident blocks per SM guaranteed for every K4 variant: the grid is
// persistent (tiles are strided over it), so it must not exceed what is
// resident at once -- a second partial wave costs ~20% on C5.
cudaError_t route_occupancy(int block, int *per_sm) {
  void *ks[] = {reinterpret_cast<void *>(&k4_route<true, true, true>),
                reinterpret_cast<void *>(&k4_route<true, true, false>),
                reinterpret_cast<void *>(&k4_route<true, false, true>),
                reinterpret_cast<void *>(&k4_route<true, false, false>),
                reinterpret_cast<void *>(&k4_route<false, true, false>),
                reinterpret_cast<void *>(&k4_route<false, false, false>)};
  int best = 1 << 30;
  for (void *k : ks) {
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, block, 0);
    if (e != cudaSuccess) return e;
    best = std::min(best, n);
  }
  *per_sm = std::max(1, best);
  return cudaSuccess;
}

cudaError_t launch_route(const RouteArgs &a0, int grid, int block, cudaStream_t s) {
  if (a0.n == 0) return cudaSuccess;
  if (block > 512 || (block & 31)) return cudaErrorInvalidValue;
  const bool small = a0.cl < (1u << 28);
  // u32 per-thread counters: at most 2^31 requests per thread per launch
  const uint64_t cap = (uint64_t)grid * block * (1ull << 31);
  RouteArgs a = a0;
  for (uint64_t off = 0; off < a0.n; off += cap) {
    a.len = a0.len + off;
    a.decision = a0.decision ? a0.decision + off : nullptr;
    a.n = std::min<uint64_t>(cap, a0.n - off);
    const uint64_t tiles = (a.n / 4 + (uint64_t)block * kUnroll - 1) / ((uint64_t)block * kUnroll);
    const int g = (int)std::min<uint64_t>((uint64_t)grid, std::max<uint64_t>(1, tiles));
    const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(a.len) & 15u) >> 2);
    const uint64_t head = mis ? std::min<uint64_t>(a.n, 4u - mis) : 0u;
    const bool dvec = a.decision && ((reinterpret_cast<uintptr_t>(a.decision + head) & 3u) == 0u);
#define FP_K4(D, S, V) k4_route<D, S, V><<<g, block, 0, s>>>(a)
    if (a.decision) {
      if (small) { if (dvec) FP_K4(true, true, true); else FP_K4(true, true, false); }
      else { if (dvec) FP_K4(true, false, true); else FP_K4(true, false, false); }
    } else {
      if (small) FP_K4(false, true, false); else FP_K4(false, false, false);
    }
#undef FP_K4
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fp

// ============================ K4r: route_batch_raw ====================================
// NEXT-1: route_batch from the raw columns. Per request the conservative
// ratio c* (Eq. `conservative`; shared-memory table per block)
// gives L_total = ceil(|r| / c*) + max_output (Eq. `budget`, P:425-429;
// estimate.cuh), which is routed as in K4. With the true prompt tokens the
// kernel also counts Table 5's mis-routes: requests sent to a
// pool whose C_max their TRUE total exceeds. Per-block tiles of 4 requests
// per thread (128-bit loads of each u32 column, 32-bit load of 4 category
// bytes, 32-bit store of 4 decisions) when the columns share a 16-B phase;
// scalar grid-stride otherwise.
#include "estimate.cuh"

namespace fp {
namespace {

// Per-thread tallies, all u32 (a thread routes < 2^31 requests; checked at
// launch): ns = #short (L <= B), nsv = #served (L <= C_L), the mis-route
// counts, and per-step partial masses (SMALL: 4 requests x C_L < 2^30 fit a
// u32) folded into u64 once per step. n_long = nsv - ns and n_reject =
// n - nsv are derived at the end (B <= C_S <= C_L: short = !pa).
struct RawAcc {
  uint32_t n = 0, ns = 0, nsv = 0, mis_s = 0, mis_l = 0;
  unsigned long long ms = 0, msv = 0;
};

// One request as predicated PTX: decision a + 4b + 9c, the two counts, the
// two partial masses and (TRUE_TOK) the mis-route counts, where the true
// total t = prompt_tokens + max_output exceeds a window C iff
// mo > C || tp > C - mo (no 64-bit add).
template <bool TRUE_TOK>
__device__ __forceinline__ uint32_t route_raw_u32(uint32_t L, uint32_t mo, uint32_t tp, uint32_t B, uint32_t CS,
                                                  uint32_t CL, RawAcc &c, uint32_t &gms, uint32_t &gmsv) {
  uint32_t d;
  if constexpr (TRUE_TOK) {
    asm("{\n\t.reg .pred pa, pb, pc, qs, ql, ms, ml;\n\t.reg .u32 ts, tl;\n\t"
        "setp.gt.u32 pa, %7, %10;\n\t"
        "setp.gt.u32 pb, %7, %11;\n\t"
        "setp.gt.u32 pc, %7, %12;\n\t"
        "selp.u32 %0, 1, 0, pa;\n\t"
        "@pb add.u32 %0, %0, 4;\n\t"
        "@pc add.u32 %0, %0, 9;\n\t"
        "@!pa add.u32 %1, %1, 1;\n\t"
        "@!pa add.u32 %3, %3, %7;\n\t"
        "@!pc add.u32 %2, %2, 1;\n\t"
        "@!pc add.u32 %4, %4, %7;\n\t"
        "sub.u32 ts, %11, %8;\n\t"
        "sub.u32 tl, %12, %8;\n\t"
        "setp.gt.u32 qs, %8, %11;\n\t"
        "setp.gt.or.u32 qs, %9, ts, qs;\n\t"
        "setp.gt.u32 ql, %8, %12;\n\t"
        "setp.gt.or.u32 ql, %9, tl, ql;\n\t"
        "not.pred ms, pa;\n\t"
        "and.pred ms, ms, qs;\n\t"
        "not.pred ml, pc;\n\t"
        "and.pred ml, ml, pa;\n\t"
        "and.pred ml, ml, ql;\n\t"
        "@ms add.u32 %5, %5, 1;\n\t"
        "@ml add.u32 %6, %6, 1;\n\t"
        "}"
        : "=r"(d), "+r"(c.ns), "+r"(c.nsv), "+r"(gms), "+r"(gmsv), "+r"(c.mis_s), "+r"(c.mis_l)
        : "r"(L), "r"(mo), "r"(tp), "r"(B), "r"(CS), "r"(CL));
  } else {
    asm("{\n\t.reg .pred pa, pb, pc;\n\t"
        "setp.gt.u32 pa, %5, %6;\n\t"
        "setp.gt.u32 pb, %5, %7;\n\t"
        "setp.gt.u32 pc, %5, %8;\n\t"
        "selp.u32 %0, 1, 0, pa;\n\t"
        "@pb add.u32 %0, %0, 4;\n\t"
        "@pc add.u32 %0, %0, 9;\n\t"
        "@!pa add.u32 %1, %1, 1;\n\t"
        "@!pa add.u32 %3, %3, %5;\n\t"
        "@!pc add.u32 %2, %2, 1;\n\t"
        "@!pc add.u32 %4, %4, %5;\n\t"
        "}"
        : "=r"(d), "+r"(c.ns), "+r"(c.nsv), "+r"(gms), "+r"(gmsv)
        : "r"(L), "r"(B), "r"(CS), "r"(CL));
  }
  return d;
}

// generic single request (any C_L: u64 masses)
template <bool TRUE_TOK>
__device__ __forceinline__ uint32_t route_raw_one(uint32_t L, uint32_t mo, uint32_t tp, uint32_t B, uint32_t CS,
                                                  uint32_t CL, RawAcc &c) {
  uint32_t ms = 0, msv = 0;
  const uint32_t d = route_raw_u32<TRUE_TOK>(L, mo, tp, B, CS, CL, c, ms, msv);
  c.ms += ms;
  c.msv += msv;
  ++c.n;
  return d;
}

// VEC: every column in the same 16-B phase; TRUE_TOK: true prompt tokens
// given (mis-routes); DEC / LT: decision / L_total outputs; SMALL: C_L < 2^30.
template <bool VEC, bool TRUE_TOK, bool DEC, bool LT, bool SMALL>
__global__ void __launch_bounds__(512, 2) k4_route_raw(RouteRawArgs a) {
  __shared__ __align__(16) double2 cst[kCatTable];
  __shared__ unsigned long long red[7][16];
  setup_cstar(a.calib, a.n_cats, a.gamma, a.c_floor, cst);
  __syncthreads();
  const uint32_t B = a.b, CS = a.cs, CL = a.cl;
  RawAcc acc;
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t me = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto one = [&](uint64_t i) {
    const uint32_t mo = a.maxout[i];
    const uint32_t L = estimate_l_total(a.body[i], mo, a.cat[i], cst);
    const uint32_t d = route_raw_one<TRUE_TOK>(L, mo, TRUE_TOK ? a.true_prompt[i] : 0u, B, CS, CL, acc);
    if (DEC) a.decision[i] = (uint8_t)d;
    if (LT) a.l_total[i] = L;
  };
  if constexpr (!VEC) {
    for (uint64_t i = me; i < a.n; i += S) one(i);
  } else {
    const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(a.body) & 15u) >> 2);
    const uint64_t head = mis ? (a.n < 4u - mis ? a.n : 4u - mis) : 0u;
    const uint64_t n4 = (a.n - head) >> 2;
    const uint64_t tail_first = head + (n4 << 2);
    if (blockIdx.x == 0 && threadIdx.x < head) one(threadIdx.x);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < a.n - tail_first) one(tail_first + threadIdx.x);
    const uint4 *b4 = reinterpret_cast<const uint4 *>(a.body + head);
    const uint4 *m4 = reinterpret_cast<const uint4 *>(a.maxout + head);
    const uint4 *t4 = TRUE_TOK ? reinterpret_cast<const uint4 *>(a.true_prompt + head) : nullptr;
    const uint32_t *c4 = reinterpret_cast<const uint32_t *>(a.cat + head);
    uint32_t *d4 = DEC ? reinterpret_cast<uint32_t *>(a.decision + head) : nullptr;
    uint4 *l4 = LT ? reinterpret_cast<uint4 *>(a.l_total + head) : nullptr;
    // two quads per thread per iteration, both loaded before either is routed
    // (twice the bytes in flight; the second may be past the end)
    for (uint64_t i0 = me; i0 < n4; i0 += 2 * S) {
      const bool has2 = i0 + S < n4;
      const uint64_t i1 = has2 ? i0 + S : i0;
      const uint4 b0 = ldg_stream(b4 + i0), m0 = ldg_stream(m4 + i0);
      const uint4 t0 = TRUE_TOK ? ldg_stream(t4 + i0) : make_uint4(0u, 0u, 0u, 0u);
      const uint32_t k0 = __ldg(c4 + i0);
      const uint4 b1 = ldg_stream(b4 + i1), m1 = ldg_stream(m4 + i1);
      const uint4 t1 = TRUE_TOK ? ldg_stream(t4 + i1) : make_uint4(0u, 0u, 0u, 0u);
      const uint32_t k1 = __ldg(c4 + i1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
      if (h == 1 && !has2) break;
      const uint64_t i = h ? i1 : i0;
      const uint4 b = h ? b1 : b0, m = h ? m1 : m0;
      const uint4 t = h ? t1 : t0;
      const uint32_t k = h ? k1 : k0;
      const uint4 L = make_uint4(estimate_l_total(b.x, m.x, k & 0xFFu, cst),
                                 estimate_l_total(b.y, m.y, (k >> 8) & 0xFFu, cst),
                                 estimate_l_total(b.z, m.z, (k >> 16) & 0xFFu, cst),
                                 estimate_l_total(b.w, m.w, k >> 24, cst));
      uint32_t w;
      if constexpr (SMALL) {
        uint32_t gms = 0, gmsv = 0;
        w = route_raw_u32<TRUE_TOK>(L.x, m.x, t.x, B, CS, CL, acc, gms, gmsv) |
            (route_raw_u32<TRUE_TOK>(L.y, m.y, t.y, B, CS, CL, acc, gms, gmsv) << 8) |
            (route_raw_u32<TRUE_TOK>(L.z, m.z, t.z, B, CS, CL, acc, gms, gmsv) << 16) |
            (route_raw_u32<TRUE_TOK>(L.w, m.w, t.w, B, CS, CL, acc, gms, gmsv) << 24);
        acc.ms += gms;
        acc.msv += gmsv;
        acc.n += 4;
      } else {
        w = route_raw_one<TRUE_TOK>(L.x, m.x, t.x, B, CS, CL, acc) |
            (route_raw_one<TRUE_TOK>(L.y, m.y, t.y, B, CS, CL, acc) << 8) |
            (route_raw_one<TRUE_TOK>(L.z, m.z, t.z, B, CS, CL, acc) << 16) |
            (route_raw_one<TRUE_TOK>(L.w, m.w, t.w, B, CS, CL, acc) << 24);
      }
      if (DEC) asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(d4 + i), "r"(w) : "memory");
      if (LT) l4[i] = L;
      }
    }
  }
  // counts: short, long, rejected, mass short, mass long, mis-routes short, long
  unsigned long long v[7] = {acc.ns, (unsigned long long)acc.nsv - acc.ns, (unsigned long long)acc.n - acc.nsv,
                             acc.ms, acc.msv - acc.ms, acc.mis_s, acc.mis_l};
#pragma unroll
  for (int k = 0; k < 7; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 7; ++k) red[k][w] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    unsigned long long t = 0;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) t += red[threadIdx.x][j];
    if (t) atomicAdd(threadIdx.x < 5 ? a.g_counts + threadIdx.x : a.g_mis + (threadIdx.x - 5), t);
  }
}

template <bool VEC, bool TRUE_TOK, bool DEC, bool LT>
void *k4r_ptr(bool small) {
  return small ? reinterpret_cast<void *>(&k4_route_raw<VEC, TRUE_TOK, DEC, LT, true>)
               : reinterpret_cast<void *>(&k4_route_raw<VEC, TRUE_TOK, DEC, LT, false>);
}

template <bool VEC>
void *k4r_pick(const RouteRawArgs &a) {
  const bool small = a.cl < (1u << 30);
  const int sel = (a.true_prompt ? 4 : 0) | (a.decision ? 2 : 0) | (a.l_total ? 1 : 0);
  switch (sel) {
    case 0: return k4r_ptr<VEC, false, false, false>(small);
    case 1: return k4r_ptr<VEC, false, false, true>(small);
    case 2: return k4r_ptr<VEC, false, true, false>(small);
    case 3: return k4r_ptr<VEC, false, true, true>(small);
    case 4: return k4r_ptr<VEC, true, false, false>(small);
    case 5: return k4r_ptr<VEC, true, false, true>(small);
    case 6: return k4r_ptr<VEC, true, true, false>(small);
    default: return k4r_ptr<VEC, true, true, true>(small);
  }
}

}  // namespace

cudaError_t launch_route_raw(const RouteRawArgs &a, int grid, int block, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  if (block > 512 || (block & 31) || a.n_cats == 0 || a.n_cats > 256) return cudaErrorInvalidValue;
  // vector path: every column in the same 16-B phase (cat / decision in the same 4-B phase)
  const uintptr_t b = reinterpret_cast<uintptr_t>(a.body);
  const uint64_t mis = (b & 15u) >> 2, head = mis ? 4 - mis : 0;
  auto same16 = [&](const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == (b & 15u); };
  auto al4 = [&](const void *p) { return p == nullptr || ((reinterpret_cast<uintptr_t>(p) + head) & 3u) == 0; };
  const bool vec = (b & 3u) == 0 && same16(a.maxout) && same16(a.true_prompt) && same16(a.l_total) && al4(a.cat) &&
                   al4(a.decision);
  void *k = vec ? k4r_pick<true>(a) : k4r_pick<false>(a);
  // grid-stride over a persistent grid: never more blocks than are resident
  // at once (a partial second wave leaves most SMs idle at the end)
  int per_sm = 0, dev = 0, sms = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, 0);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t need = (a.n + block - 1) / block;
  const int g = (int)std::min<uint64_t>((uint64_t)std::min(grid, std::max(1, per_sm) * sms),
                                        std::max<uint64_t>(1, need));
  if (a.n / ((uint64_t)g * block) >= (1ull << 31)) return cudaErrorInvalidValue;   // u32 per-thread tallies
  RouteRawArgs arg = a;
  void *args[] = {&arg};
  e = cudaLaunchKernel(k, dim3(g), dim3(block), args, 0, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace fp

// ============================ K4b: route from bins =====================================
// sweep_and_route's second pass: the trace pass already wrote each request's
// bin b = #{e in E : e < L} (1 B), and E contains B, C_S and C_L, so every
// comparison of Alg. 1 is a bin comparison: L > e_j <=> b > j. Reads 1 B and
// writes 1 B per request (16 per thread with 128-bit loads/stores when the two
// buffers share a 16-B phase). The pool counts and masses of the split are
// the best candidate's record (the same histogram), so no reduction here.
namespace fp {
namespace {

// A split {iB, iCS, iCL, ok} written by the predecessor kernel (K3 / the pick
// kernel), read after griddepcontrol.wait. A programmatic dependent starts
// while its predecessor still runs, so this must be a coherent load that the
// compiler cannot hoist above the wait: a const __restrict__ (ld.global.nc,
// "invariant") load was moved above it and read a stale split
// (test_raw_step_forced_miss caught it once K3 triggered its dependents early).
__device__ __forceinline__ uint4 ld_split(const uint32_t *p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)
               : "memory");
  return r;
}

__device__ __forceinline__ uint32_t dec_byte(uint32_t b, uint32_t iB, uint32_t iCS, uint32_t iCL) {
  return (b > iB ? 1u : 0u) + (b > iCS ? 4u : 0u) + (b > iCL ? 9u : 0u);
}

// Four packed bins -> four decision bytes. SWAR when every bin < 128: adding
// 0x7F - j to a byte sets its top bit iff the byte is > j (no carry out of
// any byte), so a word compare costs one add and one and.
struct SwarK {
  uint32_t kB, kCS, kCL;   // (0x7F - j) replicated in every byte
};

__device__ __forceinline__ uint32_t dec_word_swar(uint32_t w, const SwarK &k) {
  const uint32_t gB = (w + k.kB) & 0x80808080u;
  const uint32_t gS = (w + k.kCS) & 0x80808080u;
  const uint32_t gL = (w + k.kCL) & 0x80808080u;
  return (gB >> 7) + (gS >> 5) + (gL >> 7) * 9u;     // a + 4 b + 9 c per byte
}

// SWAR for full bytes (bins up to 255): b > j <=> b >= y, y = j + 1 <= 255.
// d = (b | 0x80) - (y & 0x7F) per byte never borrows across bytes, and its top
// bit is [b & 0x7F >= y & 0x7F]; then b >= y is (b7 | d7) when y < 128 and
// (b7 & d7) when y >= 128: ((b & d) | ((b | d) & o)) & 0x80 with o = 0x80 or 0.
// j >= 255 (only with the routing pass's escapes, which rewrite byte 255) is
// taken as j = 254.
struct SwarU {
  uint32_t ylow[3], o[3];
};

__device__ __forceinline__ SwarU swar_u(uint32_t iB, uint32_t iCS, uint32_t iCL) {
  SwarU k;
  const uint32_t j[3] = {iB, iCS, iCL};
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const uint32_t y = (j[t] < 254u ? j[t] : 254u) + 1u;
    k.ylow[t] = (y & 0x7Fu) * 0x01010101u;
    k.o[t] = y < 128u ? 0x80808080u : 0u;
  }
  return k;
}

__device__ __forceinline__ uint32_t dec_word_u8(uint32_t w, const SwarU &k) {
  uint32_t g[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const uint32_t d = (w | 0x80808080u) - k.ylow[t];
    g[t] = (((w & d) | ((w | d) & k.o[t])) >> 7) & 0x01010101u;
  }
  return g[0] + g[1] * 4u + g[2] * 9u;                // a + 4 b + 9 c per byte
}

// The split to route with, picked on the device so that the step needs no
// host round trip between the sweep and the routing pass: per-model argmin
// over the ranks' best records (feasible, min cost, ties to the lowest index:
// fp_merge_best's rule), then the edge indices of its B, C_S, C_L
// (#{e in E : e < v}, one ballot per 32 edges). out = {iB, iCS, iCL, ok}.
__global__ void k_pick_route(const fp_candidate *recs, int ranks, uint32_t n_models, uint32_t m,
                             const uint32_t *edges, uint32_t n_edges, uint32_t *out) {
  const int lane = threadIdx.x;
  bool ok = false;
  double cost = 0.0;
  uint32_t idx = 0xffffffffu;
  int who = lane;
  if (lane < ranks) {
    const fp_candidate &c = recs[(size_t)lane * n_models + m];
    ok = (c.flags & FP_CAND_FEASIBLE) != 0;
    cost = c.cost_dual;
    idx = c.index;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const bool ok2 = __shfl_down_sync(0xffffffffu, ok, o);
    const double cost2 = __shfl_down_sync(0xffffffffu, cost, o);
    const uint32_t idx2 = __shfl_down_sync(0xffffffffu, idx, o);
    const int who2 = __shfl_down_sync(0xffffffffu, who, o);
    if (lane + o < 32 && ok2 && (!ok || cost2 < cost || (cost2 == cost && idx2 < idx))) {
      ok = true; cost = cost2; idx = idx2; who = who2;
    }
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  who = __shfl_sync(0xffffffffu, who, 0);
  if (!ok) {
    if (lane == 0) out[3] = 0u;
    return;
  }
  const fp_candidate &c = recs[(size_t)who * n_models + m];
  const uint32_t vb = c.b_short, vs = c.c_short, vl = c.c_long;
  uint32_t nb = 0, ns = 0, nl = 0;
  for (uint32_t base = 0; base < n_edges; base += 32) {
    const uint32_t e = base + lane < n_edges ? edges[base + lane] : 0xffffffffu;
    nb += __popc(__ballot_sync(0xffffffffu, e < vb));
    ns += __popc(__ballot_sync(0xffffffffu, e < vs));
    nl += __popc(__ballot_sync(0xffffffffu, e < vl));
  }
  if (lane == 0) { out[0] = nb; out[1] = ns; out[2] = nl; out[3] = 1u; }
}

// Clamped bytes (|E| >= 255, k1_trace bin_byte): byte 255 = "bin >= 255". When
// every edge index of the split is < 255 that byte is above all three and the
// decision needs nothing else; otherwise (esc) such requests read L_total back
// from the trace and compare it with the split's edge values: a stand-in bin
// with the same order relations to iB <= iCS <= iCL (rare: L above the 255th
// edge).
__device__ __forceinline__ uint32_t escape_bin(uint32_t L, uint32_t iB, uint32_t iCS, uint32_t iCL,
                                               const uint32_t *edges) {
  uint32_t fb = 0;
  if (L > __ldg(edges + iB)) fb = iB + 1;
  if (L > __ldg(edges + iCS)) fb = iCS + 1;
  if (L > __ldg(edges + iCL)) fb = iCL + 1;
  return fb;
}

// byte 0xFF in any lane of w
__device__ __forceinline__ bool has_ff(uint32_t w) { return ((~w - 0x01010101u) & w & 0x80808080u) != 0u; }

// the decisions of the 0xFF bytes of v (requests len[0..16)) from L_total
__device__ __noinline__ uint4 fix_escapes(uint4 v, uint4 o, const uint32_t *len, uint32_t iB, uint32_t iCS,
                                          uint32_t iCL, const uint32_t *edges) {
  uint32_t *ow = &o.x;
  const uint32_t *vw = &v.x;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (((vw[k] >> (8 * e)) & 0xFFu) == 0xFFu) {
        const uint32_t d = dec_byte(escape_bin(__ldg(len + 4 * k + e), iB, iCS, iCL, edges), iB, iCS, iCL);
        ow[k] = (ow[k] & ~(0xFFu << (8 * e))) | (d << (8 * e));
      }
  return o;
}

template <bool VEC, bool SWAR>
__global__ void __launch_bounds__(512) k4_route_bins(const uint8_t *__restrict__ bins, uint8_t *__restrict__ dec,
                                                      uint64_t n, const uint32_t *route,
                                                      const uint32_t *__restrict__ len, const uint32_t *__restrict__ edges) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // K3's split (PDL launch)
  const uint4 rt = ld_split(route);
  if (!rt.w) return;                        // no feasible split: nothing to route (the host reports it)
  const uint32_t iB = rt.x, iCS = rt.y, iCL = rt.z;
  const bool esc = len && iCL >= 255u;      // iB <= iCS <= iCL
  // the decision of request i from its byte b
  auto one = [&](uint64_t i, uint32_t b) {
    return dec_byte(esc && b == 255u ? escape_bin(__ldg(len + i), iB, iCS, iCL, edges) : b, iB, iCS, iCL);
  };
  const SwarK sk{(0x7Fu - (iB < 0x7Fu ? iB : 0x7Fu)) * 0x01010101u, (0x7Fu - (iCS < 0x7Fu ? iCS : 0x7Fu)) * 0x01010101u,
                 (0x7Fu - (iCL < 0x7Fu ? iCL : 0x7Fu)) * 0x01010101u};
  const SwarU su = swar_u(iB, iCS, iCL);
  auto word = [&](uint32_t w) { return SWAR ? dec_word_swar(w, sk) : dec_word_u8(w, su); };
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t me = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (!VEC) {
    for (uint64_t i = me; i < n; i += S) dec[i] = (uint8_t)one(i, bins[i]);
  } else {
    const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(bins) & 15u);
    const uint64_t head = mis ? (n < 16u - mis ? n : 16u - mis) : 0u;
    const uint64_t n16 = (n - head) >> 4;
    const uint64_t tail_first = head + (n16 << 4);
    if (blockIdx.x == 0 && threadIdx.x < head) dec[threadIdx.x] = (uint8_t)one(threadIdx.x, bins[threadIdx.x]);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - tail_first) {
      const uint64_t i = tail_first + threadIdx.x;
      dec[i] = (uint8_t)one(i, bins[i]);
    }
    const uint4 *b16 = reinterpret_cast<const uint4 *>(bins + head);
    uint4 *d16 = reinterpret_cast<uint4 *>(dec + head);
    // 16 decisions from 16 bytes; the rare escapes (esc only, warp-uniform)
    // out of line so the streaming loop keeps its registers
    auto sixteen = [&](uint64_t q, const uint4 &v) {
      uint4 o = make_uint4(word(v.x), word(v.y), word(v.z), word(v.w));
      if (esc && (has_ff(v.x) | has_ff(v.y) | has_ff(v.z) | has_ff(v.w)))
        o = fix_escapes(v, o, len + head + 16 * q, iB, iCS, iCL, edges);
      return o;
    };
    // KQ quads in flight per thread (small traces are latency-bound: a 1e8-
    // request pass needs ~10 MB in flight to reach the copy rate)
    constexpr int KQ = 4;
    for (uint64_t i = me; i < n16; i += KQ * S) {
      uint4 v[KQ];
#pragma unroll
      for (int k = 0; k < KQ; ++k) v[k] = i + k * S < n16 ? ldg_stream(b16 + i + k * S) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int k = 0; k < KQ; ++k) {
        if (i + k * S < n16) {
          const uint4 o = sixteen(i + k * S, v[k]);
          asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d16 + i + k * S), "r"(o.x), "r"(o.y),
                       "r"(o.z), "r"(o.w)
                       : "memory");
        }
      }
    }
  }
}

// The 6-bit packed bins of K1 (|E| < 64; TraceArgs::bins_pack): chunk
// c = k S + t holds the bins of the trace pass's step k, thread t -- uint4
// j = 4 k S + u S + t, u < 4 -- as a u64 of low nibbles and a u32 of high
// 2-bit parts, so the step moves 0.75 B of bins per request each way instead
// of 1 B. Launched with the trace pass's own grid x block: thread t reads its
// chunks with one 8-B and one 4-B coalesced load per 16 requests and writes
// 4 decision words (each warp store 128 B contiguous).

template <bool VEC>
__global__ void __launch_bounds__(512) k4_route_packed(const unsigned long long *__restrict__ lo,
                                                       const uint32_t *__restrict__ hi,
                                                       const uint8_t *__restrict__ side, uint8_t *__restrict__ dec,
                                                       uint64_t n, uint32_t head, const uint32_t *route) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // K3's split (PDL launch)
  const uint4 rt = ld_split(route);
  if (!rt.w) return;                        // no feasible split: nothing to route (the host reports it)
  const uint32_t iB = rt.x, iCS = rt.y, iCL = rt.z;
  const SwarK sk{(0x7Fu - (iB < 0x7Fu ? iB : 0x7Fu)) * 0x01010101u, (0x7Fu - (iCS < 0x7Fu ? iCS : 0x7Fu)) * 0x01010101u,
                 (0x7Fu - (iCL < 0x7Fu ? iCL : 0x7Fu)) * 0x01010101u};
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t h = head < n ? head : n;
  const uint64_t n4 = (n - h) >> 2;
  const uint64_t tail_first = h + (n4 << 2);
  if (blockIdx.x == 0 && threadIdx.x < h) dec[threadIdx.x] = (uint8_t)dec_byte(side[threadIdx.x], iB, iCS, iCL);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < n - tail_first)
    dec[tail_first + threadIdx.x] = (uint8_t)dec_byte(side[4 + threadIdx.x], iB, iCS, iCL);
  uint8_t *body = dec + h;
  const uint64_t nsteps = (n4 + 4 * S - 1) / (4 * S);
  const uint64_t full = n4 / (4 * S);             // steps whose 4 uint4 all exist
  auto put = [&](uint8_t *q, uint32_t d) {
    if (VEC) {
      asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(q), "r"(d) : "memory");
    } else {
      q[0] = (uint8_t)d; q[1] = (uint8_t)(d >> 8); q[2] = (uint8_t)(d >> 16); q[3] = (uint8_t)(d >> 24);
    }
  };
  // K1's pack_step layout: bins (u, e) -> byte e of word u, low nibble from the
  // u-th nibble lane of lo, high 2 bits from bits 2u of byte e of hi
  auto word = [&](unsigned long long l, uint32_t c, int u) {
    const uint32_t half = (uint32_t)(l >> (32 * (u >> 1)));
    const uint32_t n = (half >> (4 * (u & 1))) & 0x0F0F0F0Fu;
    const uint32_t h = (u == 3 ? (c >> 2) : (c << (4 - 2 * u))) & 0x30303030u;
    return dec_word_swar(n | h, sk);
  };
  const uint64_t ustride = 4 * S;                 // bytes between a chunk's uint4 u and u + 1
  // full steps: four steps' chunks in flight per thread (48 B of loads), no bounds checks
  constexpr int KU = 4;
  uint64_t k = 0;
  for (; k + KU <= full; k += KU) {
    unsigned long long l[KU];
    uint32_t c[KU];
#pragma unroll
    for (int q = 0; q < KU; ++q) {
      l[q] = __ldcs(lo + (k + q) * S + t);
      c[q] = __ldcs(hi + (k + q) * S + t);
    }
#pragma unroll
    for (int q = 0; q < KU; ++q) {
      uint8_t *d = body + 16 * S * (k + q) + 4 * t;
#pragma unroll
      for (int u = 0; u < 4; ++u) put(d + u * ustride, word(l[q], c[q], u));
    }
  }
  // the remaining steps (the last one partial)
  for (; k < nsteps; ++k) {
    const unsigned long long l = __ldcs(lo + k * S + t);
    const uint32_t c = __ldcs(hi + k * S + t);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t j = 4 * k * S + u * S + t;
      if (j < n4) put(body + 4 * j, word(l, c, u));
    }
  }
}

// FP_FLAG_SPECULATE verify / fix-up: nothing to do when the speculated split
// is the final one (the trace pass already wrote its decisions); otherwise
// every request is re-routed from L_total with the final split (escape_bin's
// stand-in bin has the same order relations to iB <= iCS <= iCL as the bin).
__global__ void __launch_bounds__(512) k4_route_verify(const uint32_t *__restrict__ len, uint8_t *__restrict__ dec,
                                                       uint64_t n, const uint32_t *spec,
                                                       const uint32_t *route,
                                                       const uint32_t *__restrict__ edges, unsigned int *misses) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the full K3's split (PDL launch)
  const uint4 rt = ld_split(route);
  const uint4 sp = ld_split(spec);
  if (!rt.w) return;                           // no feasible split: decisions unspecified (header)
  if (sp.w && sp.x == rt.x && sp.y == rt.y && sp.z == rt.z) return;
  if (blockIdx.x == 0 && threadIdx.x == 0 && misses) atomicAdd(misses, 1u);
  const uint32_t iB = rt.x, iCS = rt.y, iCL = rt.z;
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += S)
    dec[i] = (uint8_t)dec_byte(escape_bin(__ldg(len + i), iB, iCS, iCL, edges), iB, iCS, iCL);
}

// FP_FLAG_SPECULATE, raw columns (sweep_and_route_raw): the same check; a
// miss re-routes every request from its estimated L_total (Eq. `budget`
// with the plan's conservative ratios, estimate.cuh -- the trace pass's value)
__global__ void __launch_bounds__(512) k4_route_verify_raw(RouteRawArgs a, const uint32_t *spec,
                                                           const uint32_t *route,
                                                           const uint32_t *__restrict__ edges, unsigned int *misses) {
  __shared__ double2 cst[kCatTable];
  setup_cstar(a.calib, a.n_cats, a.gamma, a.c_floor, cst);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the full K3's split (PDL launch)
  const uint4 rt = ld_split(route);
  const uint4 sp = ld_split(spec);
  if (!rt.w) return;
  if (sp.w && sp.x == rt.x && sp.y == rt.y && sp.z == rt.z) return;
  if (blockIdx.x == 0 && threadIdx.x == 0 && misses) atomicAdd(misses, 1u);
  const uint32_t iB = rt.x, iCS = rt.y, iCL = rt.z;
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += S) {
    const uint32_t L = estimate_l_total(__ldg(a.body + i), __ldg(a.maxout + i), a.cat[i], cst);
    a.decision[i] = (uint8_t)dec_byte(escape_bin(L, iB, iCS, iCL, edges), iB, iCS, iCL);
  }
}

}  // namespace

cudaError_t launch_route_verify_raw(const RouteRawArgs &a, const uint32_t *spec, const uint32_t *route,
                                    const uint32_t *edges, unsigned int *misses, int grid, int block, cudaStream_t s) {
  return launch_pdl(k4_route_verify_raw, dim3(grid), dim3(block), 0, s, a, spec, route, edges, misses);
}

cudaError_t launch_pick_route(const fp_candidate *recs, int ranks, uint32_t n_models, uint32_t model,
                              const uint32_t *edges, uint32_t n_edges, uint32_t *route, cudaStream_t s) {
  k_pick_route<<<1, 32, 0, s>>>(recs, ranks, n_models, model, edges, n_edges, route);
  return cudaGetLastError();
}

cudaError_t launch_route_verify(const uint32_t *len, uint8_t *decision, uint64_t n, const uint32_t *spec,
                                const uint32_t *route, const uint32_t *edges, unsigned int *misses, int grid,
                                int block, cudaStream_t s) {
  return launch_pdl(k4_route_verify, dim3(grid), dim3(block), 0, s, len, decision, n, spec, route, edges, misses);
}

cudaError_t launch_route_packed(const uint8_t *lo, const uint8_t *hi, const uint8_t *side, uint32_t head,
                                uint8_t *decision, uint64_t n, const fp_candidate *recs, int ranks, uint32_t n_models,
                                uint32_t model, const uint32_t *edges, uint32_t n_edges, uint32_t *route, int k1_grid,
                                int k1_block, cudaStream_t s) {
  if (recs) k_pick_route<<<1, 32, 0, s>>>(recs, ranks, n_models, model, edges, n_edges, route);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || n == 0) return e;
  const uint64_t h = head < n ? head : n;
  const bool vec = (reinterpret_cast<uintptr_t>(decision + h) & 3u) == 0;
  const auto *l8 = reinterpret_cast<const unsigned long long *>(lo);
  const auto *h4 = reinterpret_cast<const uint32_t *>(hi);
  return vec ? launch_pdl(k4_route_packed<true>, dim3(k1_grid), dim3(k1_block), 0, s, l8, h4, side, decision, n, head,
                          (const uint32_t *)route)
             : launch_pdl(k4_route_packed<false>, dim3(k1_grid), dim3(k1_block), 0, s, l8, h4, side, decision, n, head,
                          (const uint32_t *)route);
}

cudaError_t launch_route_bins(const uint8_t *bins, uint8_t *decision, uint64_t n, const fp_candidate *recs,
                              int ranks, uint32_t n_models, uint32_t model, const uint32_t *edges, uint32_t n_edges,
                              uint32_t *route, int grid, int block, cudaStream_t s, const uint32_t *len) {
  // recs == NULL: K3 already wrote route (one rank's grid is the whole grid)
  if (recs) k_pick_route<<<1, 32, 0, s>>>(recs, ranks, n_models, model, edges, n_edges, route);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || n == 0) return e;
  const bool vec = ((reinterpret_cast<uintptr_t>(bins) ^ reinterpret_cast<uintptr_t>(decision)) & 15u) == 0;
  const uint64_t need = (n / (vec ? 16 : 1) + block - 1) / block;
  const int g = (int)std::min<uint64_t>((uint64_t)grid, std::max<uint64_t>(1, need));
  // SWAR needs every bin < 128: bins go up to |E|, and j = iB, iCS, iCL < |E|
  const bool swar = n_edges < 128;
  const uint32_t *rt = route;
  // clamped bytes (n_edges >= 255): escapes may read the trace (len, device)
  const uint32_t *lv = n_edges >= 255 ? len : nullptr;
  if (vec && swar) return launch_pdl(k4_route_bins<true, true>, dim3(g), dim3(block), 0, s, bins, decision, n, rt, lv, edges);
  if (vec) return launch_pdl(k4_route_bins<true, false>, dim3(g), dim3(block), 0, s, bins, decision, n, rt, lv, edges);
  return launch_pdl(k4_route_bins<false, false>, dim3(g), dim3(block), 0, s, bins, decision, n, rt, lv, edges);
}

}  // namespace fp
