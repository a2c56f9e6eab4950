// K1: the trace pass of sweep_thresholds, and K4: route_batch.
//
// K1 streams the u32 L_total column once (128-bit loads, one contiguous
// 32 KB tile per block per step, several tiles in flight per SM) and routes
// every request against EVERY candidate at once: its bin
//     b(L) = #{e in E : e < L}          (E = sortuniq(B u C_L), "<=")
// is read from a fine-cell LUT in shared memory (cell = ceil(L / 2^s); every
// edge is a multiple of 2^s, so the LUT is exact), and the request adds 1 to
// cnt[b] and L to mass[b]. A request in bin b is short for every candidate
// with B >= e_b, long for B < L <= C_L and rejected for L > C_L, so the scan
// of this histogram (K3 prologue) gives every candidate's routing outcome of
// Alg. 1 with bit-exact integer counts.
//
// Histogram layout: R replicas x (|E|+1) bins of u32 counters in shared
// memory; with R = 32 every lane owns a replica ("lane-private"), so the 32
// atomics of one warp instruction hit 32 distinct banks whatever the length
// distribution (no same-address serialisation on skewed traces). Mass uses
// u32 slots flushed into a u64 per-bin accumulator before they can overflow
// (64-bit shared atomics are a CAS loop on sm_100a: ATOMS.CAST.SPIN.64).
// When L can exceed the u32 flush bound the mass is split into 16-bit halves.
#include <algorithm>
#include <cstdio>
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

// bin = #{e in E : e < L}
template <int LUTW>
__device__ __forceinline__ uint32_t bin_of(uint32_t L, const unsigned char *lut, const uint32_t *edges,
                                           uint32_t shift, uint32_t cell_last, uint32_t n_edges) {
  if (LUTW == 1 || LUTW == 2) {
    uint32_t cell = (L >> shift) + ((L & ((1u << shift) - 1u)) != 0u);   // ceil(L / 2^s), no overflow
    cell = min(cell, cell_last);
    return LUTW == 1 ? (uint32_t)lut[cell] : (uint32_t)reinterpret_cast<const uint16_t *>(lut)[cell];
  } else {
    // binary search (large or irregular edge sets): lower_bound of L in E
    uint32_t lo = 0, n = n_edges;
    while (n > 0) {
      uint32_t half = n >> 1;
      if (edges[lo + half] < L) { lo += half + 1; n -= half + 1; } else { n = half; }
    }
    return lo;
  }
}

struct K1Smem {
  unsigned char *lut;     // LUT bytes (or edges in binary-search mode)
  uint32_t *cnt;          // [nbins * R]
  uint32_t *m_lo;         // [nbins * R]
  uint32_t *m_hi;         // [nbins * R] (split mode)
  unsigned long long *acc;  // [nbins] u64 mass accumulator
};

template <int R, bool SPLIT>
__device__ __forceinline__ void flush_mass(const K1Smem &s, uint32_t nbins) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (R == 32) {
    for (uint32_t j = warp; j < nbins; j += nw) {
      unsigned long long v = s.m_lo[j * 32 + lane];
      if (SPLIT) v += (unsigned long long)s.m_hi[j * 32 + lane] << 16;
      s.m_lo[j * 32 + lane] = 0;
      if (SPLIT) s.m_hi[j * 32 + lane] = 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) s.acc[j] += v;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < nbins; j += blockDim.x) {
      unsigned long long v = s.m_lo[j];
      if (SPLIT) v += (unsigned long long)s.m_hi[j] << 16;
      s.m_lo[j] = 0;
      if (SPLIT) s.m_hi[j] = 0;
      s.acc[j] += v;
    }
  }
}

template <int LUTW, int R, bool SPLIT, bool MASS>
__device__ __forceinline__ void add_one(const K1Smem &s, uint32_t L, uint32_t lane, uint32_t shift,
                                        uint32_t cell_last, uint32_t n_edges, const uint32_t *edges) {
  const uint32_t b = bin_of<LUTW>(L, s.lut, edges, shift, cell_last, n_edges);
  const uint32_t slot = (R == 32) ? b * 32 + lane : b;
  atomicAdd(&s.cnt[slot], 1u);
  if (MASS && b < n_edges) {     // mass above the last edge is never used
    if (SPLIT) {
      atomicAdd(&s.m_lo[slot], L & 0xFFFFu);
      atomicAdd(&s.m_hi[slot], L >> 16);
    } else {
      atomicAdd(&s.m_lo[slot], L);
    }
  }
}

template <int LUTW, int R, bool SPLIT, bool MASS>
__global__ void __launch_bounds__(512) k1_trace(TraceArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t nbins = a.n_edges + 1;
  K1Smem s;
  uint32_t lut_bytes;
  if (LUTW == 0) lut_bytes = a.n_edges * 4;
  else lut_bytes = a.lut_cells * LUTW;
  lut_bytes = (lut_bytes + 15u) & ~15u;
  s.lut = smem;
  s.acc = reinterpret_cast<unsigned long long *>(smem + lut_bytes);
  s.cnt = reinterpret_cast<uint32_t *>(s.acc + nbins);
  s.m_lo = s.cnt + nbins * R;
  s.m_hi = s.m_lo + nbins * R;

  // stage the LUT (or the edge list) and clear the histogram
  {
    const uint32_t *src = (LUTW == 0) ? a.edges : reinterpret_cast<const uint32_t *>(a.lut);
    uint32_t *dst = reinterpret_cast<uint32_t *>(s.lut);
    for (uint32_t i = threadIdx.x; i < lut_bytes / 4; i += blockDim.x) {
      // the device LUT allocation is padded to 16 B inside the table blob
      dst[i] = src[i];
    }
    for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) s.acc[i] = 0ull;
    const uint32_t words = nbins * R * (MASS ? (SPLIT ? 3u : 2u) : 1u);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) s.cnt[i] = 0u;
  }
  __syncthreads();
  const uint32_t *edges = reinterpret_cast<const uint32_t *>(s.lut);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t shift = a.shift, cell_last = a.lut_cells ? a.lut_cells - 1 : 0, ne = a.n_edges;

  // misaligned head (< 4 elements) and the aligned uint4 body
  const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(a.len) & 15u) >> 2);
  const uint64_t head = mis ? umin64(a.n, 4u - mis) : 0u;
  const uint64_t n4 = (a.n - head) >> 2;                       // uint4 count of the body
  const uint64_t tail_first = head + (n4 << 2);
  if (blockIdx.x == 0 && threadIdx.x < head)
    add_one<LUTW, R, SPLIT, MASS>(s, a.len[threadIdx.x], lane, shift, cell_last, ne, edges);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < a.n - tail_first)
    add_one<LUTW, R, SPLIT, MASS>(s, a.len[tail_first + threadIdx.x], lane, shift, cell_last, ne, edges);

  const uint4 *body = reinterpret_cast<const uint4 *>(a.len + head);
  const uint64_t tile4 = (uint64_t)blockDim.x * kUnroll;     // uint4 per tile
  const uint64_t ntiles = (n4 + tile4 - 1) / tile4;
  uint32_t since_flush = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * tile4 + threadIdx.x;
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x;
      v[u] = i < n4 ? ldg_stream(body + i) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + (uint64_t)u * blockDim.x < n4) {
        add_one<LUTW, R, SPLIT, MASS>(s, v[u].x, lane, shift, cell_last, ne, edges);
        add_one<LUTW, R, SPLIT, MASS>(s, v[u].y, lane, shift, cell_last, ne, edges);
        add_one<LUTW, R, SPLIT, MASS>(s, v[u].z, lane, shift, cell_last, ne, edges);
        add_one<LUTW, R, SPLIT, MASS>(s, v[u].w, lane, shift, cell_last, ne, edges);
      }
    }
    if (MASS && ++since_flush == a.flush_iters) {
      since_flush = 0;
      __syncthreads();
      flush_mass<R, SPLIT>(s, nbins);
      __syncthreads();
    }
  }
  __syncthreads();
  if (MASS) {
    flush_mass<R, SPLIT>(s, nbins);
    __syncthreads();
  }
  // fold replicas and publish this block's histogram
  if (R == 32) {
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t j = warp; j < nbins; j += nw) {
      unsigned long long c = s.cnt[j * 32 + lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) {
        if (c) atomicAdd(a.g_cnt + j, c);
        if (MASS && s.acc[j]) atomicAdd(a.g_mass + j, s.acc[j]);
      }
    }
  } else {
    for (uint32_t j = threadIdx.x; j < nbins; j += blockDim.x) {
      if (s.cnt[j]) atomicAdd(a.g_cnt + j, (unsigned long long)s.cnt[j]);
      if (MASS && s.acc[j]) atomicAdd(a.g_mass + j, s.acc[j]);
    }
  }
}

// ---- variant selection ----------------------------------------------------------
struct Variant {
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
  return lut + (size_t)nbins * 8 + (size_t)nbins * v.R * words * 4;
}

Variant choose(const TraceArgs &a, int block) {
  Variant v;
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

template <int LUTW, int R, bool SPLIT, bool MASS>
void *kernel_ptr() { return reinterpret_cast<void *>(&k1_trace<LUTW, R, SPLIT, MASS>); }

void *pick_kernel(const Variant &v) {
#define FP_K(L)                                                                  \
  if (v.lutw == L) {                                                             \
    if (!v.mass) return v.R == 32 ? kernel_ptr<L, 32, false, false>() : kernel_ptr<L, 1, false, false>(); \
    if (v.R == 32) return v.split ? kernel_ptr<L, 32, true, true>() : kernel_ptr<L, 32, false, true>();   \
    return v.split ? kernel_ptr<L, 1, true, true>() : kernel_ptr<L, 1, false, true>();                    \
  }
  FP_K(0)
  FP_K(1)
  FP_K(2)
#undef FP_K
  return nullptr;
}

}  // namespace

size_t trace_smem_bytes(const TraceArgs &a, int block) { return smem_for(a, choose(a, block)); }

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
  void *k = pick_kernel(v);
  for (uint64_t off = 0; off < a0.n; off += cap) {
    a.len = a0.len + off;
    a.n = std::min<uint64_t>(cap, a0.n - off);
    void *args[] = {&a};
    cudaError_t e = cudaLaunchKernel(k, dim3(grid), dim3(block), args, smem, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ============================== K4: route_batch ===================================
// Alg. 1 for one (B, C_S, C_L): 16 requests per thread per step
// (4 x 128-bit loads in, one 128-bit store of 16 decision bytes out), counts in
// registers, one warp/block reduction and 5 global atomics per block.
namespace {

__device__ __forceinline__ uint32_t decide(uint32_t L, uint32_t B, uint32_t CS, uint32_t CL) {
  if (L > CL) return 2u | (3u << 2);          // rejected (R3)
  if (L > CS) return 1u | (1u << 2);          // step 1: feasibility
  uint32_t p = (L <= B) ? 0u : 1u;            // step 2: budget
  // step 3 (spillover) is out of scope; final safety check:
  if (L > (p == 0u ? CS : CL)) return 1u | (2u << 2);
  return p;
}

struct RouteAcc {
  uint32_t ns = 0, nl = 0, nr = 0;
  unsigned long long ms = 0, ml = 0;
  __device__ __forceinline__ uint32_t add(uint32_t L, uint32_t B, uint32_t CS, uint32_t CL) {
    uint32_t d = decide(L, B, CS, CL);
    uint32_t p = d & 3u;
    ns += p == 0u;
    nl += p == 1u;
    nr += p == 2u;
    ms += p == 0u ? L : 0u;
    ml += p == 1u ? L : 0u;
    return d;
  }
};

template <bool DEC>
__global__ void __launch_bounds__(256) k4_route(RouteArgs a) {
  RouteAcc acc;
  // align the 16-element groups to the decision buffer (or to len without one)
  const uintptr_t anchor = DEC ? reinterpret_cast<uintptr_t>(a.decision) : reinterpret_cast<uintptr_t>(a.len) >> 2;
  const uint64_t head = umin64(a.n, (16u - (uint32_t)(anchor & 15u)) & 15u);
  const uint64_t groups = (a.n - head) >> 4;
  const uint64_t tail_first = head + (groups << 4);
  const bool vec_in = ((reinterpret_cast<uintptr_t>(a.len + head)) & 15u) == 0u;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g = tid; g < groups; g += nthr) {
    const uint64_t e0 = head + (g << 4);
    uint32_t L[16];
    if (vec_in) {
      const uint4 *p = reinterpret_cast<const uint4 *>(a.len + e0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v = ldg_stream(p + q);
        L[4 * q] = v.x; L[4 * q + 1] = v.y; L[4 * q + 2] = v.z; L[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) L[q] = __ldg(a.len + e0 + q);
    }
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      w[q] = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) w[q] |= acc.add(L[4 * q + r], a.b, a.cs, a.cl) << (8 * r);
    }
    if (DEC) *reinterpret_cast<uint4 *>(a.decision + e0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  // head and tail (< 16 each)
  if (tid < head) {
    uint32_t d = acc.add(a.len[tid], a.b, a.cs, a.cl);
    if (DEC) a.decision[tid] = (uint8_t)d;
  }
  if (tid < a.n - tail_first) {
    const uint64_t i = tail_first + tid;
    uint32_t d = acc.add(a.len[i], a.b, a.cs, a.cl);
    if (DEC) a.decision[i] = (uint8_t)d;
  }
  // reduce: warp shuffles, then one atomic per warp
  unsigned long long v[5] = {acc.ns, acc.nl, acc.nr, acc.ms, acc.ml};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  __shared__ unsigned long long red[5][8];
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

cudaError_t launch_route(const RouteArgs &a, int grid, int block, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const uint64_t groups = a.n / 16 + 1;
  const uint64_t need = (groups + block - 1) / block;
  const int g = (int)std::min<uint64_t>((uint64_t)grid, std::max<uint64_t>(1, need));
  if (a.decision) k4_route<true><<<g, block, 0, s>>>(a);
  else k4_route<false><<<g, block, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace fp
