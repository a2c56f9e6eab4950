// Microbenchmark (measurement tool): best way to stream 4 GB of u32 through
// the SMs on B200 -- LDG.128 grid-stride vs block-contiguous vs TMA bulk ring.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg4(const uint4 *p) {
  uint4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r;
}
template <int UNR>
__global__ void r_gridstride(const uint4 *L, uint64_t n4, unsigned *out) {
  uint32_t acc = 0; uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n4; b += stride * UNR) {
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = (b + u * stride < n4) ? ldg4(L + b + u * stride) : make_uint4(0,0,0,0);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x9e3779b9u) out[0] = acc;
}
template <int UNR>
__global__ void r_blockchunk(const uint4 *L, uint64_t n4, unsigned *out) {
  uint32_t acc = 0;
  uint64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  uint64_t lo = blockIdx.x * per, hi = min(n4, lo + per);
  for (uint64_t b = lo + threadIdx.x; b < hi; b += (uint64_t)blockDim.x * UNR) {
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = (b + u * blockDim.x < hi) ? ldg4(L + b + u * blockDim.x) : make_uint4(0,0,0,0);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x9e3779b9u) out[0] = acc;
}
// TMA bulk ring: warp 0 lane 0 produces; all warps (incl. 0) consume.
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes)); }
__device__ __forceinline__ void mbar_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((unsigned)__cvta_generic_to_shared(b))); }
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned ph) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"((unsigned)__cvta_generic_to_shared(b)), "r"(ph));
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
    :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
template <int STAGES, int TILE>  // TILE bytes per stage
__global__ void r_tma(const uint32_t *L, uint64_t n, unsigned *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *full = (uint64_t *)sm, *empty = full + STAGES;
  unsigned char *buf = sm + 128;
  const int nw = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, nw); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint64_t tile_elems = TILE / 4;
  const uint64_t ntiles = n / tile_elems;   // tail ignored in microbench
  uint32_t acc = 0;
  uint64_t t0 = blockIdx.x;
  // prologue
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { uint64_t t = t0 + (uint64_t)s * gridDim.x; if (t < ntiles) { mbar_expect(full + s, TILE); bulk_g2s(buf + s * TILE, L + t * tile_elems, TILE, full + s); } }
  }
  int s = 0; unsigned ph = 0;
  for (uint64_t t = t0, k = 0; t < ntiles; t += gridDim.x, ++k) {
    mbar_wait(full + s, ph);
    const uint4 *p = (const uint4 *)(buf + s * TILE);
    for (int i = threadIdx.x; i < TILE / 16; i += blockDim.x) { uint4 v = p[i]; acc += v.x ^ v.y ^ v.z ^ v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
    if (threadIdx.x == 0) {
      uint64_t tn = t + (uint64_t)STAGES * gridDim.x;
      if (tn < ntiles) { mbar_wait(empty + s, ph); mbar_expect(full + s, TILE); bulk_g2s(buf + s * TILE, L + tn * tile_elems, TILE, full + s); }
    }
    if (++s == STAGES) { s = 0; ph ^= 1; }
  }
  if (acc == 0x9e3779b9u) out[0] = acc;
}

template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms); }
  return best;
}
int main() {
  uint64_t n = 1000000000ULL; uint32_t *L; unsigned *o; CK(cudaMalloc(&L, n * 4)); CK(cudaMalloc(&o, 64)); CK(cudaMemset(L, 1, n * 4));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char *nm, float ms) { printf("%-40s %8.3f ms %7.1f GB/s\n", nm, ms, n * 4 / ms / 1e6); fflush(stdout); };
  char nm[128];
  const uint4 *L4 = (const uint4 *)L; uint64_t n4 = n / 4;
  for (int thr : {128, 256, 512, 1024}) for (int tps : {256, 512, 768, 1024, 1536, 2048}) {
    if (tps < thr) continue; int bps = tps / thr;
    snprintf(nm, 128, "gridstride U1 t%d tps%d", thr, tps); rep(nm, timeit([&] { r_gridstride<1><<<nsm * bps, thr>>>(L4, n4, o); }));
    snprintf(nm, 128, "gridstride U2 t%d tps%d", thr, tps); rep(nm, timeit([&] { r_gridstride<2><<<nsm * bps, thr>>>(L4, n4, o); }));
    snprintf(nm, 128, "gridstride U4 t%d tps%d", thr, tps); rep(nm, timeit([&] { r_gridstride<4><<<nsm * bps, thr>>>(L4, n4, o); }));
    snprintf(nm, 128, "gridstride U8 t%d tps%d", thr, tps); rep(nm, timeit([&] { r_gridstride<8><<<nsm * bps, thr>>>(L4, n4, o); }));
    snprintf(nm, 128, "blockchunk U4 t%d tps%d", thr, tps); rep(nm, timeit([&] { r_blockchunk<4><<<nsm * bps, thr>>>(L4, n4, o); }));
  }
#define TMA(S, T, THR, BPS) { auto k = r_tma<S, T>; size_t sm = 128 + (size_t)S * T; CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
   snprintf(nm, 128, "tma S%d T%dK t%d b%d", S, T / 1024, THR, BPS); rep(nm, timeit([&] { k<<<nsm * BPS, THR, sm>>>(L, n, o); })); }
  TMA(4, 16384, 256, 1) TMA(8, 16384, 256, 1) TMA(4, 32768, 256, 1) TMA(6, 32768, 512, 1) TMA(4, 16384, 256, 2) TMA(3, 32768, 256, 2)
  TMA(8, 8192, 256, 2) TMA(4, 8192, 128, 4) TMA(12, 16384, 512, 1) TMA(2, 32768, 256, 3)
  return 0;
}
