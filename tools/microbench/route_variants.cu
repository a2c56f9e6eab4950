// Microbenchmark (measurement tool): read 4 B + write 1 B per element over 1e9
// elements -- the K4 route_batch access pattern -- with different load/store
// policies, to find the achievable bandwidth for this mix on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ld_nc(const uint4 *p) {
  uint4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r;
}
__device__ __forceinline__ uint4 ld_ef(const uint4 *p, uint64_t pol) {
  uint4 r; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol)); return r;
}
__device__ __forceinline__ void st_cs(uint32_t *p, uint32_t v) { asm volatile("st.global.cs.u32 [%0], %1;" :: "l"(p), "r"(v)); }
__device__ __forceinline__ void st_na(uint32_t *p, uint32_t v) { asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" :: "l"(p), "r"(v)); }
__device__ __forceinline__ void st_cs4(uint4 *p, uint4 v) { asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)); }

__device__ __forceinline__ uint32_t pack(uint4 v, uint32_t B) {
  return (v.x > B) | ((v.y > B) << 8) | ((v.z > B) << 16) | ((v.w > B) << 24);
}

// V: 0 plain store, 1 st.cs, 2 st.cs + L2 evict_first loads, 3 st.na, 4 smem-staged STG.128 cs
template <int V, int UNR>
__global__ void __launch_bounds__(512) kr(const uint4 *L, uint32_t *D, uint64_t n4, uint32_t B, unsigned *o) {
  __shared__ uint32_t stage[512 * UNR];
  uint64_t pol = 0;
  if (V == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint64_t tile4 = (uint64_t)blockDim.x * UNR;
  const uint64_t ntiles = n4 / tile4;
  uint32_t acc = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * tile4 + threadIdx.x;
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = (V == 2) ? ld_ef(L + base + u * blockDim.x, pol) : ld_nc(L + base + u * blockDim.x);
    if (V == 4) {
#pragma unroll
      for (int u = 0; u < UNR; ++u) stage[threadIdx.x + u * blockDim.x] = pack(v[u], B);
      __syncthreads();
      uint4 *dst = reinterpret_cast<uint4 *>(D + t * tile4);
      const uint4 *src = reinterpret_cast<const uint4 *>(stage);
      for (int i = threadIdx.x; i < (int)(blockDim.x * UNR / 4); i += blockDim.x) st_cs4(dst + i, src[i]);
      __syncthreads();
    } else {
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        uint32_t w = pack(v[u], B);
        uint32_t *p = D + base + u * blockDim.x;
        if (V == 0) *p = w; else if (V == 3) st_na(p, w); else st_cs(p, w);
      }
    }
  }
  if (acc == 12345) o[0] = acc;
}
// pure read for reference
template <int UNR>
__global__ void __launch_bounds__(512) kread(const uint4 *L, uint64_t n4, unsigned *o) {
  const uint64_t tile4 = (uint64_t)blockDim.x * UNR; const uint64_t ntiles = n4 / tile4; uint32_t acc = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * tile4 + threadIdx.x; uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = ld_nc(L + base + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x ^ v[u].w;
  }
  if (acc == 12345) o[0] = acc;
}

template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms); }
  return best;
}
int main() {
  uint64_t n = 1000000000ULL; uint32_t *L, *D; unsigned *o;
  CK(cudaMalloc(&L, n * 4)); CK(cudaMalloc(&D, n)); CK(cudaMalloc(&o, 64)); CK(cudaMemset(L, 7, n * 4));
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint4 *L4 = (const uint4 *)L; uint64_t n4 = n / 4;
  auto rep = [&](const char *nm, float ms, double bytes) { printf("%-34s %8.3f ms %7.1f GB/s\n", nm, ms, bytes / ms / 1e6); fflush(stdout); };
  char nm[96];
  for (int bps : {2, 3, 4}) {
    snprintf(nm, 96, "read-only U4 b%d", bps); rep(nm, timeit([&] { kread<4><<<nsm * bps, 512>>>(L4, n4, o); }), 4.0 * n);
#define RV(V, U) snprintf(nm, 96, "route V%d U%d b%d", V, U, bps); rep(nm, timeit([&] { kr<V, U><<<nsm * bps, 512>>>(L4, D, n4, 100, o); }), 5.0 * n);
    RV(0, 4) RV(1, 4) RV(2, 4) RV(3, 4) RV(4, 4) RV(1, 8) RV(0, 2)
  }
  return 0;
}
