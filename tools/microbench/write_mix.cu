// Microbenchmark (measurement tool): HBM ceilings for K4p's access mix.
// K4p reads 12 B (u64 nibble lanes + u32 crumb lanes) and writes 16 B
// (16 decision bytes) per 16-request chunk: 0.75 B in, 1 B out per request.
// Kernels: the same loads/stores with no compute (mix), write-only uint4
// stores, and a 1:1 uint4 copy; grid-stride, 444 x 512 like K4p, 4 chunks
// per thread in flight. Best of 10 over 1e9 requests (62.5 M chunks).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void mix(const unsigned long long *lo, const uint32_t *hi, uint4 *out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    unsigned long long a[4]; uint32_t b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n) { a[u] = __ldcs(lo + i + u * stride); b[u] = __ldcs(hi + i + u * stride); }
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n)
      __stcs(out + i + u * stride, make_uint4((uint32_t)a[u], (uint32_t)(a[u] >> 32), b[u], b[u] ^ 1u));
  }
}
__global__ void wonly(uint4 *out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    __stcs(out + i, make_uint4((uint32_t)i, 1u, 2u, 3u));
}
__global__ void copy(const uint4 *in, uint4 *out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n) v[u] = __ldcs(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n) __stcs(out + i + u * stride, v[u]);
  }
}
template <int U, bool CS>
__global__ void copyv(const uint4 *in, uint4 *out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n) v[u] = CS ? __ldcs(in + i + u * stride) : in[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n) { if (CS) __stcs(out + i + u * stride, v[u]); else out[i + u * stride] = v[u]; }
  }
}
template <int U, bool CS>
__global__ void mixv(const unsigned long long *lo, const uint32_t *hi, uint4 *out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += U * stride) {
    unsigned long long a[U]; uint32_t b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n) { a[u] = CS ? __ldcs(lo + i + u * stride) : lo[i + u * stride]; b[u] = CS ? __ldcs(hi + i + u * stride) : hi[i + u * stride]; }
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n) {
      const uint4 v = make_uint4((uint32_t)a[u], (uint32_t)(a[u] >> 32), b[u], b[u] ^ 1u);
      if (CS) __stcs(out + i + u * stride, v); else out[i + u * stride] = v;
    }
  }
}
// K1's mix: per thread-step 4 uint4 loads (16 requests) and one 8-B + one 4-B
// store (the packed bins), chunks c = k*S + t as in K1
template <int U>
__global__ void k1mix(const uint4 *in, unsigned long long *lo, uint32_t *hi, uint64_t nchunks) {
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += U * S) {
    uint4 v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v[u][j] = c + u * S < nchunks ? __ldcs(in + 4 * (c + u * S) + j) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c + u * S >= nchunks) continue;
      uint32_t x = 0, y = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) { x ^= v[u][j].x + v[u][j].y; y ^= v[u][j].z + v[u][j].w; }
      __stcs(lo + c + u * S, ((unsigned long long)x << 32) | y);
      __stcs(hi + c + u * S, x ^ y);
    }
  }
}
template <int U>
__global__ void ronly(const uint4 *in, uint32_t *out, uint64_t n4) {
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += U * S) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * S < n4 ? __ldcs(in + i + u * S) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x9e3779b9u) out[0] = acc;
}
template <class F> float best(F f) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float m = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float t; CK(cudaEventElapsedTime(&t, a, b)); m = t < m ? t : m;
  }
  return m;
}
int main() {
  const uint64_t chunks = 62500000ull;   // 1e9 requests / 16
  unsigned long long *lo; uint32_t *hi; uint4 *out, *in;
  CK(cudaMalloc(&lo, chunks * 8)); CK(cudaMalloc(&hi, chunks * 4));
  CK(cudaMalloc(&out, chunks * 16)); CK(cudaMalloc(&in, chunks * 16));
  CK(cudaMemset(lo, 1, chunks * 8)); CK(cudaMemset(hi, 2, chunks * 4)); CK(cudaMemset(in, 3, chunks * 16));
  const int grid = 444, block = 512;
  float t = best([&] { mix<<<grid, block>>>(lo, hi, out, chunks); });
  printf("mix (12 B in, 16 B out per chunk): %.3f ms, %.0f GB/s\n", t, chunks * 28.0 / t / 1e6);
  t = best([&] { wonly<<<grid, block>>>(out, chunks); });
  printf("write-only uint4: %.3f ms, %.0f GB/s\n", t, chunks * 16.0 / t / 1e6);
  t = best([&] { copy<<<grid, block>>>(in, out, chunks); });
  printf("copy uint4 1:1: %.3f ms, %.0f GB/s\n", t, chunks * 32.0 / t / 1e6);
  t = best([&] { wonly<<<148 * 8, 256>>>(out, chunks); });
  printf("write-only uint4 (1184x256): %.3f ms, %.0f GB/s\n", t, chunks * 16.0 / t / 1e6);
  {
    uint4 *trace;                          // 1e9 requests x 4 B
    CK(cudaMalloc(&trace, chunks * 64));
    CK(cudaMemset(trace, 5, chunks * 64));
    float t1 = best([&] { k1mix<1><<<grid, block>>>(trace, lo, hi, chunks); });
    printf("K1 mix U1 (64 B in, 12 B out per 16 requests) 444x512: %.3f ms, %.0f GB/s\n", t1, chunks * 76.0 / t1 / 1e6);
    t1 = best([&] { k1mix<2><<<grid, block>>>(trace, lo, hi, chunks); });
    printf("K1 mix U2 444x512: %.3f ms, %.0f GB/s\n", t1, chunks * 76.0 / t1 / 1e6);
    t1 = best([&] { k1mix<1><<<148 * 4, 512>>>(trace, lo, hi, chunks); });
    printf("K1 mix U1 592x512: %.3f ms, %.0f GB/s\n", t1, chunks * 76.0 / t1 / 1e6);
    t1 = best([&] { ronly<4><<<grid, block>>>(trace, hi, chunks * 4); });
    printf("read-only 4 GB U4 444x512: %.3f ms, %.0f GB/s\n", t1, chunks * 64.0 / t1 / 1e6);
    t1 = best([&] { ronly<8><<<grid, block>>>(trace, hi, chunks * 4); });
    printf("read-only 4 GB U8 444x512: %.3f ms, %.0f GB/s\n", t1, chunks * 64.0 / t1 / 1e6);
    CK(cudaFree(trace));
  }
  int bps = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, copyv<4, false>, 256, 0));
  const int g2 = 148 * bps;
  t = best([&] { copyv<4, false><<<g2, 256>>>(in, out, chunks); });
  printf("copy plain U4 (%dx256): %.3f ms, %.0f GB/s\n", g2, t, chunks * 32.0 / t / 1e6);
  t = best([&] { copyv<8, false><<<g2, 256>>>(in, out, chunks); });
  printf("copy plain U8: %.3f ms, %.0f GB/s\n", t, chunks * 32.0 / t / 1e6);
  t = best([&] { copyv<2, false><<<g2, 256>>>(in, out, chunks); });
  printf("copy plain U2: %.3f ms, %.0f GB/s\n", t, chunks * 32.0 / t / 1e6);
  t = best([&] { mixv<4, false><<<grid, block>>>(lo, hi, out, chunks); });
  printf("mix plain U4 444x512: %.3f ms, %.0f GB/s\n", t, chunks * 28.0 / t / 1e6);
  t = best([&] { mixv<8, false><<<grid, block>>>(lo, hi, out, chunks); });
  printf("mix plain U8 444x512: %.3f ms, %.0f GB/s\n", t, chunks * 28.0 / t / 1e6);
  t = best([&] { mixv<4, false><<<g2, 256>>>(lo, hi, out, chunks); });
  printf("mix plain U4 %dx256: %.3f ms, %.0f GB/s\n", g2, t, chunks * 28.0 / t / 1e6);
  t = best([&] { mixv<2, true><<<g2, 256>>>(lo, hi, out, chunks); });
  printf("mix cs U2 %dx256: %.3f ms, %.0f GB/s\n", g2, t, chunks * 28.0 / t / 1e6);
  t = best([&] { mixv<8, true><<<g2, 256>>>(lo, hi, out, chunks); });
  printf("mix cs U8 %dx256: %.3f ms, %.0f GB/s\n", g2, t, chunks * 28.0 / t / 1e6);
  return 0;
}
