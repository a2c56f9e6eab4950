// FP64 FMA peak on this GPU (the K3 denominator is not in
// MEASURED_PEAKS.json). 8 independent DFMA chains per thread, a full grid of
// resident blocks; FLOP/s = 2 * FMAs / time. Also the IEEE div.rn.f64 rate.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __fma_rn(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void ddiv_kernel(double *out, int iters, double a) {
  double x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = threadIdx.x + j + 1.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = __ddiv_rn(a, x[j]) + 1.0;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = (double)blocks * threads * iters * 8;
  printf("dfma: %.3f ms, %.2f TFLOP/s fp64 (%.1f DFMA/clk/SM at 1965 MHz)\n", ms, 2 * fmas / (ms * 1e-3) / 1e12,
         fmas / (ms * 1e-3) / sms / 1.965e9);
  ddiv_kernel<<<blocks, threads>>>(d, 100, 3.0);
  cudaEventRecord(e0);
  ddiv_kernel<<<blocks, threads>>>(d, iters / 4, 3.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double divs = (double)blocks * threads * (iters / 4) * 4;
  printf("ddiv: %.3f ms, %.3e div.rn.f64/s (%.2f per clk per SM)\n", ms, divs / (ms * 1e-3),
         divs / (ms * 1e-3) / sms / 1.965e9);
  return 0;
}
