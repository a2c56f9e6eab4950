/* CUDA synthetic trace generator K0 (INPUT MODULE; not part of the product
 * library and never timed). Grid-stride over [0, count); request first+j. */
#include <cuda_runtime.h>
#include "synth_philox.h"

__global__ void synth_gen_kernel(const uint32_t *__restrict__ luts, const uint8_t *__restrict__ interp,
                                 const uint32_t *__restrict__ cuts, uint32_t n_comp, uint64_t seed,
                                 uint64_t first, uint64_t count, uint32_t *__restrict__ out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
    out[j] = syn_request(luts, interp, cuts, n_comp, seed, first + j);
}

extern "C" int synth_generate_device(const uint32_t *d_luts, const uint8_t *d_interp,
                                     const uint32_t *d_cuts, uint32_t n_comp, uint64_t seed,
                                     uint64_t first, uint64_t count, uint32_t *d_out,
                                     cudaStream_t stream) {
  if (n_comp == 0) return 1;
  if (count == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256;
  uint64_t cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  synth_gen_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d_luts, d_interp, d_cuts, n_comp, seed,
                                                         first, count, d_out);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

__global__ void synth_gen_raw_kernel(const uint32_t *__restrict__ luts, const uint8_t *__restrict__ interp,
                                     const uint32_t *__restrict__ cuts, uint32_t n_comp,
                                     const uint32_t *__restrict__ ratio, const uint32_t *__restrict__ cat_cuts,
                                     uint32_t n_cat, uint64_t seed, uint64_t first, uint64_t count,
                                     uint32_t *bytes, uint32_t *max_out, uint8_t *cat, uint32_t *true_prompt) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
    syn_request_raw(luts, interp, cuts, n_comp, ratio, cat_cuts, n_cat, seed, first + j, bytes + j,
                    max_out + j, cat + j, true_prompt + j);
}

extern "C" int synth_generate_raw_device(const uint32_t *d_luts, const uint8_t *d_interp,
                                         const uint32_t *d_cuts, uint32_t n_comp, const uint32_t *d_ratio,
                                         const uint32_t *d_cat_cuts, uint32_t n_cat, uint64_t seed,
                                         uint64_t first, uint64_t count, uint32_t *bytes, uint32_t *max_out,
                                         uint8_t *cat, uint32_t *true_prompt, cudaStream_t stream) {
  if (n_comp == 0 || n_cat == 0) return 1;
  if (count == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256;
  uint64_t cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  synth_gen_raw_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d_luts, d_interp, d_cuts, n_comp, d_ratio,
                                                             d_cat_cuts, n_cat, seed, first, count, bytes,
                                                             max_out, cat, true_prompt);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

__global__ void synth_gaps_kernel(const uint32_t *__restrict__ gap_table, const uint32_t *__restrict__ burst8,
                                  uint64_t seed, uint64_t first, uint64_t count, uint32_t *out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
    out[j] = syn_gap(gap_table, burst8, seed, first + j);
}

extern "C" int synth_gaps_device(const uint32_t *d_gap_table, const uint32_t *d_burst8, uint64_t seed,
                                 uint64_t first, uint64_t count, uint32_t *d_out, cudaStream_t stream) {
  if (count == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256, cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  synth_gaps_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d_gap_table, d_burst8, seed, first, count, d_out);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
