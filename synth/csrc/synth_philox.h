/* Philox4x32-10 and table sampling for the synthetic trace generator.
 * INPUT MODULE (shared by the host-C and CUDA generators only; the product
 * library and the oracle do not include this file). See synth/gen.py for the
 * definition of a trace. */
#ifndef SYNTH_PHILOX_H
#define SYNTH_PHILOX_H
#include <stdint.h>

#ifdef __CUDACC__
#define SYN_HD __host__ __device__ __forceinline__
#else
#define SYN_HD static inline
#endif

#define SYN_LUT_SIZE 65537u

SYN_HD void syn_philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
}

SYN_HD uint32_t syn_sample(const uint32_t *q, uint8_t interp, uint32_t w) {
  uint32_t i = w >> 16;
  uint32_t a = q[i];
  if (!interp) return a;
  uint32_t b = q[i + 1];
  return a + (uint32_t)((((uint64_t)(b - a)) * (uint64_t)(w & 0xFFFFu)) >> 16);
}

/* luts: [n_comp][2][SYN_LUT_SIZE]; interp: [n_comp][2]; cuts: [n_comp-1] */
SYN_HD uint32_t syn_request(const uint32_t *luts, const uint8_t *interp,
                            const uint32_t *cuts, uint32_t n_comp,
                            uint64_t seed, uint64_t i) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0u, 0u};
  syn_philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t comp = 0;
  for (uint32_t k = 0; k + 1 < n_comp; ++k) comp += (c[2] >= cuts[k]) ? 1u : 0u;
  const uint32_t *qi = luts + (uint64_t)comp * 2u * SYN_LUT_SIZE;
  const uint32_t *qo = qi + SYN_LUT_SIZE;
  return syn_sample(qi, interp[2 * comp], c[0]) + syn_sample(qo, interp[2 * comp + 1], c[1]);
}
/* Raw request columns (NEXT-1): see synth/shapes.py "Raw request columns".
 * ratio: [n_cat][65536] 16.16 fixed point; cat_cuts: [n_cat-1] on 16 bits. */
SYN_HD void syn_request_raw(const uint32_t *luts, const uint8_t *interp, const uint32_t *cuts,
                            uint32_t n_comp, const uint32_t *ratio, const uint32_t *cat_cuts,
                            uint32_t n_cat, uint64_t seed, uint64_t i, uint32_t *bytes,
                            uint32_t *max_out, uint8_t *cat, uint32_t *true_prompt) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0u, 0u};
  syn_philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t comp = 0;
  for (uint32_t k = 0; k + 1 < n_comp; ++k) comp += (c[2] >= cuts[k]) ? 1u : 0u;
  const uint32_t *qi = luts + (uint64_t)comp * 2u * SYN_LUT_SIZE;
  const uint32_t *qo = qi + SYN_LUT_SIZE;
  uint32_t lin = syn_sample(qi, interp[2 * comp], c[0]);
  uint32_t lout = syn_sample(qo, interp[2 * comp + 1], c[1]);
  uint32_t k = 0, lo = c[3] & 0xFFFFu;
  for (uint32_t j = 0; j + 1 < n_cat; ++j) k += (lo >= cat_cuts[j]) ? 1u : 0u;
  uint64_t r = ratio[(uint64_t)k * 65536u + (c[3] >> 16)];
  *bytes = (uint32_t)(((uint64_t)lin * r + 0x8000u) >> 16);
  *max_out = lout;
  *cat = (uint8_t)k;
  *true_prompt = lin;
}
/* Arrival gaps (NEXT-4): see synth/shapes.py "Arrival times". */
SYN_HD uint32_t syn_gap(const uint32_t *gap_table, const uint32_t *burst8, uint64_t seed, uint64_t i) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), 1u, 0u};
  syn_philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t g = gap_table[c[0] >> 16];
  return (uint32_t)((g * burst8[(i >> 20) & 7u]) >> 3);
}
#endif
