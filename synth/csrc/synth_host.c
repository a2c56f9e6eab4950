/* Host-C synthetic trace generator (INPUT MODULE). Fills out[0..count) with
 * requests first..first+count-1. OpenMP-parallel; every element depends only
 * on its index, so the result is independent of the thread count. */
#include "synth_philox.h"

int synth_generate_host(const uint32_t *luts, const uint8_t *interp, const uint32_t *cuts,
                        uint32_t n_comp, uint64_t seed, uint64_t first, uint64_t count,
                        uint32_t *out) {
  if (n_comp == 0 || (count && !out)) return 1;
  int64_t n = (int64_t)count;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j)
    out[j] = syn_request(luts, interp, cuts, n_comp, seed, first + (uint64_t)j);
  return 0;
}

int synth_generate_raw_host(const uint32_t *luts, const uint8_t *interp, const uint32_t *cuts,
                            uint32_t n_comp, const uint32_t *ratio, const uint32_t *cat_cuts,
                            uint32_t n_cat, uint64_t seed, uint64_t first, uint64_t count,
                            uint32_t *bytes, uint32_t *max_out, uint8_t *cat, uint32_t *true_prompt) {
  if (n_comp == 0 || n_cat == 0) return 1;
  int64_t n = (int64_t)count;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j)
    syn_request_raw(luts, interp, cuts, n_comp, ratio, cat_cuts, n_cat, seed, first + (uint64_t)j,
                    bytes + j, max_out + j, cat + j, true_prompt + j);
  return 0;
}

int synth_gaps_host(const uint32_t *gap_table, const uint32_t *burst8, uint64_t seed, uint64_t first,
                    uint64_t count, uint32_t *out) {
  int64_t n = (int64_t)count;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) out[j] = syn_gap(gap_table, burst8, seed, first + (uint64_t)j);
  return 0;
}
