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
