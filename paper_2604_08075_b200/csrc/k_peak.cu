// NEXT-4: peak-window provisioning.
//
// A trace is in arrival order, so the requests of window
// w = floor(arrival / W) are one contiguous index range [start[w], start[w+1]).
// That turns the two-dimensional histogram cnt[w][b] into K1's problem on
// sub-ranges and removes the arrival column from the streaming pass:
//   K0w  start[w] = lower_bound(arrival, w * W): n_windows + 1 binary searches
//        (O(windows * log n) scattered 8-B reads, not 8 B per request)
//   K1w  each block streams a contiguous slice of L_total (4 B / request,
//        16-B vector loads), bins through the same fine-cell LUT as K1 into a
//        lane-private shared histogram [bin][lane] and flushes one row of
//        nbins global counters per window it touched; windows too short to
//        amortise a flush go straight to global atomics
//   K2w  per chunk of windows: inclusive scan of every row (cnt_le[w][j] =
//        #{requests of w with L <= e_j}) and the maxima over windows that K3
//        needs: colmax[j] = max_w cnt_le[w][j] and, for every (B, C_L) pair,
//        pairmax = max_w (cnt_le[w][C_L] - cnt_le[w][B]). The cumulative rows
//        are never written back.
// The arrival order is the caller's contract; FP_FLAG_CHECK_ORDER adds Kc, a
// full pass that verifies it (8 B / request).
#include <algorithm>
#include <cmath>
#include "internal.cuh"

namespace fp {
namespace {

constexpr int kHistBlock = 512;
constexpr uint64_t kSmallSegment = 2048;   // below this a window goes to global atomics

// one warp per window: a 32-way search (each round 32 probes, one ballot),
// so the dependent chain is ~log32(n) = 6 loads instead of log2(n) = 30 --
// for few windows (the chain is the whole kernel); 6x the probes of the
// binary search, so many windows take k0w_bounds_multi
__global__ void k0w_bounds_warp(PeakArgs a) {
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w > a.n_windows) return;                 // warp-uniform
  if (w == a.n_windows) {
    if (lane == 0) a.start[w] = a.n;
    return;
  }
  const uint64_t t = w * a.window_ns;          // no overflow: checked on the host
  // lower_bound(arrival, t) lies in [lo, hi]: arrival[lo - 1] < t (or lo = 0),
  // arrival[hi] >= t (or hi = n)
  uint64_t lo = 0, hi = a.n;
  while (hi - lo > 32) {
    const uint64_t step = (hi - lo + 31) / 32;
    const uint64_t idx = min(lo + (lane + 1) * step - 1, hi - 1);
    const bool below = __ldg(a.arrival + idx) < t;
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, below));   // probes below t: a prefix
    const uint64_t nlo = c ? min(lo + c * step - 1, hi - 1) + 1 : lo;
    const uint64_t nhi = c < 32 ? min(lo + (c + 1) * step - 1, hi - 1) : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint64_t idx = lo + lane;
  const bool below = idx < hi && __ldg(a.arrival + idx) < t;
  const uint32_t c = __popc(__ballot_sync(0xffffffffu, below));
  if (lane == 0) a.start[w] = lo + c;
}

// many windows: one warp per 32 consecutive windows. Shared 32-way rounds
// narrow one range that holds all 32 answers (probes compared with the first
// and the last target) while that still shrinks it; then every lane takes the
// probe interval of its own target (32 ballots, no loads) and finishes with a
// binary search inside it. ~4 shared rounds + log2(interval) dependent loads
// instead of log2(n) = 30 (1-s windows on 1e9 requests: ~18).
__global__ void k0w_bounds_multi(PeakArgs a) {
  const uint64_t w0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) << 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w0 > a.n_windows) return;                               // warp-uniform
  const uint64_t w = w0 + lane;
  const uint64_t last = min(w0 + 31, a.n_windows);            // the warp's last window (<= n_windows)
  const uint64_t t = min(w, last) * a.window_ns;              // lanes past the end repeat the last target
  const uint64_t tf = __shfl_sync(0xffffffffu, t, 0), tl = __shfl_sync(0xffffffffu, t, 31);
  // every answer lower_bound(arrival, t_lane) lies in [lo, hi]
  uint64_t lo = 0, hi = a.n;
  uint64_t step = 0;
  uint64_t pv = 0;                                            // this lane's probe value (last round)
  uint64_t pidx = 0;
  while (hi - lo > 32) {
    step = (hi - lo + 31) / 32;
    pidx = min(lo + (lane + 1) * step - 1, hi - 1);
    pv = __ldg(a.arrival + pidx);
    const uint32_t cf = __popc(__ballot_sync(0xffffffffu, pv < tf));
    const uint32_t cl = __popc(__ballot_sync(0xffffffffu, pv < tl));
    const uint64_t nlo = cf ? min(lo + cf * step - 1, hi - 1) + 1 : lo;
    const uint64_t nhi = cl < 32 ? min(lo + (cl + 1) * step - 1, hi - 1) : hi;
    if (nhi - nlo > (hi - lo) / 2) break;                     // the targets span the range: split per lane
    lo = nlo;
    hi = nhi;
    step = 0;
  }
  uint64_t mlo = lo, mhi = hi;
  if (step) {
    // this lane's interval from the last round's probes (probe j at pidx_j)
    uint32_t c = 0;
    for (uint32_t j = 0; j < 32; ++j) {
      const uint64_t tj = __shfl_sync(0xffffffffu, t, j);
      const uint32_t cj = __popc(__ballot_sync(0xffffffffu, pv < tj));
      if (lane == j) c = cj;
    }
    mlo = c ? min(lo + c * step - 1, hi - 1) + 1 : lo;
    mhi = c < 32 ? min(lo + (c + 1) * step - 1, hi - 1) : hi;
  }
  // lower_bound(arrival, t) in [mlo, mhi]: arrival[mlo - 1] < t, arrival[mhi] >= t (or mhi = n).
  // Interpolation search on the bracketing values (arrivals of a Poisson trace
  // grow almost linearly inside an interval: ~4 dependent probes instead of the
  // ~14 of a binary search over a 1-s window's interval), with a bisection
  // step whenever an interpolation step kept more than 3/4 of the interval
  uint64_t vlo = mlo ? __ldg(a.arrival + mlo - 1) : 0ull;
  uint64_t vhi = mhi < a.n ? __ldg(a.arrival + mhi) : ~0ull;
  bool bisect = false;
  while (mhi > mlo) {
    const uint64_t len = mhi - mlo;
    uint64_t g = mlo + len / 2;
    if (!bisect && mhi < a.n && vhi > vlo) {
      const double f = (double)(t - vlo) / (double)(vhi - vlo);   // vlo < t <= vhi
      g = mlo + min((uint64_t)(f * (double)len), len - 1);
    }
    const uint64_t v = __ldg(a.arrival + g);
    if (v < t) { mlo = g + 1; vlo = v; } else { mhi = g; vhi = v; }
    bisect = !bisect && (mhi - mlo) * 4 > len * 3;
  }
  if (w <= a.n_windows) a.start[w] = w == a.n_windows ? a.n : mlo;
}

__global__ void kc_check_order(PeakArgs a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < a.n; i += stride)
    bad |= __ldcs(a.arrival + i) > __ldg(a.arrival + i + 1);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.error, 1u);
}

template <int LUTW>
__device__ __forceinline__ uint32_t bin_of(uint32_t L, const unsigned char *lut, uint32_t clampv, uint32_t round,
                                           uint32_t shift, uint32_t ne) {
  if (LUTW == 1) return lut[(min(L, clampv) + round) >> shift];
  if (LUTW == 2) return reinterpret_cast<const uint16_t *>(lut)[(min(L, clampv) + round) >> shift];
  const uint32_t *edges = reinterpret_cast<const uint32_t *>(lut);
  uint32_t lo = 0, n = ne;
  while (n > 0) {
    const uint32_t half = n >> 1;
    if (edges[lo + half] < L) { lo += half + 1; n -= half + 1; } else { n = half; }
  }
  return lo;
}

template <int LUTW>
__global__ void __launch_bounds__(kHistBlock) k1w_hist(PeakArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t nbins = a.nbins;
  uint32_t lut_bytes = LUTW ? a.lut_cells * LUTW : (nbins - 1) * 4;
  lut_bytes = (lut_bytes + 15u) & ~15u;
  unsigned char *lut = smem;
  uint32_t *acc = reinterpret_cast<uint32_t *>(smem + lut_bytes);      // [nbins][32]
  {
    const uint32_t *src = LUTW ? reinterpret_cast<const uint32_t *>(a.lut) : a.edges;
    for (uint32_t i = threadIdx.x; i < lut_bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(lut)[i] = src[i];
    for (uint32_t i = threadIdx.x; i < nbins * 32; i += blockDim.x) acc[i] = 0u;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t clampv = a.clampv, round = a.round, shift = a.shift, ne = nbins - 1;
  const uint32_t *len = a.len;
  // contiguous slice per block, a multiple of 4 requests
  const uint64_t per = ((a.n + gridDim.x - 1) / gridDim.x + 3) & ~3ull;
  const uint64_t lo = min((uint64_t)blockIdx.x * per, a.n), hi = min(lo + per, a.n);
  if (lo >= hi) return;
  // window holding request lo: the last w with start[w] <= lo
  uint64_t w = 0;
  {
    uint64_t l = 0, n = a.n_windows + 1;
    while (n > 0) {
      const uint64_t half = n >> 1;
      if (a.start[l + half] <= lo) { l += half + 1; n -= half + 1; } else { n = half; }
    }
    w = l - 1;
  }
  // first index whose address is 16-B aligned (len is 4-B aligned)
  const uint64_t off = ((16u - ((uintptr_t)len & 15u)) & 15u) >> 2;
  auto add = [&](uint32_t L) { atomicAdd(&acc[bin_of<LUTW>(L, lut, clampv, round, shift, ne) * 32 + lane], 1u); };
  for (uint64_t s = lo; s < hi; ++w) {
    const uint64_t e = min(hi, a.start[w + 1]);
    if (e - s >= kSmallSegment) {
      const uint64_t s4 = min(e, s + ((off - s) & 3));          // first aligned index >= s
      const uint64_t q0 = (s4 - off) >> 2, q1 = (e - off) >> 2;  // aligned quads [q0, q1)
      const uint64_t e4 = off + 4 * q1;
      for (uint64_t i = s + threadIdx.x; i < s4; i += blockDim.x) add(__ldcs(len + i));
      const uint4 *v = reinterpret_cast<const uint4 *>(len + off);
      uint64_t q = q0 + threadIdx.x;
      for (; q + blockDim.x < q1; q += 2 * blockDim.x) {
        const uint4 x = __ldcs(v + q), y = __ldcs(v + q + blockDim.x);
        add(x.x); add(x.y); add(x.z); add(x.w);
        add(y.x); add(y.y); add(y.z); add(y.w);
      }
      if (q < q1) {
        const uint4 x = __ldcs(v + q);
        add(x.x); add(x.y); add(x.z); add(x.w);
      }
      for (uint64_t i = max(e4, s4) + threadIdx.x; i < e; i += blockDim.x) add(__ldcs(len + i));
      __syncthreads();
      uint32_t *row = a.hist2d + w * nbins;
      for (uint32_t j = warp; j < nbins; j += nwarps) {
        uint32_t c = acc[j * 32 + lane];
        acc[j * 32 + lane] = 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0 && c) atomicAdd(row + j, c);
      }
      __syncthreads();
    } else {
      uint32_t *row = a.hist2d + w * nbins;
      for (uint64_t i = s + threadIdx.x; i < e; i += blockDim.x)
        atomicAdd(row + bin_of<LUTW>(__ldcs(len + i), lut, clampv, round, shift, ne), 1u);
    }
    s = e;
  }
}

// K1w, per-warp form (small E): every warp streams its own contiguous slice
// into a warp-private lane-column histogram [nbins][32 lanes], so a window
// boundary costs that warp alone a flush -- no block barrier anywhere in the
// loop. Tiles of 32 lanes x kWU quads, the next tile's loads in flight. A tile
// inside one window adds every request to the histogram; a tile with <= 3
// boundaries makes one predicated pass per window it touches and flushes each
// window that ends in it; a tile with more boundaries (windows of < ~128
// requests) goes to global atomics.
constexpr int kWarpBlock = 256;
constexpr int kWU = 4;

// last window w with start[w] <= i, searching w in [lo, hi] (start[lo] <= i)
__device__ __forceinline__ uint64_t window_of(const uint64_t *start, uint64_t i, uint64_t lo, uint64_t hi) {
  uint64_t n = hi - lo + 1;
  while (n > 0) {
    const uint64_t half = n >> 1;
    if (start[lo + half] <= i) { lo += half + 1; n -= half + 1; } else { n = half; }
  }
  return lo - 1;
}

template <int LUTW>
__global__ void __launch_bounds__(kWarpBlock, 3) k1w_hist_warp(PeakArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t nbins = a.nbins;
  uint32_t lut_bytes = LUTW ? a.lut_cells * LUTW : (nbins - 1) * 4;
  lut_bytes = (lut_bytes + 15u) & ~15u;
  unsigned char *lut = smem;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *acc_all = reinterpret_cast<uint32_t *>(smem + lut_bytes);  // [warps][nbins][32]
  {
    const uint32_t *src = LUTW ? reinterpret_cast<const uint32_t *>(a.lut) : a.edges;
    for (uint32_t i = threadIdx.x; i < lut_bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(lut)[i] = src[i];
    for (uint32_t i = threadIdx.x; i < (blockDim.x >> 5) * nbins * 32; i += blockDim.x) acc_all[i] = 0u;
  }
  // K0w's window starts (and the memset of the 2-D histogram before it) are
  // complete past this point; the LUT and counter setup above overlap K0w
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  uint32_t *acc = acc_all + warp * nbins * 32;
  const uint32_t acc_s = (uint32_t)__cvta_generic_to_shared(acc) + lane * 4u;
  const uint32_t clampv = a.clampv, round = a.round, shift = a.shift, ne = nbins - 1;
  const uint32_t *len = a.len;
  const uint64_t *start = a.start;
  const uint32_t n = (uint32_t)a.n, nw = (uint32_t)a.n_windows;   // < 2^32, <= 2^26 (host checks)
  auto bin = [&](uint32_t L) { return bin_of<LUTW>(L, lut, clampv, round, shift, ne); };
  auto inc = [&](uint32_t L) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(acc_s + bin(L) * 128u) : "memory"); };
  auto global_add = [&](uint32_t w, uint32_t L) { atomicAdd(a.hist2d + (size_t)w * nbins + bin(L), 1u); };
  const uint32_t off = min(n, (uint32_t)(((16u - ((uintptr_t)len & 15u)) & 15u) >> 2));
  const uint32_t nq = (n - off) >> 2;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp, W = gridDim.x * (blockDim.x >> 5);
  if (gw == 0) {      // requests before the first aligned address and after the last full quad
    for (uint32_t i = lane; i < off; i += 32) global_add((uint32_t)window_of(start, i, 0, nw), __ldcs(len + i));
    for (uint32_t i = off + 4 * nq + lane; i < n; i += 32) global_add((uint32_t)window_of(start, i, 0, nw), __ldcs(len + i));
  }
  const uint32_t per = (nq + W - 1) / W;
  const uint32_t qlo = min(gw * per, nq), qhi = min(qlo + per, nq);
  if (qlo >= qhi) return;
  // window f's lane columns -> one global row; lane j sums bin j's 32 columns
  // (8 x 16-B loads, rotated so the lanes of a phase hit distinct banks)
  auto flush = [&](uint32_t f) {
    __syncwarp();
    uint32_t *row = a.hist2d + (size_t)f * nbins;
    for (uint32_t j = lane; j < nbins; j += 32) {
      uint4 *r = reinterpret_cast<uint4 *>(acc + j * 32);
      uint32_t c = 0;
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t kk = (k + j) & 7u;
        const uint4 x = r[kk];
        r[kk] = make_uint4(0u, 0u, 0u, 0u);
        c += x.x + x.y + x.z + x.w;
      }
      if (c) atomicAdd(row + j, c);
    }
    __syncwarp();
  };
  const uint4 *v = reinterpret_cast<const uint4 *>(len + off);
  constexpr uint32_t kT = 32u * kWU;
  uint32_t w = (uint32_t)window_of(start, off + 4ull * qlo, 0, nw);
  uint32_t nb = w < nw ? (uint32_t)__ldg(start + w + 1) : n;      // first request of window w + 1
  uint4 cur[kWU], nxt[kWU];
#pragma unroll
  for (int k = 0; k < kWU; ++k) {
    const uint32_t q = qlo + lane + 32u * k;
    cur[k] = q < qhi ? __ldcs(v + q) : make_uint4(0u, 0u, 0u, 0u);
  }
  for (uint32_t q0 = qlo; q0 < qhi; q0 += kT) {
    const uint32_t q1 = min(q0 + kT, qhi);
    if (q1 < qhi) {
#pragma unroll
      for (int k = 0; k < kWU; ++k) {
        const uint32_t q = q1 + lane + 32u * k;
        nxt[k] = q < qhi ? __ldcs(v + q) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    const uint32_t e1 = off + 4 * q1;
    if (e1 <= nb) {                                    // the tile lies in window w
#pragma unroll
      for (int k = 0; k < kWU; ++k)
        if (q0 + lane + 32u * k < q1) { inc(cur[k].x); inc(cur[k].y); inc(cur[k].z); inc(cur[k].w); }
    } else {
      // windows w .. wl touch the tile; their starts (warp-uniform loads)
      uint32_t bs[4];                                  // bs[d] = start[w + 1 + d]
      bs[0] = nb;
      uint32_t wl = w;
#pragma unroll
      for (int d = 1; d < 4; ++d) bs[d] = (w + 1 + d <= nw) ? (uint32_t)__ldg(start + w + 1 + d) : n;
      while (wl - w < 4 && bs[wl - w] < e1) ++wl;     // wl - w boundaries inside the tile (capped at 4)
      if (wl - w < 4) {
        for (uint32_t d = 0; d <= wl - w; ++d) {
          const uint32_t lo = d ? bs[d - 1] : 0u, hi = bs[d];   // window w + d = [lo, hi)
#pragma unroll
          for (int k = 0; k < kWU; ++k) {
            const uint32_t q = q0 + lane + 32u * k;
            if (q < q1) {
              const uint32_t i0 = off + 4 * q;
              const uint32_t x[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (i0 + c >= lo && (d == wl - w || i0 + c < hi)) inc(x[c]);
            }
          }
          if (d < wl - w) flush(w + d);
        }
        w = wl;
      } else {
        // more than 3 boundaries: flush w, then global atomics for the tile
        flush(w);
        const uint32_t wlast = (uint32_t)window_of(start, e1 - 1, w, nw);
#pragma unroll
        for (int k = 0; k < kWU; ++k) {
          const uint32_t q = q0 + lane + 32u * k;
          if (q < q1) {
            const uint32_t x[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
            uint32_t ww = (uint32_t)window_of(start, off + 4 * q, w, wlast);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t i = off + 4 * q + c;
              while (ww < wlast && __ldg(start + ww + 1) <= i) ++ww;
              global_add(ww, x[c]);
            }
          }
        }
        w = wlast;
      }
      nb = w < nw ? (uint32_t)__ldg(start + w + 1) : n;
    }
#pragma unroll
    for (int k = 0; k < kWU; ++k) cur[k] = nxt[k];
  }
  flush(w);
}

// K2w: inclusive scan of each window's row in shared memory, then the window
// maxima per bin and per (B, C_L) pair; one atomicMax per entry per block
__global__ void __launch_bounds__(256) k2w_peaks(PeakArgs a) {
  extern __shared__ __align__(16) uint32_t sm2[];
  const uint32_t nbins = a.nbins, R = a.rows, n_pairs = a.n_b * a.n_cl;
  uint32_t *rows = sm2;                       // [R][nbins]
  uint32_t *pmax = rows + R * nbins;          // [n_pairs]
  uint32_t *cmax = pmax + n_pairs;            // [nbins]
  for (uint32_t i = threadIdx.x; i < n_pairs; i += blockDim.x) pmax[i] = 0u;
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) cmax[i] = 0u;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // K1w's 2-D histogram (PDL launch)
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (uint64_t w0 = (uint64_t)blockIdx.x * R; w0 < a.n_windows; w0 += (uint64_t)gridDim.x * R) {
    const uint32_t rn = (uint32_t)min((uint64_t)R, a.n_windows - w0);
    __syncthreads();
    const uint32_t *src = a.hist2d + w0 * nbins;
    // 8 independent loads in flight per thread (the rows come from L2)
    for (uint32_t base = threadIdx.x; base < rn * nbins; base += 8 * blockDim.x) {
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = base + k * blockDim.x;
        v[k] = i < rn * nbins ? __ldcg(src + i) : 0u;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = base + k * blockDim.x;
        if (i < rn * nbins) rows[i] = v[k];
      }
    }
    __syncthreads();
    for (uint32_t r = warp; r < rn; r += nwarps) {
      uint32_t *row = rows + r * nbins, carry = 0;
      for (uint32_t base = 0; base < nbins; base += 32) {
        const uint32_t j = base + lane;
        uint32_t v = j < nbins ? row[j] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += y;
        }
        v += carry;
        if (j < nbins) row[j] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < n_pairs; p += blockDim.x) {
      const uint32_t eb = a.b_edge[p / a.n_cl], el = a.cl_edge[p % a.n_cl];
      if (eb > el) continue;                  // B > C_L: no valid candidate uses it
      uint32_t m = pmax[p];
      for (uint32_t r = 0; r < rn; ++r) m = max(m, rows[r * nbins + el] - rows[r * nbins + eb]);
      pmax[p] = m;
    }
    for (uint32_t j = threadIdx.x; j < nbins; j += blockDim.x) {
      uint32_t m = cmax[j];
      for (uint32_t r = 0; r < rn; ++r) m = max(m, rows[r * nbins + j]);
      cmax[j] = m;
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_pairs; i += blockDim.x)
    if (pmax[i]) atomicMax(a.pairmax + i, pmax[i]);
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x)
    if (cmax[i]) atomicMax(a.colmax + i, cmax[i]);
}

template <int LUTW>
cudaError_t launch_hist(const PeakArgs &a, int sm_count, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k1w_hist<LUTW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1w_hist<LUTW>, kHistBlock, smem);
  if (e != cudaSuccess) return e;
  const uint64_t want = (uint64_t)sm_count * (uint64_t)std::max(per_sm, 1);
  const uint64_t useful = std::max<uint64_t>(1, (a.n + 4095) / 4096);
  k1w_hist<LUTW><<<(unsigned)std::min(want, useful), kHistBlock, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

size_t peak_smem_bytes(const PeakArgs &a) {
  const size_t lut = a.lutw ? (size_t)a.lut_cells * a.lutw : (size_t)(a.nbins - 1) * 4;
  return ((lut + 15) & ~size_t(15)) + (size_t)a.nbins * 32 * 4;
}

size_t peak_scan_smem_bytes(const PeakArgs &a) {
  return ((size_t)a.rows * a.nbins + (size_t)a.n_b * a.n_cl + a.nbins) * 4;
}

size_t warp_hist_smem(const PeakArgs &a) {
  const size_t lut = a.lutw ? (size_t)a.lut_cells * a.lutw : (size_t)(a.nbins - 1) * 4;
  return ((lut + 15) & ~size_t(15)) + (size_t)(kWarpBlock / 32) * a.nbins * 32 * 4;
}

template <int LUTW>
cudaError_t launch_hist_warp(const PeakArgs &a, int sm_count, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k1w_hist_warp<LUTW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1w_hist_warp<LUTW>, kWarpBlock, smem);
  if (e != cudaSuccess) return e;
  const uint64_t want = (uint64_t)sm_count * (uint64_t)std::max(per_sm, 1);
  const uint64_t useful = std::max<uint64_t>(1, (a.n + 4095) / 4096);
  return launch_pdl(k1w_hist_warp<LUTW>, dim3((unsigned)std::min(want, useful)), dim3(kWarpBlock), smem, s, a);
}

cudaError_t launch_peak_hist(const PeakArgs &a, int sm_count, cudaStream_t s) {
  cudaError_t e;
  if (a.check_order) {
    kc_check_order<<<sm_count * 4, 512, 0, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (a.n_windows < 16384)
    k0w_bounds_warp<<<(unsigned)((a.n_windows + 1 + 7) / 8), 256, 0, s>>>(a);   // one warp per window
  else
    k0w_bounds_multi<<<(unsigned)((a.n_windows + 1 + 255) / 256), 256, 0, s>>>(a);     // 32 windows per warp
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // per-warp histograms while they fit 3 blocks per SM (|E| + 1 <= ~140 bins)
  const size_t wsmem = warp_hist_smem(a);
  if (wsmem <= 72 * 1024)
    return a.lutw == 1 ? launch_hist_warp<1>(a, sm_count, wsmem, s)
           : a.lutw == 2 ? launch_hist_warp<2>(a, sm_count, wsmem, s)
                         : launch_hist_warp<0>(a, sm_count, wsmem, s);
  const size_t smem = peak_smem_bytes(a);
  e = a.lutw == 1 ? launch_hist<1>(a, sm_count, smem, s)
      : a.lutw == 2 ? launch_hist<2>(a, sm_count, smem, s)
                    : launch_hist<0>(a, sm_count, smem, s);
  if (e != cudaSuccess) return e;
  return cudaSuccess;
}

cudaError_t launch_peak_scan(const PeakArgs &a, int sm_count, cudaStream_t s) {
  const size_t smem2 = peak_scan_smem_bytes(a);
  cudaError_t e = cudaFuncSetAttribute(k2w_peaks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  if (e != cudaSuccess) return e;
  const uint64_t chunks = (a.n_windows + a.rows - 1) / a.rows;
  return launch_pdl(k2w_peaks, dim3((unsigned)std::min<uint64_t>(chunks, (uint64_t)sm_count * 4)), dim3(256), smem2, s,
                    a);
}

}  // namespace fp
