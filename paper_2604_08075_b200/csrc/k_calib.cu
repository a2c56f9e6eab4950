// NEXT-3: calibration replay on the GPU -- Alg. 1 OnResponse with
// Eq. `ema` over a feedback stream in arrival order:
//   c_obs = |r| / usage.prompt_tokens
//   c_k   <- beta c_k + (1 - beta) c_obs
//   s_k   <- beta s_k + (1 - beta) |c_obs - c_k(before)|          (R26)
// Both recurrences are affine in their state, x -> a x + b, and affine maps
// compose associatively: (a2, b2) o (a1, b1) = (a2 a1, a2 b1 + b2). The
// stream is cut into one contiguous segment per thread:
//   C1  each thread composes, per category, the maps of its segment (c_hat)
//   C2  one block per category scans the per-thread maps (exclusive prefix)
//   C3  each thread replays its segment from its prefix state (exactly the
//       sequential update), which yields every c_hat(before) and so the
//       sigma maps; records the n = snap_at snapshot of c_hat
//   C2  again for the sigma maps, C4 replays the segments holding a snapshot
// The composition reassociates the fp64 sums, so results agree with the
// sequential oracle to rounding (tests: <= 1e-12 relative), not bit for bit.
#include <cmath>
#include "internal.cuh"

namespace fp {

namespace {

constexpr int kCalBlock = 256;

__device__ __forceinline__ uint64_t umin(uint64_t x, uint64_t y) { return x < y ? x : y; }

struct Obs {
  bool valid;
  uint32_t k;
  double c;
};

__device__ __forceinline__ Obs load_obs(const CalibArgs &a, uint64_t i) {
  Obs o;
  const uint32_t t = a.tokens[i];
  o.valid = t != 0;                                   // invalid feedback dropped
  const uint32_t k = a.cat[i];
  o.k = k < a.n_cats ? k : a.n_cats - 1;              // R23
  o.c = o.valid ? __ddiv_rn(__uint2double_rn(a.bytes[i]), __uint2double_rn(t)) : 0.0;
  return o;
}

// per-thread map state in shared memory: [k][thread] (conflict-free)
struct MapSmem {
  double *A, *B;
  uint32_t *cnt;
  __device__ double &a(uint32_t k) { return A[k * kCalBlock + threadIdx.x]; }
  __device__ double &b(uint32_t k) { return B[k * kCalBlock + threadIdx.x]; }
  __device__ uint32_t &n(uint32_t k) { return cnt[k * kCalBlock + threadIdx.x]; }
};

__device__ __forceinline__ MapSmem map_smem(unsigned char *smem, uint32_t n_cats) {
  MapSmem m;
  m.A = reinterpret_cast<double *>(smem);
  m.B = m.A + n_cats * kCalBlock;
  m.cnt = reinterpret_cast<uint32_t *>(m.B + n_cats * kCalBlock);
  return m;
}

__device__ __forceinline__ void segment(const CalibArgs &a, uint64_t t, uint64_t &lo, uint64_t &hi) {
  lo = umin(a.n, t * a.seg);
  hi = umin(a.n, lo + a.seg);
}

// C1: per-thread composed maps of the c_hat recurrence
__global__ void __launch_bounds__(kCalBlock) c1_maps(CalibArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  MapSmem s = map_smem(smem, a.n_cats);
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t k = 0; k < a.n_cats; ++k) { s.a(k) = 1.0; s.b(k) = 0.0; s.n(k) = 0; }
  uint64_t lo, hi;
  segment(a, t, lo, hi);
  const double w = __dsub_rn(1.0, a.beta);
  for (uint64_t i = lo; i < hi; ++i) {
    const Obs o = load_obs(a, i);
    if (!o.valid) continue;
    s.a(o.k) = __dmul_rn(a.beta, s.a(o.k));
    s.b(o.k) = __dadd_rn(__dmul_rn(a.beta, s.b(o.k)), __dmul_rn(w, o.c));
    s.n(o.k) += 1;
  }
  if (t < a.threads)
    for (uint32_t k = 0; k < a.n_cats; ++k) {
      a.mapA[k * a.threads + t] = s.a(k);
      a.mapB[k * a.threads + t] = s.b(k);
      a.mapN[k * a.threads + t] = s.n(k);
    }
}

// C2: exclusive scan of the per-thread maps of one category (block = category)
__global__ void __launch_bounds__(1024) c2_scan(CalibArgs a, int which) {
  __shared__ double sA[1024], sB[1024];
  __shared__ unsigned long long sN[1024];
  const uint32_t k = blockIdx.x;
  double *A = (which ? a.sigA : a.mapA) + (uint64_t)k * a.threads;
  double *B = (which ? a.sigB : a.mapB) + (uint64_t)k * a.threads;
  uint32_t *N = a.mapN + (uint64_t)k * a.threads;
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  const uint64_t per = (a.threads + T - 1) / T;
  const uint64_t lo = umin(a.threads, tid * per), hi = umin(a.threads, lo + per);
  // compose my run: later maps on the outside
  double ra = 1.0, rb = 0.0;
  unsigned long long rn = 0;
  for (uint64_t j = lo; j < hi; ++j) {
    rb = __dadd_rn(__dmul_rn(A[j], rb), B[j]);
    ra = __dmul_rn(A[j], ra);
    rn += N[j];
  }
  sA[tid] = ra; sB[tid] = rb; sN[tid] = rn;
  __syncthreads();
  if (tid == 0) {   // exclusive scan over the 1,024 run maps (cheap, sequential)
    double pa = 1.0, pb = 0.0;
    unsigned long long pn = 0;
    for (uint32_t j = 0; j < T; ++j) {
      const double ja = sA[j], jb = sB[j];
      const unsigned long long jn = sN[j];
      sA[j] = pa; sB[j] = pb; sN[j] = pn;
      pb = __dadd_rn(__dmul_rn(ja, pb), jb);
      pa = __dmul_rn(ja, pa);
      pn += jn;
    }
    // final state = the total composed map applied to the initial state
    if (which == 0) { a.totA[k] = __dadd_rn(__dmul_rn(pa, a.c0[k]), pb); a.totN[k] = pn; }
    else { a.totSA[k] = __dadd_rn(__dmul_rn(pa, a.s0[k]), pb); }
  }
  __syncthreads();
  double pa = sA[tid], pb = sB[tid];
  unsigned long long pn = sN[tid];
  for (uint64_t j = lo; j < hi; ++j) {          // rewrite as exclusive prefixes
    const double ja = A[j], jb = B[j];
    const uint32_t jn = N[j];
    A[j] = pa; B[j] = pb;
    if (which == 0) a.preN[(uint64_t)k * a.threads + j] = pn;
    pb = __dadd_rn(__dmul_rn(ja, pb), jb);
    pa = __dmul_rn(ja, pa);
    pn += jn;
  }
}

// C3: replay each segment from its c_hat prefix; sigma maps; c_hat snapshot
__global__ void __launch_bounds__(kCalBlock) c3_replay(CalibArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  MapSmem s = map_smem(smem, a.n_cats);            // a/b: sigma map, c state in cst
  double *cst = reinterpret_cast<double *>(s.cnt + a.n_cats * kCalBlock);
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < a.threads;
  for (uint32_t k = 0; k < a.n_cats; ++k) {
    s.a(k) = 1.0; s.b(k) = 0.0;
    s.n(k) = live ? (uint32_t)0 : 0u;
    cst[k * kCalBlock + threadIdx.x] =
        live ? __dadd_rn(__dmul_rn(a.mapA[k * a.threads + t], a.c0[k]), a.mapB[k * a.threads + t]) : 0.0;
  }
  uint64_t lo, hi;
  segment(a, t, lo, hi);
  const double w = __dsub_rn(1.0, a.beta);
  for (uint64_t i = lo; i < hi; ++i) {
    const Obs o = load_obs(a, i);
    if (!o.valid) continue;
    double &c = cst[o.k * kCalBlock + threadIdx.x];
    const double prev = c;
    c = __dadd_rn(__dmul_rn(a.beta, prev), __dmul_rn(w, o.c));
    const double d = fabs(__dsub_rn(o.c, prev));
    s.a(o.k) = __dmul_rn(a.beta, s.a(o.k));
    s.b(o.k) = __dadd_rn(__dmul_rn(a.beta, s.b(o.k)), __dmul_rn(w, d));
    const uint32_t seen = ++s.n(o.k);
    if (a.preN[(uint64_t)o.k * a.threads + t] + seen == a.snap_at) {
      a.snap_c[o.k] = c;
      a.snap_thread[o.k] = t;
    }
  }
  if (live)
    for (uint32_t k = 0; k < a.n_cats; ++k) {
      a.sigA[k * a.threads + t] = s.a(k);
      a.sigB[k * a.threads + t] = s.b(k);
    }
}

// C4: sigma snapshot -- replay the segment that holds each category's snapshot
__global__ void __launch_bounds__(32) c4_snap(CalibArgs a) {
  const uint32_t k = blockIdx.x;
  if (threadIdx.x != 0 || a.snap_thread[k] == ~0ull) return;
  const uint64_t t = a.snap_thread[k];
  double c = __dadd_rn(__dmul_rn(a.mapA[k * a.threads + t], a.c0[k]), a.mapB[k * a.threads + t]);
  double sg = __dadd_rn(__dmul_rn(a.sigA[k * a.threads + t], a.s0[k]), a.sigB[k * a.threads + t]);
  uint64_t lo, hi;
  segment(a, t, lo, hi);
  const double w = __dsub_rn(1.0, a.beta);
  uint64_t seen = a.preN[(uint64_t)k * a.threads + t];
  for (uint64_t i = lo; i < hi; ++i) {
    const Obs o = load_obs(a, i);
    if (!o.valid || o.k != k) continue;
    const double prev = c;
    c = __dadd_rn(__dmul_rn(a.beta, prev), __dmul_rn(w, o.c));
    sg = __dadd_rn(__dmul_rn(a.beta, sg), __dmul_rn(w, fabs(__dsub_rn(o.c, prev))));
    if (++seen == a.snap_at) {
      a.snap_s[k] = sg;
      return;
    }
  }
}

}  // namespace

size_t calib_scratch_bytes(uint64_t threads, uint32_t n_cats) {
  // mapA, mapB, sigA, sigB (double), mapN (u32), preN (u64) per (category, thread)
  return (size_t)threads * n_cats * (8 * 4 + 4 + 8);
}

cudaError_t launch_calibrate(CalibArgs a, cudaStream_t s) {
  const size_t sm1 = (size_t)a.n_cats * kCalBlock * (8 * 2 + 4);
  const size_t sm3 = sm1 + (size_t)a.n_cats * kCalBlock * 8;
  cudaError_t e = cudaFuncSetAttribute(c1_maps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(c3_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)((a.threads + kCalBlock - 1) / kCalBlock);
  c1_maps<<<blocks, kCalBlock, sm1, s>>>(a);
  c2_scan<<<a.n_cats, 1024, 0, s>>>(a, 0);
  c3_replay<<<blocks, kCalBlock, sm3, s>>>(a);
  c2_scan<<<a.n_cats, 1024, 0, s>>>(a, 1);
  c4_snap<<<a.n_cats, 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace fp
