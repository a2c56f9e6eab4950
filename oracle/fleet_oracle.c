/* ==========================================================================
 * oracle/fleet_oracle.c -- CPU ORACLE for the two-pool fleet-sizing sweep.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load or run this.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2604_08075_b200/, include/); neither side includes the other.
 *
 * It is the paper's definitions written out plainly, in the paper's order,
 * fp64 where the paper computes real numbers, u64 / u128 for byte and count
 * arithmetic. No blocking, no fusion, no reordering beyond the definitions.
 * Citations: P:n = /root/reference/PAPER.md line n (LaTeX source);
 * readings R1..R20 = DESIGN.md "Readings of the paper".
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp (x86-64 SSE2).
 * Every function below is pinned by tests/test_oracle_*.py -m "not gpu".
 * ========================================================================== */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ---- Eq. (1) `eq:kv-per-seq`, P:23-31 ------------------------------------
 * M_seq = 2 * n_l * n_h * d_h * b_dtype * C_max  (bytes, all GPUs of an
 * instance). Per token per GPU it is divided by the TP degree ("23.5 KB
 * per token per GPU"). */
uint64_t or_kv_bytes_per_seq(uint32_t n_l, uint32_t n_h, uint32_t d_h, uint32_t b,
                             uint64_t c_max) {
  u128 m = (u128)2 * n_l * n_h * d_h * b * c_max;
  return (uint64_t)m;
}

/* Per-token per-GPU KV bytes, exact quotient. Returns the remainder
 * through *rem so callers can see when tp does not divide the product. */
uint64_t or_kv_bytes_per_token_per_gpu(uint32_t n_l, uint32_t n_h, uint32_t d_h,
                                       uint32_t b, uint32_t tp, uint64_t *rem) {
  uint64_t tot = or_kv_bytes_per_seq(n_l, n_h, d_h, b, 1);
  if (rem) *rem = tot % tp;
  return tot / tp;
}

/* ---- Eq. (2) numerator with activation reserve, P:32-39, P:997-999 --------
 * budget = M_gpu * u - M_model - M_act, u = util_num / util_den (R9, a
 * rational so the result is an integer: floor(M_gpu * num / den)); clamped at
 * 0 when the weights do not fit. */
uint64_t or_kv_budget(uint64_t hbm, uint32_t u_num, uint32_t u_den, uint64_t weights_per_gpu,
                      uint64_t act_reserve) {
  u128 usable = ((u128)hbm * u_num) / u_den;
  u128 need = (u128)weights_per_gpu + act_reserve;
  if (usable <= need) return 0;
  return (uint64_t)(usable - need);
}

/* ---- Eq. (2) `eq:max-seqs`, P:32-39 ----------------------------------------
 * N_seq = floor(budget / M_seq_per_gpu), M_seq_per_gpu = M_seq / tp, computed
 * exactly as floor(budget * tp / M_seq) (R8: bytes are integers). */
uint64_t or_max_seqs(uint64_t budget, uint64_t m_seq_total, uint32_t tp) {
  if (m_seq_total == 0) return 0;
  return (uint64_t)(((u128)budget * tp) / m_seq_total);
}

/* ---- empirical CDF, "alpha = F(B_short)", closed right boundary (R1)
 * cnt[j]  = #{ i : L_i <= x_j }
 * mass[j] = sum_i L_i * [L_i <= x_j]
 * The literal double loop over (request, threshold). */
void or_count_le(const uint32_t *L, uint64_t n, const uint32_t *x, uint32_t nx,
                 uint64_t *cnt, uint64_t *mass) {
  for (uint32_t j = 0; j < nx; ++j) { cnt[j] = 0; mass[j] = 0; }
  int64_t nn = (int64_t)n;
#pragma omp parallel
  {
    uint64_t *c = (uint64_t *)calloc(nx ? nx : 1, sizeof(uint64_t));
    uint64_t *m = (uint64_t *)calloc(nx ? nx : 1, sizeof(uint64_t));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < nn; ++i) {
      uint32_t l = L[i];
      for (uint32_t j = 0; j < nx; ++j) {
        uint64_t le = (l <= x[j]) ? 1u : 0u;
        c[j] += le;
        m[j] += le * (uint64_t)l;
      }
    }
#pragma omp critical
    for (uint32_t j = 0; j < nx; ++j) { cnt[j] += c[j]; mass[j] += m[j]; }
    free(c);
    free(m);
  }
}

/* ---- Alg. 1 Route, applied literally to one request -----------
 * pool: 0 short, 1 long, 2 rejected. stage: 0 budget (step 2), 1 feasibility
 * (step 1), 2 final safety check, 3 rejection.
 * Rejection (L > C_max of the long pool, the largest window, R3)
 * is checked first. Step 3 (load-aware spillover) needs live queue
 * state and is out of scope for a static trace. */
int or_route(uint32_t L, uint32_t B, uint32_t c_short, uint32_t c_long, int *stage) {
  int p, st;
  if (L > c_long) { if (stage) *stage = 3; return 2; }          /* rejected         */
  if (L > c_short) { if (stage) *stage = 1; return 1; }         /* step 1    */
  if (L <= B) { p = 0; st = 0; } else { p = 1; st = 0; }         /* step 2    */
  /* step 3 spillover: out of scope */
  if (L > (p == 0 ? c_short : c_long)) { p = 1; st = 2; }        /* safety    */
  if (stage) *stage = st;
  return p;
}

/* route_batch semantics: decision byte = pool | stage << 2; counts[5] =
 * {n_short, n_long, n_reject, mass_short, mass_long}. */
void or_route_batch(const uint32_t *L, uint64_t n, uint32_t B, uint32_t c_short, uint32_t c_long,
                    uint8_t *decision, uint64_t counts[5]) {
  for (int k = 0; k < 5; ++k) counts[k] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    int st = 0;
    int p = or_route(L[i], B, c_short, c_long, &st);
    if (decision) decision[i] = (uint8_t)(p | (st << 2));
    counts[p] += 1;
    if (p == 0) counts[3] += L[i];
    if (p == 1) counts[4] += L[i];
  }
}

/* ---- one pool's instance count, Sec. 3 P:571-579 -------------------------
 * I = ceil(lambda_p / mu_p)  (G_homo = ceil(lambda / mu(C_H)); Eq. (6) G_dual
 * is the sum of two such ceilings). R13: lambda_p = 0 -> I = 0; lambda_p > 0
 * with N_seq = 0 or mu <= 0 -> the pool cannot be built (infeasible). A
 * quotient above 2^53 is not representable as an exact count -> infeasible. */
int or_pool_instances(double lam, double mu, uint64_t nseq, uint64_t *inst) {
  *inst = 0;
  if (lam == 0.0) return 1;
  if (nseq == 0 || !(mu > 0.0)) return 0;
  double x = lam / mu;
  if (!(x <= 9007199254740992.0)) return 0;
  *inst = (uint64_t)ceil(x);
  return 1;
}

/* ---- Eq. (7) `eq:savings`, P:581-590 -------------------------------------
 * predicted = alpha * (1 - 1/rho), rho = mu(C_S) / mu(C_H). */
double or_predicted_savings(double alpha, double rho) {
  return alpha * (1.0 - (1.0 / rho));
}

/* Annual cost = GPUs x $/GPU-hr x hours (R7). */
double or_cost(uint64_t gpus, double price, double hours) {
  double c = (double)gpus * price;
  c = c * hours;
  return c;
}

/* ---- candidate record (oracle's own layout) ------------------------------ */
enum { OR_VALID = 1, OR_FEASIBLE = 2, OR_HOMO_FEASIBLE = 4 };
typedef struct {
  uint32_t index, model, gpu, b_short, c_short, c_long, flags, _pad;
  uint64_t nseq_short, nseq_long;
  uint64_t n_short, n_long, n_reject, mass_short, mass_long;
  uint64_t inst_short, inst_long, inst_homo, gpus_dual, gpus_homo;
  double alpha, rho, predicted_savings, savings, cost_dual, cost_homo;
  double occupancy_short, occupancy_long;
} or_candidate;

uint32_t or_candidate_size(void) { return (uint32_t)sizeof(or_candidate); }

static uint32_t find_u32(const uint32_t *a, uint32_t n, uint32_t v) {
  for (uint32_t i = 0; i < n; ++i)
    if (a[i] == v) return i;
  return UINT32_MAX;
}

/* ---- the whole sweep ------------------------------------------------------
 * Inputs (flat arrays, all host):
 *   arch[m*4 + {0,1,2,3}]          = n_l, n_h, d_h, b_dtype of model m
 *   gpu_u64[g*4 + {0,1,2,3}]       = hbm, util_num, util_den, activation reserve
 *   gpu_price[g]                   = $ per GPU-hour
 *   deploy[(m*G+g)*3 + {0,1,2}]    = tp, weight bytes per GPU, GPUs per instance
 *   grid b[n_b], cs[n_cs] (n_cs == 0 -> C_S = B, R16), cl[n_cl]
 *   windows[n_w], mu[(m*G+g)*n_w + w] requests/s per instance (R5: data)
 * Candidate order (m, g, C_L, C_S, B), B fastest (R12). Returns 0, or
 * 1 for an empty trace, 2 for a window missing from `windows`.
 * out (nullable) receives every candidate; best[m] the per-model argmin of
 * cost_dual over feasible candidates, strict '<' so ties keep the lowest
 * index (R12); index = UINT32_MAX when a model has no feasible candidate. */
int or_sweep(const uint32_t *L, uint64_t n, uint32_t n_models, const uint32_t *arch,
             uint32_t n_gpus, const uint64_t *gpu_u64, const double *gpu_price,
             const uint64_t *deploy, const uint32_t *b, uint32_t n_b, const uint32_t *cs,
             uint32_t n_cs, const uint32_t *cl, uint32_t n_cl, const uint32_t *windows,
             uint32_t n_w, const double *mu, double rate, double hours, or_candidate *out,
             or_candidate *best) {
  if (n == 0) return 1;
  /* counts at every threshold value a candidate uses: B and C_L */
  uint32_t nx = n_b + n_cl;
  uint32_t *x = (uint32_t *)malloc(sizeof(uint32_t) * nx);
  uint64_t *cnt = (uint64_t *)malloc(sizeof(uint64_t) * nx);
  uint64_t *mass = (uint64_t *)malloc(sizeof(uint64_t) * nx);
  for (uint32_t k = 0; k < n_b; ++k) x[k] = b[k];
  for (uint32_t k = 0; k < n_cl; ++k) x[n_b + k] = cl[k];
  or_count_le(L, n, x, nx, cnt, mass);

  uint32_t n_cs_eff = n_cs ? n_cs : 1;
  for (uint32_t m = 0; m < n_models; ++m) {
    or_candidate bm;
    memset(&bm, 0, sizeof bm);
    bm.index = UINT32_MAX;
    bm.model = m;
    bm.cost_dual = INFINITY;
    bm.cost_homo = INFINITY;
    int have = 0;
    for (uint32_t g = 0; g < n_gpus; ++g)
      for (uint32_t l = 0; l < n_cl; ++l)
        for (uint32_t s = 0; s < n_cs_eff; ++s)
          for (uint32_t k = 0; k < n_b; ++k) {
            uint64_t idx = ((((uint64_t)m * n_gpus + g) * n_cl + l) * n_cs_eff + s) * n_b + k;
            or_candidate c;
            memset(&c, 0, sizeof c);
            c.index = (uint32_t)idx;
            c.model = m;
            c.gpu = g;
            c.b_short = b[k];
            c.c_short = n_cs ? cs[s] : b[k];
            c.c_long = cl[l];
            c.cost_dual = INFINITY;
            c.cost_homo = INFINITY;
            /* validity: B <= C_S <= C_L (R16) */
            if (c.b_short <= c.c_short && c.c_short <= c.c_long) {
              const uint64_t *dp = deploy + ((uint64_t)m * n_gpus + g) * 3;
              uint32_t tp = (uint32_t)dp[0];
              uint64_t wpg = dp[1], gpi = dp[2];
              const uint64_t *gu = gpu_u64 + (uint64_t)g * 4;
              const uint32_t *ar = arch + (uint64_t)m * 4;
              uint32_t ws = find_u32(windows, n_w, c.c_short);
              uint32_t wl = find_u32(windows, n_w, c.c_long);
              if (ws == UINT32_MAX || wl == UINT32_MAX) {
                free(x); free(cnt); free(mass);
                return 2;
              }
              double mu_s = mu[((uint64_t)m * n_gpus + g) * n_w + ws];
              double mu_l = mu[((uint64_t)m * n_gpus + g) * n_w + wl];

              /* routing counts from the CDF (Alg. 1 steps 1-2 + rejection, R1-R3) */
              uint64_t n_s = cnt[k], n_sl = cnt[n_b + l];
              c.n_short = n_s;
              c.n_long = n_sl - n_s;
              c.n_reject = n - n_sl;
              c.mass_short = mass[k];
              c.mass_long = mass[n_b + l] - mass[k];

              /* Eq. (1)-(2) per pool window */
              uint64_t budget = or_kv_budget(gu[0], (uint32_t)gu[1], (uint32_t)gu[2], wpg, gu[3]);
              c.nseq_short = or_max_seqs(budget, or_kv_bytes_per_seq(ar[0], ar[1], ar[2], ar[3], c.c_short), tp);
              c.nseq_long = or_max_seqs(budget, or_kv_bytes_per_seq(ar[0], ar[1], ar[2], ar[3], c.c_long), tp);

              /* loads: alpha = F(B); rejected traffic is in no pool (R3) */
              c.alpha = (double)n_s / (double)n;
              double lam_s = c.alpha * rate;
              double lam_l = ((double)c.n_long / (double)n) * rate;
              double lam_h = ((double)n_sl / (double)n) * rate;

              /* Sec. 3: G_dual (Eq. 6) and G_homo at C_H = C_L */
              int ok_s = or_pool_instances(lam_s, mu_s, c.nseq_short, &c.inst_short);
              int ok_l = or_pool_instances(lam_l, mu_l, c.nseq_long, &c.inst_long);
              int ok_h = or_pool_instances(lam_h, mu_l, c.nseq_long, &c.inst_homo);
              int ok_d = ok_s && ok_l;
              if (!ok_d) { c.inst_short = 0; c.inst_long = 0; }
              c.gpus_dual = gpi * (c.inst_short + c.inst_long);
              c.gpus_homo = gpi * c.inst_homo;
              c.cost_dual = ok_d ? or_cost(c.gpus_dual, gpu_price[g], hours) : INFINITY;
              c.cost_homo = ok_h ? or_cost(c.gpus_homo, gpu_price[g], hours) : INFINITY;
              c.savings = (ok_d && ok_h && c.gpus_homo > 0)
                              ? ((double)c.gpus_homo - (double)c.gpus_dual) / (double)c.gpus_homo
                              : 0.0;
              /* Eq. (7): rho = mu(C_S) / mu(C_H), predicted = alpha (1 - 1/rho) */
              c.rho = (mu_s > 0.0 && mu_l > 0.0) ? mu_s / mu_l : 0.0;
              c.predicted_savings = (c.rho > 0.0) ? or_predicted_savings(c.alpha, c.rho) : 0.0;
              /* occupancy = token mass / reserved tokens (R20) */
              c.occupancy_short = c.n_short ? (double)c.mass_short / ((double)c.n_short * (double)c.c_short) : 0.0;
              c.occupancy_long = c.n_long ? (double)c.mass_long / ((double)c.n_long * (double)c.c_long) : 0.0;
              c.flags = OR_VALID | (ok_d ? OR_FEASIBLE : 0) | (ok_h ? OR_HOMO_FEASIBLE : 0);
            }
            if (out) out[idx] = c;
            if ((c.flags & OR_FEASIBLE) && (!have || c.cost_dual < bm.cost_dual)) {
              bm = c;
              have = 1;
            }
          }
    best[m] = bm;
  }
  free(x);
  free(cnt);
  free(mass);
  return 0;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the OpenMP loops (bench.py's single-thread timing). */
void or_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ==========================================================================
 * Token-budget estimation (NEXT-1; TEST INFRASTRUCTURE like the rest).
 * ========================================================================== */

/* Eq. (5) `eq:conservative` P:453-457 / Alg. 1 line P:494:
 *   c* = c_hat_k - gamma * sigma_hat_k,
 * bounded below by c_floor > 0 (the paper does not bound it; DESIGN R22). */
double or_route_ratio(double c_hat, double sigma, double gamma, double c_floor) {
  double t = gamma * sigma;
  double c = c_hat - t;
  if (!(c >= c_floor)) c = c_floor;
  return c;
}

/* Eq. (3) `eq:budget` P:425-429 / Alg. 1 line P:496:
 *   L_total = ceil(|r| / c*) + max_output_tokens, saturating at 2^32 - 1. */
uint32_t or_estimate_one(uint32_t bytes, uint32_t max_out, double cstar) {
  double lin = ceil((double)bytes / cstar);
  if (!(lin < 4294967296.0)) return 0xFFFFFFFFu;
  uint64_t t = (uint64_t)lin + (uint64_t)max_out;
  return t > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)t;
}

/* Per request: category k (k >= n_cats -> the last category, the "mixed /
 * other" bucket, R23), c* from the frozen snapshot, then L_total. */
void or_estimate(const uint32_t *bytes, const uint32_t *max_out, const uint8_t *cat, uint64_t n,
                 const double *c_hat, const double *sigma, uint32_t n_cats, double gamma,
                 double c_floor, uint32_t *out) {
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t k = cat[i] < n_cats ? cat[i] : n_cats - 1;
    double cs = or_route_ratio(c_hat[k], sigma[k], gamma, c_floor);
    out[i] = or_estimate_one(bytes[i], max_out[i], cs);
  }
}

/* Alg. 1 on the estimates plus Table 5's mis-route count (P:925-927:
 * "sending a request to a pool that cannot serve it"): a request routed to
 * pool p whose TRUE total (true_prompt_tokens + max_output_tokens) exceeds
 * C_max(p). misroute[0] = short pool, misroute[1] = long pool. */
void or_route_batch_est(const uint32_t *bytes, const uint32_t *max_out, const uint8_t *cat,
                        const uint32_t *true_prompt, uint64_t n, const double *c_hat,
                        const double *sigma, uint32_t n_cats, double gamma, double c_floor,
                        uint32_t B, uint32_t c_short, uint32_t c_long, uint8_t *decision,
                        uint32_t *l_total, uint64_t counts[5], uint64_t misroute[2]) {
  for (int k = 0; k < 5; ++k) counts[k] = 0;
  misroute[0] = misroute[1] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t k = cat[i] < n_cats ? cat[i] : n_cats - 1;
    double cs = or_route_ratio(c_hat[k], sigma[k], gamma, c_floor);
    uint32_t L = or_estimate_one(bytes[i], max_out[i], cs);
    int st = 0;
    int p = or_route(L, B, c_short, c_long, &st);
    if (decision) decision[i] = (uint8_t)(p | (st << 2));
    if (l_total) l_total[i] = L;
    counts[p] += 1;
    if (p == 0) counts[3] += L;
    if (p == 1) counts[4] += L;
    if (true_prompt) {
      uint64_t t = (uint64_t)true_prompt[i] + max_out[i];
      if (p == 0 && t > c_short) misroute[0] += 1;
      if (p == 1 && t > c_long) misroute[1] += 1;
    }
  }
}

/* ==========================================================================
 * NEXT-2: three pools ("additional pools (e.g. 4K/16K/64K) yield
 * only marginal incremental savings (~2%)"). TEST INFRASTRUCTURE.
 * Pools 1, 2, 3 with windows C1 = B1 < C2 = B2 <= C3 = C_L (the Fig. 6
 * convention C_S = B for the inner pools, R16). Alg. 1 generalised: a request
 * goes to the first pool whose threshold it meets (L <= B1, else L <= B2,
 * else L <= C_L), otherwise it is rejected (R3). Each pool is sized as in
 * Sec. 3: I_i = ceil(lambda_i / mu(C_i)), lambda_i = (n_i / N) lambda.
 * ========================================================================== */
typedef struct {
  uint32_t index, model, gpu, b1, b2, c_long, flags, _pad;
  uint64_t n1, n2, n3, n_reject;
  uint64_t nseq1, nseq2, nseq3;
  uint64_t inst1, inst2, inst3, inst_homo, gpus, gpus_homo;
  double cost, cost_homo, savings;
} or_pool3;

uint32_t or_pool3_size(void) { return (uint32_t)sizeof(or_pool3); }

/* Candidate order (m, g, C_L, pair), pairs (i, j) of B-grid indices with
 * i < j in lexicographic order; valid iff b[i] < b[j] <= C_L. */
int or_sweep3(const uint32_t *L, uint64_t n, uint32_t n_models, const uint32_t *arch, uint32_t n_gpus,
              const uint64_t *gpu_u64, const double *gpu_price, const uint64_t *deploy, const uint32_t *b,
              uint32_t n_b, const uint32_t *cl, uint32_t n_cl, const uint32_t *windows, uint32_t n_w,
              const double *mu, double rate, double hours, or_pool3 *out, or_pool3 *best) {
  if (n == 0) return 1;
  uint32_t nx = n_b + n_cl;
  uint32_t *x = (uint32_t *)malloc(sizeof(uint32_t) * nx);
  uint64_t *cnt = (uint64_t *)malloc(sizeof(uint64_t) * nx);
  uint64_t *mass = (uint64_t *)malloc(sizeof(uint64_t) * nx);
  for (uint32_t k = 0; k < n_b; ++k) x[k] = b[k];
  for (uint32_t k = 0; k < n_cl; ++k) x[n_b + k] = cl[k];
  or_count_le(L, n, x, nx, cnt, mass);
  uint64_t n_pairs = (uint64_t)n_b * (n_b - 1) / 2;
  int rc = 0;
  for (uint32_t m = 0; m < n_models && !rc; ++m) {
    or_pool3 bm;
    memset(&bm, 0, sizeof bm);
    bm.index = UINT32_MAX;
    bm.model = m;
    bm.cost = bm.cost_homo = INFINITY;
    int have = 0;
    for (uint32_t g = 0; g < n_gpus && !rc; ++g)
      for (uint32_t l = 0; l < n_cl && !rc; ++l) {
        uint64_t p = 0;
        for (uint32_t i = 0; i < n_b; ++i)
          for (uint32_t j = i + 1; j < n_b; ++j, ++p) {
            uint64_t idx = (((uint64_t)m * n_gpus + g) * n_cl + l) * n_pairs + p;
            or_pool3 c;
            memset(&c, 0, sizeof c);
            c.index = (uint32_t)idx;
            c.model = m;
            c.gpu = g;
            c.b1 = b[i];
            c.b2 = b[j];
            c.c_long = cl[l];
            c.cost = c.cost_homo = INFINITY;
            if (c.b1 < c.b2 && c.b2 <= c.c_long) {
              const uint64_t *dp = deploy + ((uint64_t)m * n_gpus + g) * 3;
              uint32_t tp = (uint32_t)dp[0];
              uint64_t wpg = dp[1], gpi = dp[2];
              const uint64_t *gu = gpu_u64 + (uint64_t)g * 4;
              const uint32_t *ar = arch + (uint64_t)m * 4;
              uint32_t w1 = find_u32(windows, n_w, c.b1), w2 = find_u32(windows, n_w, c.b2);
              uint32_t w3 = find_u32(windows, n_w, c.c_long);
              if (w1 == UINT32_MAX || w2 == UINT32_MAX || w3 == UINT32_MAX) { rc = 2; break; }
              const double *mg = mu + ((uint64_t)m * n_gpus + g) * n_w;
              /* first-fit routing counts from the CDF */
              uint64_t c1 = cnt[i], c2 = cnt[j], c3 = cnt[n_b + l];
              c.n1 = c1;
              c.n2 = c2 - c1;
              c.n3 = c3 - c2;
              c.n_reject = n - c3;
              uint64_t budget = or_kv_budget(gu[0], (uint32_t)gu[1], (uint32_t)gu[2], wpg, gu[3]);
              c.nseq1 = or_max_seqs(budget, or_kv_bytes_per_seq(ar[0], ar[1], ar[2], ar[3], c.b1), tp);
              c.nseq2 = or_max_seqs(budget, or_kv_bytes_per_seq(ar[0], ar[1], ar[2], ar[3], c.b2), tp);
              c.nseq3 = or_max_seqs(budget, or_kv_bytes_per_seq(ar[0], ar[1], ar[2], ar[3], c.c_long), tp);
              double lam1 = ((double)c.n1 / (double)n) * rate;
              double lam2 = ((double)c.n2 / (double)n) * rate;
              double lam3 = ((double)c.n3 / (double)n) * rate;
              double lamh = ((double)c3 / (double)n) * rate;
              int ok1 = or_pool_instances(lam1, mg[w1], c.nseq1, &c.inst1);
              int ok2 = or_pool_instances(lam2, mg[w2], c.nseq2, &c.inst2);
              int ok3 = or_pool_instances(lam3, mg[w3], c.nseq3, &c.inst3);
              int okh = or_pool_instances(lamh, mg[w3], c.nseq3, &c.inst_homo);
              int ok = ok1 && ok2 && ok3;
              if (!ok) { c.inst1 = c.inst2 = c.inst3 = 0; }
              c.gpus = gpi * (c.inst1 + c.inst2 + c.inst3);
              c.gpus_homo = gpi * c.inst_homo;
              c.cost = ok ? or_cost(c.gpus, gpu_price[g], hours) : INFINITY;
              c.cost_homo = okh ? or_cost(c.gpus_homo, gpu_price[g], hours) : INFINITY;
              c.savings = (ok && okh && c.gpus_homo > 0)
                              ? ((double)c.gpus_homo - (double)c.gpus) / (double)c.gpus_homo
                              : 0.0;
              c.flags = OR_VALID | (ok ? OR_FEASIBLE : 0) | (okh ? OR_HOMO_FEASIBLE : 0);
            }
            if (out) out[idx] = c;
            if ((c.flags & OR_FEASIBLE) && (!have || c.cost < bm.cost)) {
              bm = c;
              have = 1;
            }
          }
      }
    best[m] = bm;
  }
  free(x);
  free(cnt);
  free(mass);
  return rc;
}

/* ==========================================================================
 * NEXT-3: calibration replay -- Alg. 1 OnResponse with Eq. (4)
 * `eq:ema` applied to a feedback stream in arrival order.
 * TEST INFRASTRUCTURE.
 *   c_obs = |r| / usage.prompt_tokens
 *   c_hat_k <- beta c_hat_k + (1 - beta) c_obs                    (Eq. ema)
 *   sigma_k <- beta sigma_k + (1 - beta) |c_obs - c_hat_k(before)| (R26)
 * Feedback with prompt_tokens == 0 is discarded; categories >= n_cats
 * use the last category (R23). The state after the snap_at-th observation of
 * each category is recorded (Table 5 reports n = 50).
 * ========================================================================== */
void or_calibrate(const uint32_t *bytes, const uint32_t *tokens, const uint8_t *cat, uint64_t n,
                  uint32_t n_cats, double beta, const double *c0, const double *s0, double *c_hat,
                  double *sigma, uint64_t *n_obs, uint64_t snap_at, double *snap_c, double *snap_s) {
  for (uint32_t k = 0; k < n_cats; ++k) {
    c_hat[k] = c0[k];
    sigma[k] = s0[k];
    n_obs[k] = 0;
    if (snap_c) snap_c[k] = NAN;
    if (snap_s) snap_s[k] = NAN;
  }
  const double w = 1.0 - beta;
  for (uint64_t i = 0; i < n; ++i) {
    if (tokens[i] == 0) continue;
    uint32_t k = cat[i] < n_cats ? cat[i] : n_cats - 1;
    double obs = (double)bytes[i] / (double)tokens[i];
    double prev = c_hat[k];
    double t1 = beta * prev;
    double t2 = w * obs;
    c_hat[k] = t1 + t2;
    double u1 = beta * sigma[k];
    double u2 = w * fabs(obs - prev);
    sigma[k] = u1 + u2;
    n_obs[k] += 1;
    if (n_obs[k] == snap_at) {
      if (snap_c) snap_c[k] = c_hat[k];
      if (snap_s) snap_s[k] = sigma[k];
    }
  }
}

/* ==========================================================================
 * NEXT-4: peak-window provisioning ("transient overload ... during
 * traffic bursts"). TEST INFRASTRUCTURE.
 * Arrival times split the trace into windows w = floor(arrival_ns / W). For
 * each candidate, every pool is sized for its busiest window instead of the
 * mean rate: lambda_p = max_w n_p(w) * (1e9 / W), I_p = ceil(lambda_p / mu_p)
 * (Sec. 3 sizing; R27). Same candidate grid and flat order as or_sweep.
 * ========================================================================== */
typedef struct {
  uint32_t index, model, gpu, b_short, c_short, c_long, flags, _pad;
  uint64_t peak_short, peak_long, peak_homo;
  uint64_t inst_short, inst_long, inst_homo, gpus_dual, gpus_homo;
  double lambda_short, lambda_long, lambda_homo, cost_dual, cost_homo, savings;
} or_peak;

uint32_t or_peak_size(void) { return (uint32_t)sizeof(or_peak); }

int or_sweep_peak(const uint32_t *L, const uint64_t *arrival_ns, uint64_t n, uint64_t window_ns,
                  uint32_t n_models, const uint32_t *arch, uint32_t n_gpus, const uint64_t *gpu_u64,
                  const double *gpu_price, const uint64_t *deploy, const uint32_t *b, uint32_t n_b,
                  const uint32_t *cs, uint32_t n_cs, const uint32_t *cl, uint32_t n_cl, const uint32_t *windows,
                  uint32_t n_w, const double *mu, double hours, or_peak *out, or_peak *best) {
  if (n == 0 || window_ns == 0) return 1;
  uint64_t nwin = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (arrival_ns[i] / window_ns + 1 > nwin) nwin = arrival_ns[i] / window_ns + 1;
  /* per window, per threshold value (B and C_L): #{L <= x} by definition */
  uint32_t nx = n_b + n_cl;
  uint64_t *cnt = (uint64_t *)calloc((size_t)nwin * nx, sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t w = arrival_ns[i] / window_ns;
    for (uint32_t j = 0; j < nx; ++j) {
      uint32_t x = j < n_b ? b[j] : cl[j - n_b];
      cnt[w * nx + j] += (L[i] <= x) ? 1u : 0u;
    }
  }
  const double inv_w = 1e9 / (double)window_ns;   /* windows per second */
  uint32_t n_cs_eff = n_cs ? n_cs : 1;
  int rc = 0;
  for (uint32_t m = 0; m < n_models && !rc; ++m) {
    or_peak bm;
    memset(&bm, 0, sizeof bm);
    bm.index = UINT32_MAX;
    bm.model = m;
    bm.cost_dual = bm.cost_homo = INFINITY;
    int have = 0;
    for (uint32_t g = 0; g < n_gpus && !rc; ++g)
      for (uint32_t l = 0; l < n_cl && !rc; ++l)
        for (uint32_t s = 0; s < n_cs_eff && !rc; ++s)
          for (uint32_t k = 0; k < n_b; ++k) {
            uint64_t idx = ((((uint64_t)m * n_gpus + g) * n_cl + l) * n_cs_eff + s) * n_b + k;
            or_peak c;
            memset(&c, 0, sizeof c);
            c.index = (uint32_t)idx;
            c.model = m;
            c.gpu = g;
            c.b_short = b[k];
            c.c_short = n_cs ? cs[s] : b[k];
            c.c_long = cl[l];
            c.cost_dual = c.cost_homo = INFINITY;
            if (c.b_short <= c.c_short && c.c_short <= c.c_long) {
              const uint64_t *dp = deploy + ((uint64_t)m * n_gpus + g) * 3;
              uint32_t tp = (uint32_t)dp[0];
              uint64_t wpg = dp[1], gpi = dp[2];
              const uint64_t *gu = gpu_u64 + (uint64_t)g * 4;
              const uint32_t *ar = arch + (uint64_t)m * 4;
              uint32_t ws = find_u32(windows, n_w, c.c_short), wl = find_u32(windows, n_w, c.c_long);
              if (ws == UINT32_MAX || wl == UINT32_MAX) { rc = 2; break; }
              const double *mg = mu + ((uint64_t)m * n_gpus + g) * n_w;
              for (uint64_t w = 0; w < nwin; ++w) {
                uint64_t s_ = cnt[w * nx + k], sl = cnt[w * nx + n_b + l];
                if (s_ > c.peak_short) c.peak_short = s_;
                if (sl - s_ > c.peak_long) c.peak_long = sl - s_;
                if (sl > c.peak_homo) c.peak_homo = sl;
              }
              uint64_t budget = or_kv_budget(gu[0], (uint32_t)gu[1], (uint32_t)gu[2], wpg, gu[3]);
              uint64_t nseq_s = or_max_seqs(budget, or_kv_bytes_per_seq(ar[0], ar[1], ar[2], ar[3], c.c_short), tp);
              uint64_t nseq_l = or_max_seqs(budget, or_kv_bytes_per_seq(ar[0], ar[1], ar[2], ar[3], c.c_long), tp);
              c.lambda_short = (double)c.peak_short * inv_w;
              c.lambda_long = (double)c.peak_long * inv_w;
              c.lambda_homo = (double)c.peak_homo * inv_w;
              int ok_s = or_pool_instances(c.lambda_short, mg[ws], nseq_s, &c.inst_short);
              int ok_l = or_pool_instances(c.lambda_long, mg[wl], nseq_l, &c.inst_long);
              int ok_h = or_pool_instances(c.lambda_homo, mg[wl], nseq_l, &c.inst_homo);
              int ok_d = ok_s && ok_l;
              if (!ok_d) { c.inst_short = 0; c.inst_long = 0; }
              c.gpus_dual = gpi * (c.inst_short + c.inst_long);
              c.gpus_homo = gpi * c.inst_homo;
              c.cost_dual = ok_d ? or_cost(c.gpus_dual, gpu_price[g], hours) : INFINITY;
              c.cost_homo = ok_h ? or_cost(c.gpus_homo, gpu_price[g], hours) : INFINITY;
              c.savings = (ok_d && ok_h && c.gpus_homo > 0)
                              ? ((double)c.gpus_homo - (double)c.gpus_dual) / (double)c.gpus_homo
                              : 0.0;
              c.flags = OR_VALID | (ok_d ? OR_FEASIBLE : 0) | (ok_h ? OR_HOMO_FEASIBLE : 0);
            }
            if (out) out[idx] = c;
            if ((c.flags & OR_FEASIBLE) && (!have || c.cost_dual < bm.cost_dual)) {
              bm = c;
              have = 1;
            }
          }
    best[m] = bm;
  }
  free(cnt);
  return rc;
}
