"""Synthetic request-length shapes (INPUT MODULE; no method arithmetic).

Each shape is a pair of 65,537-entry u32 inverse-CDF tables: one for the
prompt length L_in and one for the output budget L_out (`max_output_tokens`).
A request's routing key is L_total = L_in + L_out (PAPER.md Eq. `budget`,
P:425-429; "route on L_total").

Sampling a table with a 32-bit Philox word w (same rule in numpy, host C and
CUDA):  i = w >> 16, f = w & 0xFFFF,
        interp:   L = q[i] + (((q[i+1] - q[i]) * f) >> 16)   (u64 product)
        discrete: L = q[i]
Tables are built here once per shape from a stated distribution by integer
inverse-CDF search: q[i] = min{x integer : CDF(x) >= i / 65536}, q[65536] = cap.

The shape targets follow SURVEY.md §8(d) "Synthetic inputs" and the paper's
trace statements; `fit_shapes.py` reproduces the fitted numbers recorded in
DESIGN.md. Real traces are not available.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
from scipy import stats

LUT_LEVELS = 65536          # 2^16 quantile levels
LUT_SIZE = LUT_LEVELS + 1   # plus the cap entry


@dataclass(frozen=True)
class Table:
    q: np.ndarray           # uint32[LUT_SIZE], non-decreasing
    interp: bool


@dataclass(frozen=True)
class Shape:
    name: str
    t_in: Table
    t_out: Table
    notes: str = ""


@dataclass(frozen=True)
class Mixture:
    """Per-request component choice: comp = #{k : w2 >= cut[k]}."""
    name: str
    shapes: tuple
    cut: tuple = field(default_factory=tuple)   # u32 cumulative thresholds


def _inverse_cdf_table(cdf_on_grid: np.ndarray, interp: bool) -> Table:
    """cdf_on_grid[x] = P(X <= x) for x = 0..cap (cap = len-1)."""
    cap = len(cdf_on_grid) - 1
    cdf = np.maximum.accumulate(np.clip(cdf_on_grid, 0.0, 1.0))
    cdf[-1] = 1.0
    levels = np.arange(LUT_SIZE, dtype=np.float64) / LUT_LEVELS
    levels[0] = 1e-12          # q[0] = smallest value with positive mass
    q = np.searchsorted(cdf, levels, side="left").astype(np.int64)
    q = np.clip(q, 0, cap)
    q[-1] = cap
    return Table(q=q.astype(np.uint32), interp=interp)


def _grid(cap):
    return np.arange(cap + 1, dtype=np.float64)


def lognormal_cdf(x, mu, sigma):
    with np.errstate(divide="ignore"):
        return stats.norm.cdf((np.log(np.maximum(x, 1e-300)) - mu) / sigma)


def table_lognormal_ceil(mu, sigma, cap, lo=1) -> Table:
    """L = clamp(ceil(X), lo, cap), X ~ LogNormal(mu, sigma).  P(L <= x) = F(x)."""
    x = _grid(cap)
    cdf = lognormal_cdf(x, mu, sigma)
    cdf[: lo] = 0.0
    return _inverse_cdf_table(cdf, interp=True)


def table_discrete(values, weights) -> Table:
    values = np.asarray(values, dtype=np.int64)
    w = np.asarray(weights, dtype=np.float64)
    w = w / w.sum()
    cap = int(values.max())
    pmf = np.zeros(cap + 1)
    np.add.at(pmf, values, w)
    return _inverse_cdf_table(np.cumsum(pmf), interp=False)


def table_from_cdf(cdf_fn, cap, interp=True, lo=1) -> Table:
    x = _grid(cap)
    cdf = cdf_fn(x)
    cdf[: lo] = 0.0
    return _inverse_cdf_table(cdf, interp=interp)


# --------------------------------------------------------------------------
# Shape parameters (stated)
# --------------------------------------------------------------------------
# AZ (Azure / BurstGPT): L_in log-normal through P80 = 2,048 and P95 = 8,192
# ("80% of requests fit in 2K tokens and 95% fit in 8K"),
# capped at 65,536 ("tail extending to 64K").  L_out budget: 8-point
# power-of-two mix fitted (fit_shapes.py) so that alpha(L_total <= 1,024) ~ 0.35
# and alpha(L_total <= 8,192) ~ 0.80.
_Z80, _Z95 = stats.norm.ppf(0.80), stats.norm.ppf(0.95)
AZ_SIGMA = (np.log(8192.0) - np.log(2048.0)) / (_Z95 - _Z80)
AZ_MU = np.log(2048.0) - _Z80 * AZ_SIGMA
AZ_IN_CAP = 65536
AZ_OUT_VALUES = (64, 128, 256, 512, 1024, 2048, 4096, 8192)
AZ_OUT_WEIGHTS = (0.109, 0.078, 0.283, 0.109, 0.066, 0.140, 0.066, 0.149)

# LM (LMSYS-Chat-1M): L_in log-normal with mean 69.5,
# sigma_log = 1.0; L_out budget: with prob 1 - LM_P_UNSET a log-normal with
# mean 214.5, otherwise the client left max_tokens unset and the
# gateway fills a 16,384-token long-window default (stated assumption) so
# that alpha(8,192) ~ 0.68.
LM_SIGMA = 1.0
LM_MU = np.log(69.5) - 0.5 * LM_SIGMA ** 2
LM_IN_CAP = 32768
LM_OUT_MU = np.log(214.5) - 0.5
LM_OUT_CAP = 8192
LM_P_UNSET = 0.32
LM_UNSET_BUDGET = 16384

# SG (ServeGen): 0.9 LogNormal(median 400, sigma 1) + 0.1 Pareto(x_m 2,048,
# a 1.1), capped at 262,144 ("Pareto/log-normal mixture heavily
# concentrated below 2K"); parameters stated, not from the paper.  L_out:
# log-normal median 128, sigma 1, cap 4,096 (stated).
SG_W_LOGN, SG_MED, SG_SIGMA = 0.9, 400.0, 1.0
SG_XM, SG_A = 2048.0, 1.1
SG_IN_CAP = 262144
SG_OUT_MED, SG_OUT_SIGMA, SG_OUT_CAP = 128.0, 1.0, 4096

# MIX (C5): per-request component AZ 0.5 / LM 0.3 / SG 0.2.
MIX_WEIGHTS = (0.5, 0.3, 0.2)


@lru_cache(maxsize=None)
def shape_az() -> Shape:
    return Shape(
        "AZ",
        table_lognormal_ceil(AZ_MU, AZ_SIGMA, AZ_IN_CAP),
        table_discrete(AZ_OUT_VALUES, AZ_OUT_WEIGHTS),
        notes=f"L_in ~ ceil(LogNormal(mu={AZ_MU:.4f}, sigma={AZ_SIGMA:.4f})) cap 65536",
    )


@lru_cache(maxsize=None)
def shape_lm() -> Shape:
    def out_cdf(x):
        body = lognormal_cdf(x, LM_OUT_MU, 1.0)
        body[LM_OUT_CAP:] = 1.0
        c = (1.0 - LM_P_UNSET) * body
        c[LM_UNSET_BUDGET:] += LM_P_UNSET
        return c
    return Shape(
        "LM",
        table_lognormal_ceil(LM_MU, LM_SIGMA, LM_IN_CAP),
        table_from_cdf(out_cdf, LM_UNSET_BUDGET, interp=False),
    )


@lru_cache(maxsize=None)
def shape_sg() -> Shape:
    def in_cdf(x):
        logn = lognormal_cdf(x, np.log(SG_MED), SG_SIGMA)
        par = np.where(x >= SG_XM, 1.0 - (SG_XM / np.maximum(x, SG_XM)) ** SG_A, 0.0)
        return SG_W_LOGN * logn + (1.0 - SG_W_LOGN) * par
    return Shape(
        "SG",
        table_from_cdf(in_cdf, SG_IN_CAP, interp=True),
        table_lognormal_ceil(np.log(SG_OUT_MED), SG_OUT_SIGMA, SG_OUT_CAP),
    )


def _cuts(weights):
    c = np.cumsum(np.asarray(weights, dtype=np.float64))[:-1]
    return tuple(int(min(int(x * 2 ** 32), 2 ** 32 - 1)) for x in c)


SHAPES = {"AZ": shape_az, "LM": shape_lm, "SG": shape_sg}


def mixture(name: str) -> Mixture:
    """Single shapes are 1-component mixtures (component word unused)."""
    if name == "MIX":
        return Mixture("MIX", (shape_az(), shape_lm(), shape_sg()), _cuts(MIX_WEIGHTS))
    return Mixture(name, (SHAPES[name](),), ())


# --------------------------------------------------------------------------
# Raw request columns for token-budget estimation (NEXT-1; PAPER Eq. `budget`
# P:425-429 and Table 5). A request carries its body length |r| in
# bytes, its category k and max_output_tokens; the true prompt token count is
# L_in (the same L_in as the L_total trace, so L_total_true = L_in + L_out).
#   bytes = round(L_in * ratio),  ratio = c_k * noise,  fixed point 16.16:
#   bytes = (L_in * R[k][w3 >> 16] + 2^15) >> 16   (u64 product)
#   k     = #{j : (w3 & 0xFFFF) >= CAT_CUT[j]}
# c_k: Table 5 "True c_k"; category weights and the 10% CV
# log-normal noise are stated assumptions.
# --------------------------------------------------------------------------
CATEGORIES = ("prose", "code", "cjk", "mixed")
CAT_TRUE_RATIO = (4.48, 3.52, 2.01, 3.81)
CAT_WEIGHTS = (0.55, 0.20, 0.10, 0.15)           # stated
RATIO_CV = 0.10                                   # stated


def category_cuts16():
    c = np.cumsum(np.asarray(CAT_WEIGHTS, dtype=np.float64))[:-1]
    return tuple(int(round(x * 65536)) for x in c)


@lru_cache(maxsize=None)
def ratio_tables():
    """uint32 [n_cat][65536] per-request bytes-per-token ratio in 16.16 fixed point."""
    sig = np.sqrt(np.log(1.0 + RATIO_CV ** 2))
    z = stats.norm.ppf((np.arange(65536, dtype=np.float64) + 0.5) / 65536.0)
    noise = np.exp(sig * z - 0.5 * sig * sig)
    out = np.zeros((len(CAT_TRUE_RATIO), 65536), dtype=np.uint32)
    for k, c in enumerate(CAT_TRUE_RATIO):
        out[k] = np.round(c * noise * 65536.0).astype(np.uint32)
    return out


# --------------------------------------------------------------------------
# Arrival times (NEXT-4): Poisson arrivals ("Poisson arrivals") with
# stated burst phases. gap_i = G[w >> 16] * F[(i >> 20) & 7] >> 3 ns, where G
# is the exponential inverse CDF (mean 1e9 / rate ns, 16.16-free integer ns)
# and F = {8, 8, 8, 4, 8, 8, 2, 8} halves / quarters the gaps in two of
# every eight 2^20-request phases (2x / 4x bursts, stated); w is the first
# Philox word of counter (lo32 i, hi32 i, 1, 0). arrival_i = sum_{j <= i} gap_j.
# --------------------------------------------------------------------------
BURST_FACTORS = (8, 8, 8, 4, 8, 8, 2, 8)


def gap_table(rate_rps: float):
    u = (np.arange(65536, dtype=np.float64) + 0.5) / 65536.0
    return np.round(-np.log1p(-u) * (1e9 / rate_rps)).astype(np.uint32)
