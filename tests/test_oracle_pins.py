"""Pins for the CPU oracle (-m "not gpu").

Each test pins an oracle function to something other than itself: a value
printed in the paper (tests/golden/paper_pins.json, each with its citation),
a closed form, a definition checked by brute force, or an invariant. They are
chosen so that a dropped term, a wrong sign/index or a transposed operand in
oracle/fleet_oracle.c fails at least one of them.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle

# ---------------------------------------------------------------- Eq. (1) ----


def test_kv_per_token_qwen3(golden):
    g = golden["kv_per_token_per_gpu_qwen3"]
    a = g["args"]
    q, rem = oracle.kv_bytes_per_token_per_gpu(a["n_l"], a["n_h"], a["d_h"], a["b"], a["tp"])
    assert (q, rem) == (g["bytes"], 0)
    assert q / 1024 == g["kib"]          # "23.5 KB" is KiB (reading R8)


def test_kv_per_token_llama70b(golden):
    g = golden["kv_per_token_llama70b_tp1"]
    a = g["args"]
    assert oracle.kv_bytes_per_token_per_gpu(a["n_l"], a["n_h"], a["d_h"], a["b"], a["tp"]) == (g["bytes"], 0)


def test_kv_unit_args():
    # unit arguments -> 2 bytes (the factor 2 is K and V)
    assert oracle.kv_bytes_per_seq(1, 1, 1, 1, 1) == 2


@given(st.integers(1, 200), st.integers(1, 64), st.integers(1, 256), st.sampled_from([1, 2, 4]),
       st.integers(1, 1 << 20))
@settings(max_examples=200, deadline=None)
def test_kv_per_seq_is_linear_in_each_symbol(n_l, n_h, d_h, b, c):
    # Eq. (1) is a product of its symbols: doubling any one doubles M_seq.
    base = oracle.kv_bytes_per_seq(n_l, n_h, d_h, b, c)
    assert oracle.kv_bytes_per_seq(2 * n_l, n_h, d_h, b, c) == 2 * base
    assert oracle.kv_bytes_per_seq(n_l, 2 * n_h, d_h, b, c) == 2 * base
    assert oracle.kv_bytes_per_seq(n_l, n_h, 2 * d_h, b, c) == 2 * base
    assert oracle.kv_bytes_per_seq(n_l, n_h, d_h, 2 * b, c) == 2 * base
    assert oracle.kv_bytes_per_seq(n_l, n_h, d_h, b, 2 * c) == 2 * base


# ------------------------------------------------------- Eq. (2) and budget ----


def test_budget_mi300x(golden):
    g = golden["kv_budget_mi300x"]
    a = g["args"]
    assert oracle.kv_budget(a["hbm"], a["u_num"], a["u_den"], a["weights"], a["act"]) == g["bytes"]


def test_budget_clamps_to_zero():
    # weights exceed usable memory -> 0
    assert oracle.kv_budget(80 * 10**9, 9, 10, 141_200_000_000, 0) == 0
    assert oracle.kv_budget(80 * 10**9, 9, 10, 72 * 10**9, 0) == 0       # exactly used up
    assert oracle.kv_budget(80 * 10**9, 9, 10, 72 * 10**9 - 1, 0) == 1


def test_nseq_mi300x_qwen3(golden):
    g = golden["nseq_mi300x_qwen3"]
    budget = golden["kv_budget_mi300x"]["bytes"]
    for c, want in zip(g["c_max"], g["nseq"]):
        mseq = oracle.kv_bytes_per_seq(94, 4, 128, 2, c)
        assert oracle.max_seqs(budget, mseq, 8) == want
    # "4x more concurrent sequences"
    assert g["nseq"][0] // g["nseq"][1] == 4


def test_nseq_8x_constructed(golden):
    g = golden["nseq_llama70b_a100_constructed"]
    a = g["args"]
    budget = oracle.kv_budget(a["hbm"], a["u_num"], a["u_den"], a["weights"], a["act"])
    assert budget == 43_000_000_000
    got = [oracle.max_seqs(budget, oracle.kv_bytes_per_seq(80, 8, 128, 2, c), a["tp"]) for c in g["c_max"]]
    assert got == g["nseq"]
    assert got[1] == 8 * got[0]          # the 8x concurrency gain


def test_nseq_below_one_sequence():
    # budget smaller than one sequence's allocation -> 0
    mseq = oracle.kv_bytes_per_seq(80, 8, 128, 2, 65536)
    assert oracle.max_seqs(mseq - 1, mseq, 1) == 0
    assert oracle.max_seqs(mseq, mseq, 1) == 1
    assert oracle.max_seqs(0, mseq, 8) == 0


@given(st.integers(0, 10**12), st.integers(1, 126), st.integers(1, 16), st.sampled_from([64, 128]),
       st.sampled_from([1, 2]), st.integers(1, 1 << 19), st.sampled_from([1, 2, 4, 8]))
@settings(max_examples=300, deadline=None)
def test_nseq_is_floor_by_definition(budget, n_l, n_h, d_h, b, c, tp):
    # N_seq = max n with n * (M_seq / tp) <= budget  (exact rational; Eq. 2)
    mseq = oracle.kv_bytes_per_seq(n_l, n_h, d_h, b, c)
    n = oracle.max_seqs(budget, mseq, tp)
    per_gpu = Fraction(mseq, tp)
    assert n * per_gpu <= budget < (n + 1) * per_gpu


@given(st.integers(10**9, 10**12), st.sampled_from([8192, 16384, 32768, 65536]))
@settings(max_examples=200, deadline=None)
def test_nseq_8x_iff_fractional_part_small(budget, c):
    # N(C/8) = 8 N(C) exactly iff frac(budget / M_seq(C)) < 1/8
    m = oracle.kv_bytes_per_seq(80, 8, 128, 2, c)
    m8 = oracle.kv_bytes_per_seq(80, 8, 128, 2, c // 8)
    x = Fraction(budget, m)
    frac = x - math.floor(x)
    assert (oracle.max_seqs(budget, m8, 1) == 8 * oracle.max_seqs(budget, m, 1)) == (frac < Fraction(1, 8))


def test_nseq_monotone_in_cmax_and_budget():
    rng = np.random.default_rng(1)
    for _ in range(200):
        budget = int(rng.integers(0, 10**12))
        cs = sorted(int(x) for x in rng.integers(1, 1 << 18, size=5))
        ns = [oracle.max_seqs(budget, oracle.kv_bytes_per_seq(80, 8, 128, 2, c), 2) for c in cs]
        assert all(a >= b for a, b in zip(ns, ns[1:]))            # non-increasing in C_max
        n2 = oracle.max_seqs(budget + 10**9, oracle.kv_bytes_per_seq(80, 8, 128, 2, cs[0]), 2)
        assert n2 >= ns[0]                                       # non-decreasing in budget


# ------------------------------------------------------------- Sec. 3 sizing ----


def test_g_homo(golden):
    for g in golden["g_homo"]:
        ok, inst = oracle.pool_instances(float(g["lambda"]), g["mu"], 16)
        assert ok and inst == g["gpus"], g["cite"]


def test_g_dual(golden):
    for g in golden["g_dual"]:
        lam = float(g["lambda"])
        ok_s, s = oracle.pool_instances(g["alpha"] * lam, g["mu_s"], 128)
        ok_l, l = oracle.pool_instances((1 - g["alpha"]) * lam, g["mu_l"], 16)
        assert ok_s and ok_l and (s, l) == (g["short"], g["long"]), g["cite"]


def test_pool_degenerate_cases():
    # R13: zero load -> 0 instances even with N_seq = 0 or mu = 0
    assert oracle.pool_instances(0.0, 0.0, 0) == (True, 0)
    assert oracle.pool_instances(0.0, 2.8, 0) == (True, 0)
    # load with no capacity -> infeasible
    assert oracle.pool_instances(1.0, 2.8, 0)[0] is False
    assert oracle.pool_instances(1.0, 0.0, 16)[0] is False
    assert oracle.pool_instances(1e300, 1e-300, 16)[0] is False      # not representable
    # exact integer quotient is not rounded up
    assert oracle.pool_instances(1000.0, 2.0, 1) == (True, 500)
    assert oracle.pool_instances(1000.0, 3.0, 1) == (True, 334)


@given(st.floats(0, 1e6, allow_nan=False), st.floats(0, 1e6, allow_nan=False),
       st.floats(1e-3, 1e3, allow_nan=False))
@settings(max_examples=300, deadline=None)
def test_instances_monotone_in_load_and_mu(l1, l2, mu):
    lo, hi = sorted((l1, l2))
    a = oracle.pool_instances(lo, mu, 1)[1]
    b = oracle.pool_instances(hi, mu, 1)[1]
    assert a <= b                                   # monotone in lambda
    c = oracle.pool_instances(hi, mu * 2, 1)[1]
    assert c <= b                                   # non-increasing in mu
    # and it is the ceiling of the IEEE quotient
    if hi > 0:
        assert b == math.ceil(hi / mu)


@given(st.floats(1e-2, 1e5, allow_nan=False), st.floats(1e-2, 1e3, allow_nan=False))
@settings(max_examples=300, deadline=None)
def test_instances_exact_rational_ceiling(lam, mu):
    # The double quotient's ceiling equals the exact rational ceiling unless the
    # exact quotient is within a few ulps of an integer (reading R14).
    ok, inst = oracle.pool_instances(lam, mu, 1)
    exact = Fraction(lam) / Fraction(mu)
    ce = math.ceil(exact)
    if abs(exact - round(exact)) > Fraction(1, 10**9) * exact:
        assert inst == ce


# ------------------------------------------------------------- Eq. (7) ----


def test_predicted_savings(golden):
    for g in golden["predicted_savings"]:
        assert abs(oracle.predicted_savings(g["alpha"], g["rho"]) - g["value"]) <= 1e-12, g["cite"]
    r = golden["rho_table1"]
    assert r["mu_s"] / r["mu_l"] == r["rho"]


@given(st.floats(0, 1), st.floats(0, 1), st.floats(1, 64), st.floats(1, 64))
@settings(max_examples=300, deadline=None)
def test_predicted_savings_monotone(a1, a2, r1, r2):
    # monotone increasing in alpha and in rho for rho >= 1
    (a_lo, a_hi), (r_lo, r_hi) = sorted((a1, a2)), sorted((r1, r2))
    assert oracle.predicted_savings(a_lo, r_lo) <= oracle.predicted_savings(a_hi, r_lo) + 1e-15
    assert oracle.predicted_savings(a_lo, r_lo) <= oracle.predicted_savings(a_lo, r_hi) + 1e-15
    assert 0.0 <= oracle.predicted_savings(a_hi, r_hi) < 1.0


# ------------------------------------------------------------------ cost ----


def test_cost_pins(golden):
    for g in golden["cost"]:
        c = oracle.cost(g["gpus"], g["price"], g["hours"])
        if "musd_1dp_trunc" in g:
            assert math.floor(c / 1e5) / 10 == g["musd_1dp_trunc"], (c, g["cite"])
        else:
            assert math.floor(c / 1e3) == g["kusd_trunc"], (c, g["cite"])
    s = golden["cost_savings_musd"]
    d = oracle.cost(s["homo"], s["price"], s["hours"]) - oracle.cost(s["dual"], s["price"], s["hours"])
    assert round(d / 1e6, 1) == s["musd_1dp"]
    assert round(100 * (s["homo"] - s["dual"]) / s["homo"], 1) == s["pct_1dp"]
    # $2.86M/yr = 12 x $238.68K
    assert round(12 * oracle.cost(150, 2.21, 720) / 1e6, 2) == 2.86


# --------------------------------------------------------------- routing ----


def test_route_worked_examples(golden):
    for g in golden["route"]:
        assert oracle.route(g["L"], g["B"], g["c_short"], g["c_long"]) == (g["pool"], g["stage"]), g["cite"]


def _alg1_python(L, B, cs, cl):
    """Alg. 1 re-read independently of the C oracle: returns pool."""
    if L > cl:
        return 2
    if L > cs:
        return 1
    p = 0 if L <= B else 1
    cmax = cs if p == 0 else cl
    if L > cmax:
        p = 1
    return p


@given(st.lists(st.integers(0, 300), min_size=1, max_size=64), st.integers(0, 300),
       st.integers(0, 300), st.integers(0, 300))
@settings(max_examples=300, deadline=None)
def test_route_batch_brute_force(L, B, cs, cl):
    B, cs, cl = sorted((B, cs, cl))            # valid configuration B <= C_S <= C_L
    dec, counts = oracle.route_batch(L, B, cs, cl)
    pools = [_alg1_python(x, B, cs, cl) for x in L]
    assert [int(d) & 3 for d in dec] == pools
    assert counts[0] == pools.count(0) and counts[1] == pools.count(1) and counts[2] == pools.count(2)
    assert counts[3] == sum(x for x, p in zip(L, pools) if p == 0)
    assert counts[4] == sum(x for x, p in zip(L, pools) if p == 1)
    # safety guarantee: every served request fits its pool
    for x, p in zip(L, pools):
        if p == 0:
            assert x <= cs
        elif p == 1:
            assert x <= cl


def test_route_threshold_monotone():
    # raising B never moves a request from short to long
    rng = np.random.default_rng(7)
    L = rng.integers(0, 70000, size=2000)
    prev = None
    for B in range(0, 65537, 4096):
        d, _ = oracle.route_batch(L, B, 65536, 65536)
        short = (d & 3) == 0
        if prev is not None:
            assert np.all(short[prev])
        prev = short


# --------------------------------------------------------- CDF counting ----


def test_count_le_vs_sorted_search():
    rng = np.random.default_rng(3)
    L = rng.integers(0, 1 << 20, size=100_000, dtype=np.uint32)
    x = np.array([0, 1, 5, 1000, 65536, 1 << 19, (1 << 20) - 1, 1 << 20], dtype=np.uint32)
    cnt, mass = oracle.count_le(L, x)
    s = np.sort(L.astype(np.int64))
    csum = np.concatenate([[0], np.cumsum(s)])
    k = np.searchsorted(s, x.astype(np.int64), side="right")
    assert np.array_equal(cnt, k.astype(np.uint64))
    assert np.array_equal(mass, csum[k].astype(np.uint64))


@given(st.lists(st.integers(0, 2**32 - 1), max_size=200), st.lists(st.integers(0, 2**32 - 1), min_size=1, max_size=8))
@settings(max_examples=200, deadline=None)
def test_count_le_brute_force(L, x):
    cnt, mass = oracle.count_le(L, x)
    for j, xj in enumerate(x):
        assert cnt[j] == sum(1 for v in L if v <= xj)
        assert int(mass[j]) == sum(v for v in L if v <= xj)


def test_count_le_invariants():
    rng = np.random.default_rng(5)
    L = rng.integers(0, 200000, size=50_000, dtype=np.uint32)
    x = np.sort(rng.integers(0, 200000, size=40, dtype=np.uint32))
    cnt, mass = oracle.count_le(L, x)
    assert np.all(np.diff(cnt.astype(np.int64)) >= 0) and np.all(np.diff(mass.astype(np.int64)) >= 0)
    c_all, m_all = oracle.count_le(L, [2**32 - 1])
    assert c_all[0] == L.size and int(m_all[0]) == int(L.astype(np.int64).sum())   # alpha(inf) = 1
    perm = rng.permutation(L)
    assert all(np.array_equal(a, b) for a, b in zip((cnt, mass), oracle.count_le(perm, x)))


# --------------------------------------------------------- fragmentation ----


def test_fragmentation_worst_case(golden):
    """Effect 3: 16-token blocks waste up to 15 tokens per sequence;
    with 128 short sequences at Qwen3's per-token per-GPU KV bytes (Eq. 1 / TP)
    that is ~46 MB. (The paper's "0.03% of MI300X HBM" is 0.024%: prose, R18.)"""
    g = golden["fragmentation"]
    a = golden["kv_per_token_per_gpu_qwen3"]["args"]
    per_tok, rem = oracle.kv_bytes_per_token_per_gpu(a["n_l"], a["n_h"], a["d_h"], a["b"], a["tp"])
    assert per_tok == g["per_token"] and rem == 0
    waste = g["n_seqs"] * (g["block"] - 1) * per_tok
    assert round(waste / 1e6) == g["mb_approx"]
    assert waste / 192e9 < 0.0003
