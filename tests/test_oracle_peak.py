"""Pins for the oracle's peak-window provisioning (NEXT-4; -m "not gpu")."""
import math

import numpy as np
from hypothesis import given, settings, strategies as st

import oracle
from synth import configs
from synth.configs import make_config
from synth.gen import arrivals_host, gaps_np, generate_np


def test_arrivals_host_matches_numpy_and_rate():
    a = arrivals_host(3, 200_000, 10000.0)
    assert np.array_equal(np.cumsum(gaps_np(3, 0, 200_000, 10000.0), dtype=np.uint64), a)
    assert abs(a[-1] / 1e9 - 20.0) / 20.0 < 0.02          # Poisson rate, no burst phase yet


def test_uniform_arrivals_reduce_to_mean_rate_sizing():
    # one request per ms in 1-s windows: every window holds the mean load, so
    # peak sizing equals the mean-rate sizing of Sec. 3 at lambda = 1,000
    n = 20_000
    L = generate_np("AZ", 1, 0, n)
    arr = (np.arange(n, dtype=np.uint64) * np.uint64(1_000_000))
    cfg = make_config("u", "AZ", 1, n, 1000.0, ["llama3-8b"], ["b200-180g"], [2048, 8192], [], [65536])
    pk, _ = oracle.sweep_peak(cfg, L, arr, 10**9)
    mean, _ = oracle.sweep(cfg, L)
    for p, m in zip(pk, mean):
        w = 1000
        # the busiest window's share can exceed the mean share; bound it by hand
        assert p["peak_homo"] == max(np.bincount((arr // np.uint64(10**9)).astype(int),
                                                 weights=(L <= p["c_long"]).astype(float)).astype(int))
        assert p["inst_homo"] >= m["inst_homo"] - 1


@given(st.lists(st.tuples(st.integers(1, 300), st.integers(0, 5000)), min_size=1, max_size=60),
       st.sampled_from([1000, 2500]))
@settings(max_examples=100, deadline=None)
def test_peak_brute_force(rows, window):
    rows.sort(key=lambda r: r[1])
    L = np.array([r[0] for r in rows], np.uint32)
    arr = np.array([r[1] for r in rows], np.uint64)
    cfg = make_config("p", "AZ", 1, len(rows), 100.0, ["llama3-8b"], ["b200-180g"], [64, 128], [], [256])
    allc, best = oracle.sweep_peak(cfg, L, arr, window)
    for c in allc:
        B, CL = int(c["b_short"]), int(c["c_long"])
        per = {}
        for x, t in zip(L, arr):
            w = int(t) // window
            s, l, h = per.get(w, (0, 0, 0))
            per[w] = (s + (x <= B), l + (B < x <= CL), h + (x <= CL))
        ps = max(v[0] for v in per.values())
        pl = max(v[1] for v in per.values())
        ph = max(v[2] for v in per.values())
        assert (c["peak_short"], c["peak_long"], c["peak_homo"]) == (ps, pl, ph)
        assert c["lambda_short"] == ps * (1e9 / window)


def test_bursts_raise_peak_sizing():
    # with the stated 4x burst phase inside the trace, peak-window sizing needs
    # more instances than mean-rate sizing for the same split
    n = 8 << 20
    cfg = configs.c2().with_n(n)
    L = generate_np(cfg.shape, cfg.seed, 0, n)
    arr = arrivals_host(cfg.seed, n, cfg.rate_rps)
    pk, bp = oracle.sweep_peak(cfg, L, arr, 60 * 10**9, want_all=False)
    _, bm = oracle.sweep(cfg, L, want_all=False)
    assert bp[0]["gpus_dual"] > bm[0]["gpus_dual"]
