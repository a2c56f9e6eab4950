"""Pins for the oracle's whole-sweep function or_sweep (-m "not gpu").

Brute force (Alg. 1 applied literally per request and candidate), paper
worked numbers pushed through the full sweep, closed-form identities and
invariants. See tests/test_oracle_pins.py for the per-formula pins.
"""
import math
from dataclasses import replace

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle
from synth import configs
from synth.configs import Deploy, make_config
from synth.gen import generate_np


def _table1_cfg(rate=1000.0, b=8192, cs=(8192,), cl=(65536,), mu_s=11.2, mu_l=2.8):
    """Table 1 pools with mu as data; one GPU instance counted per
    instance as in Table 2 (reading R6)."""
    return make_config(
        "T1", "AZ", 1, 0, rate, ["llama3-70b"], ["a100-80g"], [b], list(cs), list(cl),
        deploy_override={("llama3-70b", "a100-80g"): Deploy(8, 141_200_000_000 // 8, 1)},
        mu_mode="table",
        mu_values={("llama3-70b", "a100-80g", 8192): mu_s, ("llama3-70b", "a100-80g", 65536): mu_l})


def _trace(n_short, n_long, n_rej=0):
    return np.array([100] * n_short + [20000] * n_long + [70000] * n_rej, dtype=np.uint32)


def test_table2_homogeneous_and_dual_through_sweep():
    # alpha = 0.80 at lambda = 1,000: G_homo = 358, G_dual = 72 + 72,
    # predicted 60%.
    allc, best = oracle.sweep(_table1_cfg(), _trace(800, 200))
    c = best[0]
    assert c["flags"] == 7
    assert (c["inst_short"], c["inst_long"], c["inst_homo"]) == (72, 72, 358)
    assert (c["gpus_dual"], c["gpus_homo"]) == (144, 358)
    assert c["nseq_short"] == 128 and c["nseq_long"] == 16          # P:40-43 under R10
    assert abs(c["predicted_savings"] - 0.60) <= 1e-12
    assert c["rho"] == 4.0
    assert abs(c["savings"] - (358 - 144) / 358) <= 1e-15
    assert c["cost_dual"] == 144 * 2.21 * 8760


def test_alpha_zero_and_lmsys_alpha():
    _, b0 = oracle.sweep(_table1_cfg(), _trace(0, 1000))
    assert (b0[0]["inst_short"], b0[0]["inst_long"]) == (0, 358)
    _, b68 = oracle.sweep(_table1_cfg(), _trace(680, 320))
    assert (b68[0]["inst_short"], b68[0]["inst_long"]) == (61, 115)    # alpha = 0.68


def test_rejections_leave_every_pool():
    # R3: L > C_L is rejected and excluded from the dual and homogeneous loads
    _, b = oracle.sweep(_table1_cfg(), _trace(800, 190, 10))
    c = b[0]
    assert (c["n_short"], c["n_long"], c["n_reject"]) == (800, 190, 10)
    assert c["inst_homo"] == math.ceil((990 / 1000 * 1000.0) / 2.8)


def test_integer_identity_savings_equals_predicted():
    # With exact integer quotients the ceiling is inert and the integer savings
    # equal the closed form alpha (1 - 1/rho) (derivation P:573-588).
    cfg = _table1_cfg(mu_s=8.0, mu_l=2.0)
    _, b = oracle.sweep(cfg, _trace(800, 200))
    c = b[0]
    assert (c["inst_short"], c["inst_long"], c["inst_homo"]) == (100, 100, 500)
    assert abs(c["savings"] - c["predicted_savings"]) <= 1e-12


def test_scale_invariance_of_savings():
    # savings approach the formula as the fleet grows (ceiling slack
    # washes out); alpha and rho do not depend on lambda.
    L = _trace(800, 200)
    gaps = []
    for lam in (10.0, 100.0, 1000.0, 10000.0, 100000.0):
        _, b = oracle.sweep(_table1_cfg(rate=lam), L)
        c = b[0]
        gaps.append(abs(c["savings"] - c["predicted_savings"]))
        assert c["alpha"] == 0.8
    assert gaps[-1] < 1e-3 and gaps[-1] <= gaps[0]


def _literal_sweep(cfg, L):
    """Alg. 1 per (request, candidate), pure Python: counts + mass."""
    out = []
    ncs = len(cfg.c_short) if cfg.c_short else 1
    for m in range(len(cfg.models)):
        for g in range(len(cfg.gpus)):
            for cl in cfg.c_long:
                for s in range(ncs):
                    for B in cfg.b_short:
                        cs = cfg.c_short[s] if cfg.c_short else B
                        if not (B <= cs <= cl):
                            out.append(None)
                            continue
                        n = [0, 0, 0]
                        ms = [0, 0]
                        for x in L:
                            x = int(x)
                            if x > cl:
                                p = 2
                            elif x > cs:
                                p = 1
                            else:
                                p = 0 if x <= B else 1
                                if x > (cs if p == 0 else cl):
                                    p = 1
                            n[p] += 1
                            if p < 2:
                                ms[p] += x
                        out.append((n, ms))
    return out


@given(st.lists(st.integers(1, 400), min_size=1, max_size=48),
       st.lists(st.integers(1, 400), min_size=1, max_size=4),
       st.lists(st.integers(1, 400), min_size=0, max_size=3),
       st.lists(st.integers(1, 400), min_size=1, max_size=3))
@settings(max_examples=150, deadline=None)
def test_sweep_counts_brute_force(L, b, cs, cl):
    cfg = make_config("tiny", "AZ", 1, len(L), 100.0, ["llama3-8b"], ["b200-180g"], b, cs, cl)
    allc, best = oracle.sweep(cfg, np.array(L, dtype=np.uint32))
    lit = _literal_sweep(cfg, L)
    assert len(lit) == len(allc)
    for rec, ref in zip(allc, lit):
        if ref is None:
            assert rec["flags"] == 0
            continue
        (ns, nl, nr), (mss, msl) = ref
        assert rec["flags"] & 1
        assert (rec["n_short"], rec["n_long"], rec["n_reject"]) == (ns, nl, nr)
        assert (rec["mass_short"], rec["mass_long"]) == (mss, msl)
        assert ns + nl + nr == len(L)


def _check_argmin(cfg, allc, best):
    for m in range(len(cfg.models)):
        sel = allc[(allc["model"] == m) & ((allc["flags"] & 2) != 0)]
        if sel.size == 0:
            assert best[m]["index"] == 0xFFFFFFFF
            continue
        mn = sel["cost_dual"].min()
        want = sel[sel["cost_dual"] == mn]["index"].min()      # ties -> lowest index (R12)
        assert best[m]["index"] == want
        assert best[m].tobytes() == allc[want].tobytes()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_config_sweeps_invariants(name):
    cfg = configs.CONFIGS[name]()
    cfg = cfg.with_n(min(cfg.n_requests, 20000))
    L = generate_np(cfg.shape, cfg.seed, 0, cfg.n_requests)
    allc, best = oracle.sweep(cfg, L)
    assert len(allc) == cfg.n_candidates()
    assert np.array_equal(allc["index"], np.arange(len(allc), dtype=np.uint32))
    # flat order (m, g, C_L, C_S, B), B fastest (R12): the record's own fields
    nb, ncs, ncl, ng = len(cfg.b_short), cfg.n_cs_eff(), len(cfg.c_long), len(cfg.gpus)
    i = np.arange(len(allc))
    kb, ks, kl = i % nb, (i // nb) % ncs, (i // (nb * ncs)) % ncl
    assert np.array_equal(allc["b_short"], np.array(cfg.b_short, np.uint32)[kb])
    cs = np.array(cfg.c_short, np.uint32)[ks] if cfg.c_short else allc["b_short"]
    assert np.array_equal(allc["c_short"], cs)
    assert np.array_equal(allc["c_long"], np.array(cfg.c_long, np.uint32)[kl])
    assert np.array_equal(allc["gpu"], (i // (nb * ncs * ncl)) % ng)
    assert np.array_equal(allc["model"], i // (nb * ncs * ncl * ng))
    v = (allc["flags"] & 1) != 0
    assert np.all(allc["n_short"][v] + allc["n_long"][v] + allc["n_reject"][v] == cfg.n_requests)
    assert np.all(allc["b_short"][v] <= allc["c_short"][v]) and np.all(allc["c_short"][v] <= allc["c_long"][v])
    f = (allc["flags"] & 2) != 0
    assert np.all(np.isfinite(allc["cost_dual"][f])) and np.all(np.isinf(allc["cost_dual"][~f]))
    _check_argmin(cfg, allc, best)
    # permutation invariance
    perm = np.random.default_rng(0).permutation(L)
    allc2, best2 = oracle.sweep(cfg, perm)
    assert allc.tobytes() == allc2.tobytes()


def test_c1_homogeneous_matches_table2_up_to_rejections():
    cfg = configs.c1()
    L = generate_np(cfg.shape, cfg.seed, 0, cfg.n_requests)
    _, best = oracle.sweep(cfg, L)
    c = best[0]
    served = (c["n_short"] + c["n_long"]) / cfg.n_requests
    assert c["inst_homo"] == math.ceil(served * cfg.rate_rps / 2.8)
    if c["n_reject"] == 0:
        assert c["inst_homo"] == 358


def test_fig6_shape_expectation_unpinned():
    """Expectation, NOT a pin: under the stated
    pow23 mu model on the AZ shape, the closed-form savings alpha(1 - 1/rho)
    peak at B = 8K and 4K-16K stay >= 80% of the peak (Fig. 6)."""
    cfg = replace(configs.c2(), b_short=(1024, 2048, 4096, 8192, 16384, 32768), n_requests=200_000)
    L = generate_np("AZ", cfg.seed, 0, cfg.n_requests)
    allc, _ = oracle.sweep(cfg, L)
    pred = dict(zip(allc["b_short"].tolist(), allc["predicted_savings"].tolist()))
    peak_b = max(pred, key=pred.get)
    assert peak_b == 8192
    assert all(pred[b] >= 0.8 * pred[8192] for b in (4096, 8192, 16384))


def test_empty_trace_is_an_error():
    with pytest.raises(ValueError):
        oracle.sweep(_table1_cfg(), np.zeros(0, dtype=np.uint32))
