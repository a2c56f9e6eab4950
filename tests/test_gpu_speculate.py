"""FP_FLAG_SPECULATE (speculative routing in sweep_and_route): a sample pass and
its K3 pick a split, the full trace pass writes the decision bytes for it, the
full K3 picks the true split, and a verify kernel re-routes from L_total when
they differ. Whatever the sample says, every output must equal the oracle's:
best records, route counts, and every decision byte (Alg. 1 for the true best
split of the whole trace). Covers the hit path, a forced miss (a trace whose
sampled stripes are unrepresentative), the async form, and the fallbacks."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_08075_b200 as fp  # noqa: E402
from synth import configs  # noqa: E402
from synth.gen import generate_host  # noqa: E402

N = (1 << 26) + 12_345            # the speculative path needs >= 2^26 requests


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def _plan(cfg, flags=fp.FP_FLAG_SPECULATE):
    return fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=flags)


def _check_step(cfg, L, plan, dec, best, counts):
    _, obest = oracle.sweep(cfg, L, want_all=False)
    assert best.tobytes() == obest.tobytes()
    b = obest[0]
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    got = dec[:L.size].cpu().numpy()
    if not np.array_equal(got, odec):
        bad = np.nonzero(got != odec)[0]
        raise AssertionError(f"{bad.size} decisions differ, first at {bad[0]}")
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in oc]


def _sampled_stripes(plan, n, per_thread=4):
    """The request ranges the sample pass reads (white box: grid-wide stripes of
    the trace pass, every stride-th of them; per_thread = uint4 per thread per
    step: 4, raw columns 2)."""
    info = fp.fleet_plan_info(plan)
    S = info["k1_grid"] * info["k1_block"]
    stripe = S * per_thread * 4                          # requests per grid step
    nsteps = (n // 4 + S * per_thread - 1) // (S * per_thread)
    stride = max(1, nsteps // 4)
    return [(k * stripe, min(n, (k + 1) * stripe)) for k in range(0, nsteps, stride)]


def test_speculative_hit_equals_oracle():
    cfg = configs.c5().with_n(N)
    L = generate_host(cfg.shape, cfg.seed, 0, N)
    plan = _plan(cfg)
    dec = torch.full((N,), 0xEE, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(L), cfg.rate_rps, route_model=0, decision=dec)
    _check_step(cfg, L, plan, dec, best, counts)
    info = fp.fleet_plan_info(plan)
    assert info["spec_calls"] == 1 and info["spec_misses"] == 0
    # steady state: the asynchronous form, twice (the sample's accumulators are re-zeroed by the full K3)
    d = _dev(L)
    for _ in range(2):
        dec.fill_(0xEE)
        assert fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False) == (None, None)
    best2 = fp.best_split(plan)
    _check_step(cfg, L, plan, dec, best2, counts)
    assert fp.fleet_plan_info(plan)["spec_calls"] == 3


def test_speculative_forced_miss_reroutes():
    """The sampled stripes hold only short requests, so the sample's split is
    not the whole trace's: the verify kernel must re-route every request."""
    cfg = configs.c5().with_n(N)
    L = generate_host(cfg.shape, cfg.seed, 0, N).copy()
    plan = _plan(cfg)
    for lo, hi in _sampled_stripes(plan, N):
        L[lo:hi] = 100
    dec = torch.full((N,), 0xEE, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(L), cfg.rate_rps, route_model=0, decision=dec)
    _check_step(cfg, L, plan, dec, best, counts)
    assert fp.fleet_plan_info(plan)["spec_misses"] == 1


@pytest.mark.parametrize("case", ["misaligned_decision", "small_trace", "route_model_1"])
def test_speculative_fallbacks_and_models(case):
    n = 1_000_003 if case == "small_trace" else N
    cfg = configs.c5().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    plan = _plan(cfg)
    doff = 1 if case == "misaligned_decision" else 0
    model = 1 if case == "route_model_1" else 0
    buf = torch.full((n + 16,), 0xEE, dtype=torch.uint8, device="cuda")
    dec = buf[doff:doff + n]
    best, counts = fp.sweep_and_route(plan, _dev(L), cfg.rate_rps, route_model=model, decision=dec)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    assert best.tobytes() == obest.tobytes()
    b = obest[model]
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec.cpu().numpy(), odec)
    expect_spec = case == "route_model_1"
    assert fp.fleet_plan_info(plan)["spec_calls"] == (1 if expect_spec else 0)


# ---- the raw-column form (sweep_and_route_raw, NEXT-1) --------------------------------------
CALIB = [(4.39, 0.45), (3.45, 0.35), (1.97, 0.2), (3.73, 0.38)]   # a calibrated snapshot (stated)


def _raw_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else a).cuda()


def _raw_check(cfg, body, mo, cat, cats, dec, best, counts, model=0):
    L = oracle.estimate(body, mo, cat, cats, 1.0, 0.5)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    assert best.tobytes() == obest.tobytes()
    b = obest[model]
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    got = dec[:L.size].cpu().numpy()
    if not np.array_equal(got, odec):
        bad = np.nonzero(got != odec)[0]
        raise AssertionError(f"{bad.size} decisions differ, first at {bad[:5]}: got {got[bad[:5]]} "
                             f"expected {odec[bad[:5]]} (L {L[bad[:5]]})")
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in oc]


@pytest.mark.parametrize("flags,n,expect_spec", [("spec", N, True), ("plain", 700_001, False),
                                                 ("spec", 700_001, False)])
def test_raw_step_matches_oracle(flags, n, expect_spec):
    from synth.gen import generate_raw_host
    cfg = configs.c5().with_n(n)
    body, mo, cat, _ = generate_raw_host(cfg.shape, cfg.seed, 0, n)
    plan = _plan(cfg, flags=fp.FP_FLAG_SPECULATE if flags == "spec" else 0)
    dec = torch.full((n,), 0xEE, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route_raw(plan, _raw_dev(body), _raw_dev(mo), _raw_dev(cat), CALIB, cfg.rate_rps,
                                          route_model=0, decision=dec)
    _raw_check(cfg, body, mo, cat, CALIB, dec, best, counts)
    assert (fp.fleet_plan_info(plan)["spec_calls"] == 1) == expect_spec


def test_raw_step_forced_miss():
    """Sampled stripes of tiny bodies: the sample's split is not the trace's, and
    the verify kernel re-routes every request from its estimated L_total."""
    from synth.gen import generate_raw_host
    cfg = configs.c5().with_n(N)
    body, mo, cat, _ = generate_raw_host(cfg.shape, cfg.seed, 0, N)
    body, mo = body.copy(), mo.copy()
    plan = _plan(cfg)
    for lo, hi in _sampled_stripes(plan, N, per_thread=2):
        body[lo:hi] = 10
        mo[lo:hi] = 1
    dec = torch.full((N,), 0xEE, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route_raw(plan, _raw_dev(body), _raw_dev(mo), _raw_dev(cat), CALIB, cfg.rate_rps,
                                          route_model=0, decision=dec)
    _raw_check(cfg, body, mo, cat, CALIB, dec, best, counts)
    info = fp.fleet_plan_info(plan)
    assert info["spec_calls"] == 1 and info["spec_misses"] == 1


# ---- speculation for edge sets beyond the SWAR bins (u16 LUT, |E| >= 256) --------------------
def test_speculative_wide_edge_sets(monkeypatch):
    """C3's grid (|E| = 258 edges: u16 LUT, clamped byte bins) at the
    speculative size: the full pass writes decisions from L_total and the
    split's edge values (the bins no longer fit the SWAR byte compare): hit,
    then a forced miss."""
    cfg = configs.c3().with_n(N)
    L = generate_host(cfg.shape, cfg.seed, 0, N)
    # (a u16 LUT speculates from 2^28 requests by default)
    monkeypatch.setenv("FP_SPEC_MIN_WIDE_LOG2", "26")
    plan = _plan(cfg)
    info = fp.fleet_plan_info(plan)
    assert info["n_edges"] >= 256
    dec = torch.full((N,), 0xEE, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(L), cfg.rate_rps, route_model=0, decision=dec)
    _check_step(cfg, L, plan, dec, best, counts)
    info = fp.fleet_plan_info(plan)
    assert info["spec_calls"] == 1 and info["spec_misses"] == 0
    L2 = L.copy()
    for lo, hi in _sampled_stripes(plan, N):
        L2[lo:hi] = 100
    dec.fill_(0xEE)
    best, counts = fp.sweep_and_route(plan, _dev(L2), cfg.rate_rps, route_model=0, decision=dec)
    _check_step(cfg, L2, plan, dec, best, counts)
    assert fp.fleet_plan_info(plan)["spec_misses"] == 1
