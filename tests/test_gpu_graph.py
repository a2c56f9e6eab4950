"""sweep_and_route_graph: the step of sweep_and_route (asynchronous form) as the
plan's captured CUDA graph, one graph per accumulator parity. Every replay
must equal the oracle -- best records and every decision byte -- across
parity alternation, in-place trace rewrites between replays (the graph reads
the same caller buffer), speculative steps, and recapture on a new argument
tuple."""
from dataclasses import replace

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


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def _check(cfg, L, plan, dec, model=0):
    best = fp.best_split(plan)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    assert best.tobytes() == obest.tobytes()
    b = obest[model]
    odec, _ = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    got = dec[:L.size].cpu().numpy()
    if not np.array_equal(got, odec):
        bad = np.nonzero(got != odec)[0]
        raise AssertionError(f"{bad.size} decisions differ, first at {bad[0]}")


@pytest.mark.parametrize("name,n,flags", [("C1", 1000, 0), ("C2", 10_300_000, 0), ("C3", 3_000_001, 0),
                                          ("C5", (1 << 26) + 12_345, fp.FP_FLAG_SPECULATE)])
def test_graph_replays_equal_oracle(name, n, flags):
    cfg = configs.CONFIGS[name]().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=flags)
    d = _dev(L)
    dec = torch.full((n,), 0xEE, dtype=torch.uint8, device="cuda")
    for _ in range(3):                                   # capture + two replays (both parities)
        dec.fill_(0xEE)
        fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec)
        _check(cfg, L, plan, dec)
    # the trace rewritten in place: the replay reads the new content
    L2 = np.minimum(L.astype(np.uint64) * 3 // 2, 2**32 - 1).astype(np.uint32)
    d.copy_(_dev(L2))
    for _ in range(2):
        dec.fill_(0xEE)
        fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec)
        _check(cfg, L2, plan, dec)
    if flags & fp.FP_FLAG_SPECULATE:
        assert fp.fleet_plan_info(plan)["spec_calls"] >= 5
    # an eager call in between keeps the parity bookkeeping consistent
    dec.fill_(0xEE)
    fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False)
    fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec)
    _check(cfg, L2, plan, dec)
    fp.fleet_plan_destroy(plan)


def test_graph_recaptures_on_new_arguments():
    cfg = configs.c2()
    n = cfg.n_requests
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    d = _dev(L)
    dec = torch.zeros(n, dtype=torch.uint8, device="cuda")
    fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec)
    _check(cfg, L, plan, dec)
    m = n // 3                                                   # a shorter trace: new key
    fp.sweep_and_route_graph(plan, d[:m], cfg.rate_rps, dec[:m])
    _check(cfg.with_n(m), L[:m], plan, dec[:m])
    fp.sweep_and_route_graph(plan, d[:m], cfg.rate_rps * 3, dec[:m])   # another rate: new key
    _check(replace(cfg.with_n(m), rate_rps=cfg.rate_rps * 3), L[:m], plan, dec[:m])
    fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec)         # and back
    _check(cfg, L, plan, dec)


def test_graph_refuses_timing_and_host_traces():
    cfg = configs.c1()
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_TIME_TRACE)
    dec = torch.zeros(cfg.n_requests, dtype=torch.uint8, device="cuda")
    with pytest.raises(fp.FleetPlanError, match="CONFIG"):
        fp.sweep_and_route_graph(plan, _dev(L), cfg.rate_rps, dec)
    plan2 = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    with pytest.raises(ValueError):
        fp.sweep_and_route_graph(plan2, torch.from_numpy(L.view(np.int32)), cfg.rate_rps, dec)
