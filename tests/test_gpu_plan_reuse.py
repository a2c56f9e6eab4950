"""One plan driven through every entry point in turn, with growing inputs, so
that each lazily grown scratch buffer is reallocated while the others are
live (regression: a reallocation once freed unrelated buffers)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_08075_b200 as fp  # noqa: E402
from synth import configs  # noqa: E402
from synth.gen import arrivals_host, generate_host, generate_raw_host  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else a).cuda()


def test_all_entry_points_on_one_plan():
    cfg = configs.c5()
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    for n in (10_000, 1_500_000, 4_000_000):
        c = cfg.with_n(n)
        L = generate_host(c.shape, c.seed, 0, n)
        # host trace (resident copy grows), then the bin pass (bin buffer grows)
        best, _ = fp.sweep_and_route(plan, torch.from_numpy(L.view(np.int32)), c.rate_rps, route_model=0)
        dec = torch.empty(n, dtype=torch.uint8, device="cuda")
        best_d, _ = fp.sweep_and_route(plan, _dev(L), c.rate_rps, route_model=0, decision=dec)
        _, obest = oracle.sweep(c, L)
        assert best.tobytes() == obest.tobytes() and best_d.tobytes() == obest.tobytes()
        _, best3 = fp.sweep_three_pools(plan, c.rate_rps)
        _, obest3 = oracle.sweep3(c, L)
        assert best3.tobytes() == obest3.tobytes()
        arr = arrivals_host(c.seed, n, c.rate_rps)
        _, bpk = fp.sweep_peak_windows(plan, _dev(L), torch.from_numpy(arr.view(np.int64)).cuda(), 10**9)
        _, opk = oracle.sweep_peak(c, L, arr, 10**9)
        assert bpk.tobytes() == opk.tobytes()
        body, mo, cat, tp = generate_raw_host("MIX", 5, 0, n)
        g = fp.calibrate_replay(plan, _dev(body), _dev(tp), _dev(cat), [(4.0, 0.5)] * 4)
        o = oracle.calibrate(body, tp, cat, 4, beta=0.95, c0=4.0, s0=0.5)
        assert np.allclose(g["c_hat"], o["c_hat"], rtol=1e-12, atol=0)
        # the three-pool records must still be readable after the other reallocations
        _, best3b = fp.sweep_three_pools(plan, c.rate_rps)
        assert best3b.tobytes() == best3.tobytes()


def test_back_to_back_steps_see_in_stream_trace_updates():
    """Asynchronous steps issued back to back on one stream, the trace rewritten
    in place by a torch kernel between them, no host synchronisation: every
    step's records and decisions follow the trace it was given (stream order
    with programmatic dependent launches, and K3's re-zeroing of K1's
    accumulators in place of a memset)."""
    cfg = configs.c5().with_n(2_000_003)
    n = cfg.n_requests
    L0 = generate_host(cfg.shape, cfg.seed, 0, n)
    L1 = generate_host(cfg.shape, cfg.seed + 1, 0, n)
    d = torch.from_numpy(L0.view(np.int32)).cuda()
    d1 = torch.from_numpy(L1.view(np.int32)).cuda()
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    s = torch.cuda.current_stream()
    decs, bests = [], []
    for k in range(4):
        dec = torch.empty(n, dtype=torch.uint8, device="cuda")
        fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, stream=s, want_best=False)
        bests.append(torch.empty(0))                      # placeholder; records read below per step
        decs.append(dec)
        # the next step's trace: swap contents on the stream (no sync)
        tmp = d.clone()
        d.copy_(d1)
        d1.copy_(tmp)
        if k == 1:
            # read the records of the 2nd step (synchronises here only)
            bests[k] = fp.best_split(plan)
    last = fp.best_split(plan)
    _, ob0 = oracle.sweep(cfg, L0)
    _, ob1 = oracle.sweep(cfg, L1)
    assert bests[1].tobytes() == ob1.tobytes()             # step 2 ran on L1
    assert last.tobytes() == ob1.tobytes()                 # step 4 ran on L1
    for k, (L, ob) in enumerate([(L0, ob0), (L1, ob1), (L0, ob0), (L1, ob1)]):
        b = ob[0]
        odec, _ = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
        assert np.array_equal(decs[k].cpu().numpy(), odec), k
    fp.fleet_plan_destroy(plan)
