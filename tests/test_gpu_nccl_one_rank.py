"""The NCCL calls of the multi-rank path on ONE GPU: a plan with
FP_FLAG_COLLECTIVES and world = 1 takes every cross-rank step of a world > 1
plan (histogram all-reduce, candidate slicing, all-gather of best records,
the one-warp split pick, route count all-reduce, the ordered-shard
calibration exchange, the window histogram all-reduce) through a real
one-rank NCCL communicator built from ncclGetUniqueId. The results must
equal the oracle's (and the plain single-rank plan's) exactly. This is what
exercises the dlopen'ed NCCL surface (symbols, enum values, argument order,
stream ordering) on a box with one GPU; the decomposition across ranks is
covered by the world-2 tests (test_gpu_multirank*.py, gloo hooks)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _nccl_plan(fp, cfg, flags=0):
    uid = fp.fp_nccl_get_unique_id()
    return fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0, rank=0, world=1, nccl_unique_id=uid,
                                flags=flags | fp.FP_FLAG_COLLECTIVES)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else a).cuda()


def test_collectives_flag_needs_a_communicator():
    import paper_2604_08075_b200 as fp
    from synth import configs
    with pytest.raises(fp.FleetPlanError):
        fp.fleet_plan_create(**fp.desc_from_config(configs.c1()), device=0, flags=fp.FP_FLAG_COLLECTIVES)


@pytest.mark.parametrize("name,n,replicated", [("C5", 1_000_003, False), ("C3", 200_001, False),
                                               ("C4", 300_000, True), ("C1", 1000, False)])
def test_sweep_route_through_nccl(name, n, replicated):
    import oracle
    import paper_2604_08075_b200 as fp
    from synth import configs
    from synth.gen import generate_device, generate_host
    cfg = configs.CONFIGS[name]().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    d = generate_device(cfg.shape, cfg.seed, 0, n)
    plan = _nccl_plan(fp, cfg, fp.FP_FLAG_REPLICATED_GRID if replicated else 0)
    res = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
    best = fp.best_split(plan)
    allc, obest = oracle.sweep(cfg, L)
    assert res.tobytes() == allc.tobytes()
    assert best.tobytes() == obest.tobytes()
    counts = fp.route_batch(plan, d, 8192, 16384, 65536)
    _, oc = oracle.route_batch(L, 8192, 16384, 65536, want_decisions=False)
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == \
        [int(x) for x in oc]
    # the whole step: K1 (+bins) -> all-reduce -> K3 -> all-gather -> pick -> K4b
    dec = torch.empty(n, dtype=torch.uint8, device="cuda")
    b2, c2 = fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec)
    assert b2.tobytes() == obest.tobytes()
    b = obest[0]
    odec, oc2 = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec.cpu().numpy(), odec)
    assert [c2[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == \
        [int(x) for x in oc2]
    # asynchronous form (no host outputs), records read afterwards
    dec.zero_()
    fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False)
    assert fp.best_split(plan).tobytes() == obest.tobytes()
    assert np.array_equal(dec.cpu().numpy(), odec)
    fp.fleet_plan_destroy(plan)


def test_raw_and_three_pools_through_nccl():
    import paper_2604_08075_b200 as fp
    from synth import configs
    from synth.gen import generate_raw_device
    from synth.shapes import CAT_TRUE_RATIO
    cfg = configs.c5().with_n(500_001)
    body, mo, cat, tp = generate_raw_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
    cats = [(c * 0.98, 0.1 * c) for c in CAT_TRUE_RATIO]
    out = []
    for mk in (lambda: fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0), lambda: _nccl_plan(fp, cfg)):
        plan = mk()
        res = fp.sweep_thresholds_raw(plan, body, mo, cat, cats, cfg.rate_rps, want_results=True)
        best = fp.best_split(plan)
        counts, mis = fp.route_batch_raw(plan, body, mo, cat, cats, 8192, 8192, 65536, true_prompt=tp)
        _, best3 = fp.sweep_three_pools(plan, cfg.rate_rps)
        out.append((res.tobytes(), best.tobytes(), counts, mis, best3.tobytes()))
        fp.fleet_plan_destroy(plan)
    assert out[0] == out[1]


def test_calibration_and_peak_through_nccl():
    import oracle
    import paper_2604_08075_b200 as fp
    from synth import configs
    from synth.gen import arrivals_host, generate_host, generate_raw_host
    n = 400_003
    body, mo, cat, tp = generate_raw_host("MIX", 31, 0, n)
    tp[::89] = 0
    plan = _nccl_plan(fp, configs.c1())
    g = fp.calibrate_replay(plan, _dev(body), _dev(tp), _dev(cat), [(4.0, 0.5)] * 4, beta=0.95, snap_at=50)
    fp.fleet_plan_destroy(plan)
    o = oracle.calibrate(body, tp, cat, 4, beta=0.95, c0=4.0, s0=0.5, snap_at=50)
    assert [int(x) for x in g["n_obs"]] == [int(x) for x in o["n_obs"]]
    for key in ("c_hat", "sigma", "snap_c", "snap_sigma"):
        assert np.allclose(g[key], o[key], rtol=1e-12, atol=0, equal_nan=True), key

    cfg = configs.c5().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    arr = arrivals_host(cfg.seed, n, cfg.rate_rps)
    plan = _nccl_plan(fp, cfg)
    res, best = fp.sweep_peak_windows(plan, _dev(L), torch.from_numpy(arr.view(np.int64)).cuda(), 10**9,
                                      want_results=True)
    fp.fleet_plan_destroy(plan)
    oall, obest = oracle.sweep_peak(cfg, L, arr, 10**9)
    assert res.tobytes() == oall.tobytes()
    assert best.tobytes() == obest.tobytes()


def test_p2p_exchange_one_rank():
    """FP_FLAG_P2P on one rank: K3 reads the accumulators through the peer
    table (its own buffer), the flag protocol advances one epoch per sweep, and
    alternating parities give the oracle's result every step."""
    import oracle
    import paper_2604_08075_b200 as fp
    from synth import configs
    from synth.gen import generate_device, generate_host
    cfg = configs.c5().with_n(700_001)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
    allc, obest = oracle.sweep(cfg, L)
    plan = _nccl_plan(fp, cfg, fp.FP_FLAG_P2P)
    with pytest.raises(fp.FleetPlanError):
        fp.sweep_thresholds(plan, d, cfg.rate_rps)          # before the import
    fp.fp_p2p_import(plan, [fp.fp_p2p_export(plan)])
    with pytest.raises(fp.FleetPlanError):
        fp.fp_p2p_import(plan, [fp.fp_p2p_export(plan)])    # twice
    for _ in range(3):
        res = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
        assert res.tobytes() == allc.tobytes()
        assert fp.best_split(plan).tobytes() == obest.tobytes()
    dec = torch.empty(cfg.n_requests, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False)
    assert fp.best_split(plan).tobytes() == obest.tobytes()
    b = obest[0]
    odec, _ = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec.cpu().numpy(), odec)
    _, cnt, mass = fp.sweep_histogram(plan)
    assert int(cnt.sum()) == cfg.n_requests
    # NEXT-2 reuses the last sweep's summed histogram (K3 publishes it; the
    # P2P accumulators themselves alternate between parities)
    _, best3 = fp.sweep_three_pools(plan, cfg.rate_rps)
    fp.fleet_plan_destroy(plan)
    ref = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0)
    fp.sweep_thresholds(ref, d, cfg.rate_rps)
    _, ref3 = fp.sweep_three_pools(ref, cfg.rate_rps)
    fp.fleet_plan_destroy(ref)
    assert best3.tobytes() == ref3.tobytes()


def test_p2p_needs_a_multi_rank_plan():
    import paper_2604_08075_b200 as fp
    from synth import configs
    with pytest.raises(fp.FleetPlanError):
        fp.fleet_plan_create(**fp.desc_from_config(configs.c1()), device=0, flags=fp.FP_FLAG_P2P)
    plan = fp.fleet_plan_create(**fp.desc_from_config(configs.c1()), device=0)
    with pytest.raises(fp.FleetPlanError):
        fp.fp_p2p_export(plan)
    fp.fleet_plan_destroy(plan)
