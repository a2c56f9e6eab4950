"""Randomised parity of the whole path (GPU vs the CPU oracle): random grids
(threshold counts, multiples and ranges that select the u8 LUT, the u16 LUT or
the binary-search bin mode; tied or independent C_S; several C_L), random model
and GPU subsets, pow23 or random-table mu, random rates, and traces mixing the
synthetic shapes with adversarial values (0, exact edges, edge +- 1, values
above every window, 2^32 - 1) at ragged sizes and pointer phases. Every
candidate record, the best splits, the histogram, every decision byte of
sweep_and_route and a route_batch with a random split must equal the oracle's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_08075_b200 as fp  # noqa: E402
from synth import configs  # noqa: E402
from synth.configs import make_config  # noqa: E402
from synth.gen import generate_host  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def _random_case(seed):
    rng = np.random.default_rng(7000 + seed)
    mode = rng.choice(["u8", "u16", "search"])
    mult = int(rng.choice([1, 16, 256])) if mode != "search" else 1
    if mode == "u8":
        nb = int(rng.integers(1, 90))
        b = sorted(set(int(x) * mult for x in rng.integers(1, 65536 // mult, nb)))
    elif mode == "u16":
        nb = int(rng.integers(260, 700))
        b = sorted(set(int(x) * 16 for x in rng.integers(1, 8192, nb)))
    else:
        nb = int(rng.integers(5, 60))
        b = sorted(set(int(x) for x in rng.integers(1, 2_000_000_000, nb)))
    top = max(b)
    cl = sorted(set([top] + [min(int(top * f), 2**31 - 1) for f in rng.uniform(1.0, 4.0, int(rng.integers(1, 5)))]))
    if mode != "search":
        cl = [((c + mult - 1) // mult) * mult for c in cl]
        cl = sorted(set(min(c, 2**31 - mult) for c in cl))
    cs = []
    if rng.random() < 0.4:
        cs = sorted(set(int(x) for x in rng.choice(b + cl, int(rng.integers(1, 6)))))
    models = list(rng.choice(list(configs.MODELS), int(rng.integers(1, 4)), replace=False))
    gpus = list(rng.choice(list(configs.GPUS), int(rng.integers(1, 3)), replace=False))
    n = int(rng.integers(1, 300_000))
    cfg = make_config("FZ", str(rng.choice(["AZ", "LM", "SG", "MIX"])), 100 + seed, n,
                      float(rng.choice([1.0, 1000.0, 1e5])), models, gpus, b, cs, cl)
    if rng.random() < 0.5:
        from dataclasses import replace
        vals = {(m.name, g.name, int(w)): float(rng.uniform(0.05, 60.0))
                for m in cfg.models for g in cfg.gpus for w in cfg.windows()}
        cfg = replace(cfg, mu_mode="table", mu_values=vals)
    L = generate_host(cfg.shape, cfg.seed, 0, n).astype(np.uint32)
    # adversarial values at random positions
    edges = np.array(sorted(set(b) | set(cs) | set(cl)), dtype=np.uint64)
    k = max(1, n // 20)
    pos = rng.integers(0, n, k)
    pick = rng.integers(0, 6, k)
    e = edges[rng.integers(0, edges.size, k)]
    adv = np.select([pick == 0, pick == 1, pick == 2, pick == 3, pick == 4],
                    [np.zeros(k), e, e + 1, np.maximum(e, 1) - 1, np.full(k, 2**32 - 1)],
                    default=e * 3)
    L[pos] = np.minimum(adv, 2**32 - 1).astype(np.uint32)
    return cfg, L, rng


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_whole_path(seed):
    cfg, L, rng = _random_case(seed)
    off = int(rng.integers(0, 4))
    full = np.concatenate([np.zeros(off, dtype=np.uint32), L])
    d = _dev(full)[off:]
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    res = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
    best = fp.best_split(plan)
    allc, obest = oracle.sweep(cfg, L)
    assert res.tobytes() == allc.tobytes(), f"seed {seed}: candidate records differ"
    assert best.tobytes() == obest.tobytes(), f"seed {seed}: best splits differ"
    edges, cnt, _ = fp.sweep_histogram(plan)
    ocnt, _ = oracle.count_le(L, edges)
    assert np.array_equal(np.cumsum(cnt)[:-1], ocnt) and int(cnt.sum()) == L.size
    # the step, when model 0 has a feasible split
    if obest[0]["flags"] & fp.FP_CAND_FEASIBLE:
        dec = torch.zeros(L.size + 8, dtype=torch.uint8, device="cuda")
        doff = int(rng.integers(0, 4))
        b2, counts = fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec[doff:])
        assert b2.tobytes() == obest.tobytes()
        b = obest[0]
        odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
        assert np.array_equal(dec[doff:doff + L.size].cpu().numpy(), odec), f"seed {seed}: decisions differ"
        assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == \
            [int(x) for x in oc]
    # route_batch with a random valid split
    bb = int(rng.choice(cfg.b_short))
    cl_ok = [c for c in cfg.c_long if c >= bb]
    if cl_ok:
        cl = int(rng.choice(cl_ok))
        cs_ok = [c for c in (cfg.c_short or [bb]) if bb <= c <= cl]
        if cs_ok:
            cs = int(rng.choice(cs_ok))
            counts = fp.route_batch(plan, d, bb, cs, cl)
            _, oc = oracle.route_batch(L, bb, cs, cl, want_decisions=False)
            assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == \
                [int(x) for x in oc]
    fp.fleet_plan_destroy(plan)


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_speculative_step(seed, monkeypatch):
    """The speculative step (FP_FLAG_SPECULATE) on random grids at the
    speculative size: u8 LUTs with |E| < 127 (decisions by SWAR on the bins)
    and u16 LUTs (decisions from L_total; FP_SPEC_MIN_WIDE_LOG2=26), random
    route_model, adversarial values, ragged size -- every decision byte and
    the best records against the oracle, whether the sample hit or not."""
    from dataclasses import replace
    rng = np.random.default_rng(9100 + seed)
    wide = seed % 2 == 1
    mult = 256 if wide else int(rng.choice([16, 256]))       # LUT bin mode (not binary search)
    if wide:
        b = sorted(set(int(x) * mult for x in rng.integers(1, 512, 400)))[:int(rng.integers(262, 300))]
    else:
        b = sorted(set(int(x) * mult for x in rng.integers(1, 65536 // mult, int(rng.integers(3, 110)))))
        b = b[:118]
    top = max(b)
    cl = sorted(set([top] + [((min(int(top * f), 2**31 - mult) + mult - 1) // mult) * mult
                             for f in rng.uniform(1.0, 4.0, int(rng.integers(1, 4)))]))
    if not wide:
        cl = cl[:4]
    models = list(rng.choice(list(configs.MODELS), int(rng.integers(1, 4)), replace=False))
    gpus = list(rng.choice(list(configs.GPUS), int(rng.integers(1, 3)), replace=False))
    n = (1 << 26) + int(rng.integers(0, 5000))
    cfg = make_config("FZS", str(rng.choice(["AZ", "LM", "MIX"])), 500 + seed, n,
                      float(rng.choice([1000.0, 1e4])), models, gpus, b, [], cl)
    if rng.random() < 0.5:
        vals = {(m.name, g.name, int(w)): float(rng.uniform(0.05, 60.0))
                for m in cfg.models for g in cfg.gpus for w in cfg.windows()}
        cfg = replace(cfg, mu_mode="table", mu_values=vals)
    L = generate_host(cfg.shape, cfg.seed, 0, n).astype(np.uint32)
    edges = np.array(sorted(set(b) | set(cl)), dtype=np.uint64)
    k = n // 50
    pos = rng.integers(0, n, k)
    e = edges[rng.integers(0, edges.size, k)]
    pick = rng.integers(0, 4, k)
    L[pos] = np.minimum(np.select([pick == 0, pick == 1, pick == 2], [e, e + 1, np.maximum(e, 1) - 1],
                                  default=np.full(k, 2**32 - 1)), 2**32 - 1).astype(np.uint32)
    if wide:
        monkeypatch.setenv("FP_SPEC_MIN_WIDE_LOG2", "26")
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_SPECULATE)
    info = fp.fleet_plan_info(plan)
    assert info["lut_cells"] > 0 and info["k3_shape"] == 0
    assert (info["n_edges"] >= 256) == wide and (wide or info["n_edges"] < 127)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    feas = [m for m in range(len(models)) if obest[m]["flags"] & fp.FP_CAND_FEASIBLE]
    if not feas:
        pytest.skip("no model has a feasible split on this random grid")
    model = int(rng.choice(feas))
    dec = torch.full((n,), 0xEE, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(L), cfg.rate_rps, route_model=model, decision=dec)
    assert best.tobytes() == obest.tobytes(), f"seed {seed}: best splits differ"
    bm = obest[model]
    odec, oc = oracle.route_batch(L, int(bm["b_short"]), int(bm["c_short"]), int(bm["c_long"]))
    got = dec.cpu().numpy()
    assert np.array_equal(got, odec), f"seed {seed}: {(got != odec).sum()} decisions differ"
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == \
        [int(x) for x in oc]
    assert fp.fleet_plan_info(plan)["spec_calls"] == 1
    fp.fleet_plan_destroy(plan)
