"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact for every integer (routing counts, histogram, N_seq, instances,
GPUs, argmin index) and for the fp64 fields as well: both sides evaluate
the same IEEE binary64 operations in the same order without contraction
(R14), so the records must agree byte for byte. The north-star
tolerance (|d| <= 1e-9 relative) is asserted too, as the documented bound.
"""
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
from synth.gen import generate_device, generate_host  # noqa: E402

FLOAT_FIELDS = ["alpha", "rho", "predicted_savings", "savings", "cost_dual", "cost_homo",
                "occupancy_short", "occupancy_long"]
INT_FIELDS = [n for n in fp.FP_CANDIDATE.names if n not in FLOAT_FIELDS and n != "_pad"]


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def _compare_records(gpu, ref, what=""):
    assert gpu.shape == ref.shape, what
    for f in INT_FIELDS:
        bad = np.nonzero(gpu[f] != ref[f])[0]
        assert bad.size == 0, f"{what}: field {f} differs at {bad[:5]}: {gpu[f][bad[:5]]} vs {ref[f][bad[:5]]}"
    for f in FLOAT_FIELDS:
        g, r = gpu[f], ref[f]
        # NaN (only from degenerate mu tables, e.g. rho underflowing to 0 with
        # alpha = 0 in alpha (1 - 1/rho)) must be NaN on both sides; IEEE 754
        # leaves NaN payloads unspecified (x86 and the GPU differ), so they are
        # compared as NaN, every other value bit for bit (DESIGN R14)
        both_nan = np.isnan(g) & np.isnan(r)
        assert np.array_equal(np.isnan(g), np.isnan(r)), f"{what}: {f} NaN mismatch"
        both_inf = np.isinf(g) & np.isinf(r) & (np.sign(g) == np.sign(r))
        with np.errstate(invalid="ignore"):
            rel = np.where(both_inf | both_nan, 0.0, np.abs(g - r) / np.maximum(np.abs(r), 1e-300))
        assert np.all(both_inf | both_nan | (rel <= 1e-9)), f"{what}: {f} beyond 1e-9"
        assert np.array_equal(g[~both_nan].view(np.uint64), r[~both_nan].view(np.uint64)), f"{what}: {f} not bit-exact"


def _plan(cfg, **kw):
    return fp.fleet_plan_create(**fp.desc_from_config(cfg), **kw)


def _run_config(cfg, L_host):
    plan = _plan(cfg)
    res = fp.sweep_thresholds(plan, _dev(L_host), cfg.rate_rps, want_results=True)
    best = fp.best_split(plan)
    allc, obest = oracle.sweep(cfg, L_host)
    return plan, res, best, allc, obest


@pytest.mark.parametrize("name,n", [("C1", 1000), ("C2", 1_000_003), ("C3", 200_001), ("C4", 1_000_001),
                                    ("C5", 1_000_007)])
def test_config_parity(name, n):
    cfg = configs.CONFIGS[name]().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    plan, res, best, allc, obest = _run_config(cfg, L)
    _compare_records(res, allc.view(fp.FP_CANDIDATE), name)
    _compare_records(best, obest.view(fp.FP_CANDIDATE), name + " best")
    # histogram = the empirical CDF by definition at every edge
    edges, cnt, mass = fp.sweep_histogram(plan)
    ocnt, omass = oracle.count_le(L, edges)
    assert np.array_equal(np.cumsum(cnt)[:-1], ocnt) and int(cnt.sum()) == n
    assert np.array_equal(np.cumsum(mass)[:-1], omass) and mass[-1] == 0


def test_c1_paper_numbers():
    cfg = configs.c1()
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps)
    b = fp.best_split(plan)[0]
    assert (b["nseq_short"], b["nseq_long"]) == (128, 16)                    # P:40-43 (R10)
    served = (b["n_short"] + b["n_long"]) / cfg.n_requests
    assert b["inst_homo"] == int(np.ceil(served * 1000.0 / 2.8))            # Table 2 rule
    assert b["rho"] == 4.0


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 15, 16, 17, 31, 33, 4095, 32768, 32769, 65536 * 4 + 7])
@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_ragged_and_misaligned(n, offset):
    cfg = configs.c3(n)
    full = generate_host(cfg.shape, cfg.seed, 0, n + offset)
    L = full[offset:]
    d = _dev(full)[offset:]
    plan = _plan(cfg)
    res = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
    allc, _ = oracle.sweep(cfg, L)
    _compare_records(res, allc.view(fp.FP_CANDIDATE), f"n={n} off={offset}")


def test_edge_values_and_skew():
    cfg = make_config("edge", "AZ", 1, 0, 1000.0, ["llama3-70b"], ["b200-180g"],
                      [1, 256, 8192, 65536], [], [65536, 131072])
    rng = np.random.default_rng(0)
    L = np.concatenate([np.zeros(1000, np.uint32), np.full(5000, 8192, np.uint32),
                        np.full(3000, 8193, np.uint32), np.full(17, 2**32 - 1, np.uint32),
                        np.full(100_000, 300, np.uint32),            # all lanes in one bin
                        rng.integers(0, 200_000, 50_000).astype(np.uint32)])
    rng.shuffle(L)
    plan, res, best, allc, obest = _run_config(cfg.with_n(L.size), L)
    _compare_records(res, allc.view(fp.FP_CANDIDATE), "edge")
    _compare_records(best, obest.view(fp.FP_CANDIDATE), "edge best")


def test_large_edge_values_split_mass_and_binary_search():
    # edges up to 2^31 with s = 0 -> LUT too large -> binary-search bins; mass in 16-bit halves
    cfg = make_config("big", "AZ", 1, 0, 1000.0, ["llama3-8b"], ["b200-180g"],
                      [1, 3, 1000, 77777, 2**20 + 1], [], [2**31 - 1, 2**31])
    rng = np.random.default_rng(1)
    L = rng.integers(0, 2**32 - 1, 300_000, dtype=np.uint64).astype(np.uint32)
    L[:100_000] = rng.integers(0, 2**21, 100_000).astype(np.uint32)
    plan, res, best, allc, obest = _run_config(cfg.with_n(L.size), L)
    assert fp.fleet_plan_info(plan)["lut_cells"] == 0
    _compare_records(res, allc.view(fp.FP_CANDIDATE), "big")


def test_many_edges_u16_lut():
    # > 255 bins -> u16 LUT; > ~100 KB lane-private histogram -> shared replica
    b = list(range(16, 16 * 1500, 16))
    cfg = make_config("many", "AZ", 1, 0, 1000.0, ["llama3-8b"], ["b200-180g"], b, [], [65536])
    L = generate_host("AZ", 5, 0, 500_000)
    plan, res, best, allc, obest = _run_config(cfg.with_n(L.size), L)
    _compare_records(res, allc.view(fp.FP_CANDIDATE), "many")
    _compare_records(best, obest.view(fp.FP_CANDIDATE), "many best")


def test_no_mass_flag():
    cfg = configs.c2().with_n(100_000)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg, flags=fp.FP_FLAG_NO_MASS)
    res = fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps, want_results=True)
    allc, _ = oracle.sweep(cfg, L)
    ref = allc.view(fp.FP_CANDIDATE)
    for f in ["n_short", "n_long", "n_reject", "inst_short", "inst_long", "inst_homo", "cost_dual", "flags"]:
        assert np.array_equal(res[f], ref[f])
    assert np.all(res["mass_short"] == 0)


def test_host_pointer_path_matches_device():
    cfg = configs.c5().with_n(3_000_017)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    a = fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps, want_results=True)
    b = fp.sweep_thresholds(plan, L, cfg.rate_rps, want_results=True)                 # pageable host
    pinned = torch.from_numpy(L.view(np.int32)).pin_memory()
    c = fp.sweep_thresholds(plan, pinned, cfg.rate_rps, want_results=True)            # pinned host
    assert a.tobytes() == b.tobytes() == c.tobytes()


def test_empty_trace_and_invalid_args():
    cfg = configs.c1()
    plan = _plan(cfg)
    with pytest.raises(fp.FleetPlanError) as e:
        fp.sweep_thresholds(plan, torch.zeros(0, dtype=torch.int32, device="cuda"), 1000.0)
    assert e.value.status == 3
    with pytest.raises(fp.FleetPlanError):
        fp.best_split(plan)                                                              # no sweep yet
    with pytest.raises(fp.FleetPlanError):
        fp.route_batch(plan, torch.ones(4, dtype=torch.int32, device="cuda"), 9000, 8192, 65536)
    with pytest.raises(fp.FleetPlanError):
        fp.sweep_thresholds(plan, torch.ones(4, dtype=torch.int32, device="cuda"), 0.0)


def test_determinism_and_launch_count():
    cfg = configs.c4().with_n(2_000_000)
    d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    l0 = fp.fp_kernel_launches(plan)
    r1 = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
    r2 = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
    assert r1.tobytes() == r2.tobytes()
    assert fp.fp_kernel_launches(plan) - l0 == 4      # K1 + K3 per sweep


@pytest.mark.parametrize("split", [(8192, 8192, 65536), (1024, 4096, 131072), (1, 1, 1), (300, 300, 300)])
@pytest.mark.parametrize("n,off,doff", [(1, 0, 0), (17, 1, 3), (100_003, 3, 5), (1_000_000, 0, 0)])
def test_route_batch_parity(split, n, off, doff):
    B, CS, CL = split
    full = generate_host("SG", 9, 0, n + off)
    L = full[off:]
    dec = torch.zeros(n + doff + 16, dtype=torch.uint8, device="cuda")
    cfg = configs.c1()
    plan = _plan(cfg)
    counts = fp.route_batch(plan, _dev(full)[off:], B, CS, CL, decision=dec[doff:doff + n])
    odec, ocnt = oracle.route_batch(L, B, CS, CL)
    assert np.array_equal(dec[doff:doff + n].cpu().numpy(), odec)
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in ocnt]
    # the host-trace path gives the same counts
    assert fp.route_batch(plan, L, B, CS, CL) == counts


@pytest.mark.slow
def test_full_size_c5_sampled():
    """C5 at its full size (1e9 requests) in the bench's launch configuration:
    the CUDA generator's trace equals the host generator's on sampled windows,
    the global histogram satisfies the invariants, and sub-ranges of the same
    device trace swept by the same kernels match the oracle exactly."""
    cfg = configs.c5()
    n = cfg.n_requests
    d = generate_device(cfg.shape, cfg.seed, 0, n)
    rng = np.random.default_rng(0)
    for first in rng.integers(0, n - (1 << 20), 3):
        h = generate_host(cfg.shape, cfg.seed, int(first), 1 << 20)
        assert np.array_equal(d[int(first):int(first) + (1 << 20)].cpu().numpy().view(np.uint32), h)
    plan = _plan(cfg)
    fp.sweep_thresholds(plan, d, cfg.rate_rps)
    best = fp.best_split(plan)
    edges, cnt, mass = fp.sweep_histogram(plan)
    assert int(cnt.sum()) == n
    assert np.all(best["n_short"] + best["n_long"] + best["n_reject"] == n)
    for first in rng.integers(0, n - (1 << 24), 2):
        first = int(first) | 1                                       # misaligned on purpose
        L = generate_host(cfg.shape, cfg.seed, first, 1 << 24)
        res = fp.sweep_thresholds(plan, d[first:first + (1 << 24)], cfg.rate_rps, want_results=True)
        allc, _ = oracle.sweep(cfg.with_n(1 << 24), L)
        _compare_records(res, allc.view(fp.FP_CANDIDATE), f"C5 window @{first}")


@pytest.mark.parametrize("where", ["device", "pinned", "pageable"])
def test_sweep_and_route_equals_separate_calls(where):
    cfg = configs.c5().with_n(2_500_009)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    src = {"device": lambda: _dev(L), "pinned": lambda: torch.from_numpy(L.view(np.int32)).pin_memory(),
           "pageable": lambda: L}[where]()
    dec = torch.zeros(L.size, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, src, cfg.rate_rps, route_model=1, decision=dec)
    _, obest = oracle.sweep(cfg, L)
    assert best.tobytes() == obest.tobytes()
    b = obest[1]
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec.cpu().numpy(), odec)
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in oc]


@pytest.mark.parametrize("off,doff", [(0, 0), (1, 0), (2, 5), (3, 3), (0, 7)])
@pytest.mark.parametrize("name", ["C5", "C4", "C2", "C3"])
def test_sweep_and_route_bin_pass_misaligned(name, off, doff):
    # the bin pass (|E| < 256) at every pointer phase; C4 exercises C_S edges
    cfg = configs.CONFIGS[name]().with_n(1_000_003)
    full = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests + off)
    L = full[off:]
    plan = _plan(cfg)
    dec = torch.zeros(L.size + 16, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(full)[off:], cfg.rate_rps, route_model=0, decision=dec[doff:])
    _, obest = oracle.sweep(cfg, L)
    assert best.tobytes() == obest.tobytes()
    b = obest[0]
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec[doff:doff + L.size].cpu().numpy(), odec)
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in oc]
    # the misaligned host path too
    best2, counts2 = fp.sweep_and_route(plan, full[off:], cfg.rate_rps, route_model=0, decision=dec[doff:])
    assert best2.tobytes() == obest.tobytes() and counts2 == counts
    assert np.array_equal(dec[doff:doff + L.size].cpu().numpy(), odec)


def test_sweep_and_route_bin_pass_wide_edges():
    # 200 edges: u8 bins >= 128 -> the byte-wise (non-SWAR) decision path
    cfg = make_config("wide", "SG", 4, 700_001, 10000.0, ["qwen3-235b-a22b"], ["b200-180g"],
                      [256 * k for k in range(1, 200)], [], [65536, 262144])
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    assert fp.fleet_plan_info(plan)["n_edges"] >= 128
    dec = torch.zeros(L.size, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(L), cfg.rate_rps, route_model=0, decision=dec)
    _, obest = oracle.sweep(cfg, L)
    assert best.tobytes() == obest.tobytes()
    b = obest[0]
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec.cpu().numpy(), odec)


@pytest.mark.parametrize("name,model", [("C5", 3), ("C4", 0), ("C3", 2)])
def test_sweep_and_route_async_device_pick(name, model):
    """Asynchronous step (no host outputs): the split is picked and applied on
    the device; decisions and the later best_split equal the oracle's."""
    cfg = configs.CONFIGS[name]().with_n(800_001)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    dec = torch.zeros(L.size, dtype=torch.uint8, device="cuda")
    d = _dev(L)
    for _ in range(2):                       # back-to-back steps on one stream
        assert fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=model, decision=dec, want_best=False) == \
            (None, None)
    best = fp.best_split(plan)
    _, obest = oracle.sweep(cfg, L)
    assert best.tobytes() == obest.tobytes()
    b = obest[model]
    odec, _ = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec.cpu().numpy(), odec)


@pytest.mark.parametrize("n,off,doff", [(1, 0, 0), (3, 1, 0), (5, 3, 1), (17, 2, 0), (1000, 1, 2),
                                        (227_328 * 16 + 7, 0, 0), (227_328 * 16 * 3 + 5, 3, 4),
                                        (2_000_001, 2, 3)])
def test_sweep_and_route_packed_bins_63_edges(n, off, doff):
    """6-bit packed bins at the limit (63 edges -> 64 bins, bins 0..63 all
    used): tiny and ragged traces, every pointer phase of the trace and of the
    decision buffer, and sizes that end exactly on / just past a whole step of
    the trace pass's grid (its chunk layout)."""
    b = [256 * k for k in range(1, 63)]                        # 62 thresholds + C_L = 63 edges
    cfg = make_config("e63", "SG", 9, n, 10000.0, ["qwen3-235b-a22b"], ["b200-180g"], b, [], [262144])
    full = generate_host(cfg.shape, cfg.seed, 0, n + off)
    L = full[off:]
    plan = _plan(cfg)
    assert fp.fleet_plan_info(plan)["n_edges"] == 63
    dec = torch.full((n + 16,), 255, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(full)[off:], cfg.rate_rps, route_model=0, decision=dec[doff:])
    _, obest = oracle.sweep(cfg, L)
    assert best.tobytes() == obest.tobytes()
    bb = obest[0]
    odec, oc = oracle.route_batch(L, int(bb["b_short"]), int(bb["c_short"]), int(bb["c_long"]))
    got = dec.cpu().numpy()
    assert np.array_equal(got[doff:doff + n], odec)
    assert (got[:doff] == 255).all() and (got[doff + n:] == 255).all()     # nothing written outside
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in oc]


@pytest.mark.parametrize("rate", [1e-300, 3.7, 1234.5678, 1e300])
def test_divisions_random_mu_and_rates(rate):
    """K3 forms its quotients by N and by mu with reciprocals and Markstein's
    correction (csrc/k_eval.cu mdiv) when the operands are in range and with
    the IEEE division otherwise; every record must still equal the oracle's
    byte for byte. Random mu over eight decades, all-ones significands, mu far
    outside the range (tiny, subnormal, huge), and rates that push lambda below
    2^-400 and above 2^400 exercise both paths and their boundary; the
    three-pool grid uses the same divisions."""
    rng = np.random.default_rng(int(abs(np.log10(rate))) + 5)
    b = [256 * k for k in range(1, 33)]
    cl = [8192, 16384, 32768]
    base = make_config("mu", "LM", 21, 300_001, rate, ["llama3-8b", "llama3-70b"], ["a100-80g", "b200-180g"],
                       b, [], cl)
    specials = [np.nextafter(2.0, 0.0), np.nextafter(1.0, 0.0) * 8, 1e-320, 2.0 ** -401, 2.0 ** -399,
                2.0 ** 399, 2.0 ** 401, 1e300, 0.0]
    vals = {}
    i = 0
    for m in base.models:
        for g in base.gpus:
            for w in base.windows():
                v = specials[i // 7] if (i % 7 == 3 and i // 7 < len(specials)) else float(10.0 ** rng.uniform(-3, 5))
                vals[(m.name, g.name, int(w))] = v
                i += 1
    from dataclasses import replace
    cfg = replace(base, mu_mode="table", mu_values=vals)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    res = fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps, want_results=True)
    allc, obest = oracle.sweep(cfg, L)
    _compare_records(res, allc, f"rate={rate}")
    _compare_records(fp.best_split(plan), obest, "best")
    n3 = len(cfg.models) * len(cfg.gpus) * len(cl) * (len(b) * (len(b) - 1) // 2)
    r3, b3 = fp.sweep_three_pools(plan, cfg.rate_rps, want_results=True, n_results=n3)
    o3, ob3 = oracle.sweep3(cfg, L)
    assert r3.tobytes() == o3.tobytes()
    assert b3.tobytes() == ob3.tobytes()


def _all_decisions_equal(dec, L, b, what, chunk=1 << 26):
    """Every decision byte of the step against the oracle's Alg. 1 for split b,
    chunk by chunk (no sampling)."""
    n = L.size
    for first in range(0, n, chunk):
        last = min(n, first + chunk)
        odec, _ = oracle.route_batch(L[first:last], int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
        got = dec[first:last].cpu().numpy()
        if not np.array_equal(got, odec):
            bad = np.nonzero(got != odec)[0]
            raise AssertionError(f"{what}: {bad.size} decisions differ in [{first}, {last}), first at {first + bad[0]}")


def _step_against_oracle(cfg, flags=0):
    """The bench's step (sweep_and_route in its asynchronous form, the launch
    configuration bench.py times) at the config's full size, checked
    completely: the step's own histogram (read right after the step, before
    any other sweep) equals count_le at every edge, its best records equal the
    oracle's, and every one of its decision bytes equals Alg. 1 for the
    oracle's best split. Then every candidate record of a records sweep."""
    n = cfg.n_requests
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    d = generate_device(cfg.shape, cfg.seed, 0, n)
    plan = _plan(cfg, flags=flags)
    dec = torch.empty(n, dtype=torch.uint8, device="cuda")
    assert fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False) == (None, None)
    edges, cnt, mass = fp.sweep_histogram(plan)                    # the step's own K1 histogram
    best = fp.best_split(plan)
    ocnt, omass = oracle.count_le(L, edges)
    assert np.array_equal(np.cumsum(cnt)[:-1], ocnt) and int(cnt.sum()) == n
    assert np.array_equal(np.cumsum(mass)[:-1], omass)
    allc, obest = oracle.sweep(cfg, L)
    assert best.tobytes() == obest.tobytes()
    _all_decisions_equal(dec, L, obest[0], cfg.name)
    del dec
    res = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
    _compare_records(res, allc, f"{cfg.name} full")
    return plan


@pytest.mark.slow
def test_full_size_c5_step_against_oracle():
    """C5 (1e9 requests, 4,096 candidates, 6-bit packed bins) -- the bench's
    workload -- on a plan with the bench's flags: all 1e9 decision bytes, the
    step's histogram and best records, then all 4,096 records."""
    _step_against_oracle(configs.c5(), flags=fp.FP_FLAG_TIME_TRACE)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_full_size_configs_against_oracle(name):
    """C1 (1,000), C2 (10.3M), C3 (1e8) and C4 (1e8) at the sizes BASELINE.json
    names, checked as completely as C5: every decision byte of the step, its
    histogram and best records, and every candidate record (up to 30,720)."""
    _step_against_oracle(configs.CONFIGS[name]())


def _big_grid_cfg(tie_mu=False):
    """configs.k3_factored: a grid above the cluster shape's reach (per model >
    8 x 256 x 4), i.e. the factored K3 shape. With tie_mu every window gets the
    same mu, so many candidates tie on cost and the lowest index must win."""
    cfg = configs.k3_factored()
    if tie_mu:
        from dataclasses import replace
        vals = {(m.name, g.name, int(w)): 5.0 for m in cfg.models for g in cfg.gpus for w in cfg.windows()}
        cfg = replace(cfg, mu_mode="table", mu_values=vals)
    return cfg


@pytest.mark.parametrize("tie_mu", [False, True])
def test_factored_k3_matches_oracle(tie_mu, monkeypatch):
    """The factored K3 shape (per-tile instance tables, argmin only) against the
    oracle's argmin and against the grid-stride shape's records; the route
    split it picks drives the step's decisions."""
    cfg = _big_grid_cfg(tie_mu=tie_mu)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    d = _dev(L)
    plan = _plan(cfg)
    assert fp.fleet_plan_info(plan)["k3_shape"] == 1                  # factored
    fp.sweep_thresholds(plan, d, cfg.rate_rps)
    best = fp.best_split(plan)
    allc, obest = oracle.sweep(cfg, L)
    _compare_records(best, obest.view(fp.FP_CANDIDATE), "factored best")
    dec = torch.zeros(L.size, dtype=torch.uint8, device="cuda")
    b2, _ = fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=1, decision=dec)
    assert b2.tobytes() == obest.tobytes()
    _all_decisions_equal(dec, L, obest[1], "factored step")
    # records through the grid-stride shape of the same plan
    res = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
    _compare_records(res, allc.view(fp.FP_CANDIDATE), "factored plan records")
    if tie_mu:
        feas = allc[(allc["model"] == 0) & ((allc["flags"] & 2) != 0)]
        assert (feas["cost_dual"] == feas["cost_dual"].min()).sum() > 1      # real ties exercised


@pytest.mark.parametrize("variant", ["cs_descending", "cheap_gpu", "huge_hours", "huge_rate"])
def test_factored_k3_integer_argmin_fallbacks(variant):
    """k3_factored compares integer GPU counts only when the cost is strictly
    monotone in them and the C_S grid is ascending; these grids take the fp64
    comparison instead (C_S descending; a price below 1/32; hours so large
    that G * price * hours > 2^44; GPU counts above 2^32) and must still give
    the oracle's argmin."""
    from dataclasses import replace
    cfg = configs.k3_factored()
    if variant == "cs_descending":
        cfg = replace(cfg, c_short=tuple(reversed(cfg.c_short)))
    elif variant == "cheap_gpu":
        cfg = replace(cfg, gpus=tuple(replace(g, price_per_gpu_hour=0.01) for g in cfg.gpus))
    elif variant == "huge_hours":
        cfg = replace(cfg, hours_per_year=1e12)
    else:                       # GPU counts above 2^32: the block bound itself disables the integer path
        cfg = replace(cfg, rate_rps=3e13)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    assert fp.fleet_plan_info(plan)["k3_shape"] == 1                  # factored
    fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    _compare_records(fp.best_split(plan), obest.view(fp.FP_CANDIDATE), f"factored {variant}")


@pytest.mark.parametrize("seed", range(6))
def test_factored_k3_random_prices_hours_mu(seed):
    """Random GPU prices (some below 1/32), hours (1 .. 1e12), mu tables and
    C_S orders: the factored shape picks the integer or the fp64 argmin per
    block, and both must give the oracle's best records."""
    from dataclasses import replace
    rng = np.random.default_rng(1000 + seed)
    cfg = configs.k3_factored(n=200_003)
    gpus = tuple(replace(g, price_per_gpu_hour=float(rng.choice([0.01, 0.03, 0.04, 1.0, 3.67, 97.0])))
                 for g in cfg.gpus)
    cs = list(cfg.c_short)
    if rng.random() < 0.5:
        rng.shuffle(cs)
    vals = {(m.name, g.name, int(w)): float(rng.uniform(0.5, 40.0))
            for m in cfg.models for g in cfg.gpus for w in cfg.windows()}
    cfg = replace(cfg, gpus=gpus, c_short=tuple(int(x) for x in cs), mu_mode="table", mu_values=vals,
                  hours_per_year=float(rng.choice([1.0, 8760.0, 3.3e9, 1e12])),
                  rate_rps=float(rng.choice([10.0, 1e4, 1e7])))
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    assert fp.fleet_plan_info(plan)["k3_shape"] == 1                  # factored
    fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    _compare_records(fp.best_split(plan), obest.view(fp.FP_CANDIDATE), f"factored random {seed}")


@pytest.mark.parametrize("shape", ["grid", "factored", "cluster"])
@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_forced_k3_shapes_agree(shape, name, monkeypatch):
    """Every K3 shape (FP_K3_SHAPE forces one at plan creation) gives the
    oracle's best records on the paper-size grids."""
    monkeypatch.setenv("FP_K3_SHAPE", shape)
    cfg = configs.CONFIGS[name]().with_n(300_007)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = _plan(cfg)
    fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    assert fp.best_split(plan).tobytes() == obest.tobytes()


def _escape_cfg(n):
    """|E| = 301 (u16 LUT: clamped-byte bin pass) with a trace almost entirely
    above the 255th edge (65,280), so the best split's B has an edge index
    >= 255 and the routing pass must read L_total back for byte 255."""
    return make_config("ESC", "AZ", 7, n, 1000.0, ["llama3-70b"], ["b200-180g"],
                       [256 * k for k in range(1, 301)], [], [131072])


@pytest.mark.parametrize("off,doff", [(0, 0), (1, 3), (3, 0)])
def test_sweep_and_route_clamped_bins_escape(off, doff):
    n = 300_007
    cfg = _escape_cfg(n)
    rng = np.random.default_rng(11 + off)
    full = rng.integers(65_281, 76_000, n + off, dtype=np.uint64).astype(np.uint32)
    full[rng.random(n + off) < 0.02] = 100                     # a few short requests
    full[rng.random(n + off) < 0.01] = 200_000                 # and rejections
    L = full[off:]
    plan = _plan(cfg)
    assert fp.fleet_plan_info(plan)["n_edges"] >= 256
    dec = torch.zeros(L.size + 16, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route(plan, _dev(full)[off:], cfg.rate_rps, route_model=0, decision=dec[doff:])
    _, obest = oracle.sweep(cfg, L)
    assert best.tobytes() == obest.tobytes()
    b = obest[0]
    edges = sorted(set(cfg.b_short) | set(cfg.c_long))
    assert edges.index(int(b["b_short"])) >= 255, "the split must exercise the escape path"
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    assert np.array_equal(dec[doff:doff + L.size].cpu().numpy(), odec)
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in oc]
