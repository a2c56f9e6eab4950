"""GPU parity of peak-window provisioning (NEXT-4) against the oracle (bit-exact)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_08075_b200 as fp  # noqa: E402
from synth import configs  # noqa: E402
from synth.gen import arrivals_device, arrivals_host, generate_host  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


@pytest.mark.parametrize("name,n,window_s", [("C2", 4_000_003, 60), ("C5", 4_500_000, 10), ("C4", 1_000_001, 1),
                                             ("C1", 1000, 1)])
def test_peak_matches_oracle(name, n, window_s):
    cfg = configs.CONFIGS[name]().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    arr = arrivals_host(cfg.seed, n, cfg.rate_rps)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    res, best = fp.sweep_peak_windows(plan, _dev(L), torch.from_numpy(arr.view(np.int64)).cuda(),
                                      window_s * 10**9, want_results=True)
    oall, obest = oracle.sweep_peak(cfg, L, arr, window_s * 10**9)
    assert res.tobytes() == oall.tobytes()
    assert best.tobytes() == obest.tobytes()


def test_device_arrivals_match_host():
    a = arrivals_device(9, 3_000_001, 10000.0).cpu().numpy().view(np.uint64)
    assert np.array_equal(a, arrivals_host(9, 3_000_001, 10000.0))


@pytest.mark.parametrize("window_ns", [10**6, 10**8])       # ~10 and ~1,000 requests per window
def test_short_windows_and_misaligned_columns(window_ns):
    """Short windows take the global-atomic path; a 1-element offset makes the
    16-B vector loads start mid-column."""
    cfg = configs.c4().with_n(300_001)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    arr = arrivals_host(cfg.seed, cfg.n_requests, cfg.rate_rps)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    dl = _dev(np.concatenate([[0], L]).astype(np.uint32))[1:]
    res, best = fp.sweep_peak_windows(plan, dl, torch.from_numpy(arr.view(np.int64)).cuda(), window_ns,
                                      want_results=True)
    oall, obest = oracle.sweep_peak(cfg, L, arr, window_ns)
    assert res.tobytes() == oall.tobytes()
    assert best.tobytes() == obest.tobytes()


def test_unsorted_arrivals_are_rejected():
    cfg = configs.c2().with_n(100_000)
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    arr = arrivals_host(cfg.seed, cfg.n_requests, cfg.rate_rps)
    d_len = _dev(L)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    bad = arr.copy()
    bad[-1] = 0                                        # last before first: always caught
    with pytest.raises(fp.FleetPlanError):
        fp.sweep_peak_windows(plan, d_len, torch.from_numpy(bad.view(np.int64)).cuda(), 10**8)
    bad = arr.copy()
    bad[5000], bad[5001] = arr[5001] + 1, arr[5000]     # interior swap: caught with FP_FLAG_CHECK_ORDER
    checked = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_CHECK_ORDER)
    with pytest.raises(fp.FleetPlanError):
        fp.sweep_peak_windows(checked, d_len, torch.from_numpy(bad.view(np.int64)).cuda(), 10**8)
    _, best = fp.sweep_peak_windows(checked, d_len, torch.from_numpy(arr.view(np.int64)).cuda(), 10**8)
    _, obest = oracle.sweep_peak(cfg, L, arr, 10**8)
    assert best.tobytes() == obest.tobytes()


@pytest.mark.parametrize("name,window_ns", [("C5", 3 * 10**8), ("C5", 5 * 10**8), ("C5", 2 * 10**9),
                                            ("C3", 5 * 10**8), ("C2", 4 * 10**8)])
def test_windows_of_a_few_thousand_requests(name, window_ns):
    """Windows of ~1K-20K requests (bursty arrivals: sizes vary by phase), so
    K1w switches between its per-window shared histogram (flush per window) and
    the global-atomic path for windows under 2,048 requests inside one block's
    slice; C3 (259 bins) and C2 (65) for wider histograms."""
    n = 3_000_001
    cfg = configs.CONFIGS[name]().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    arr = arrivals_host(cfg.seed, n, 10_000.0)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    res, best = fp.sweep_peak_windows(plan, _dev(L), torch.from_numpy(arr.view(np.int64)).cuda(), window_ns,
                                      want_results=True)
    oall, obest = oracle.sweep_peak(cfg, L, arr, window_ns)
    assert res.tobytes() == oall.tobytes()
    assert best.tobytes() == obest.tobytes()
    fp.fleet_plan_destroy(plan)
