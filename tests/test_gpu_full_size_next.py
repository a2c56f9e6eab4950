"""Full-size parity of the NEXT rows in the bench's configuration (C5-sized
columns: 1e9 requests / feedback records), against the oracle over the whole
input -- the sizes bench.py times (`slow`; the oracle loops take seconds to
tens of seconds on the box's host cores).

* NEXT-1: sweep_thresholds_raw on the raw columns (body bytes, max_output,
  category) -> every candidate record equals the oracle's estimate + sweep;
  route_batch_raw counts and mis-routes equal the oracle's.
* NEXT-3: calibrate_replay over 1e9 feedback records equals the sequential
  replay to the documented 1e-12 relative tolerance.
* NEXT-4: sweep_peak_windows with 60-s windows: every record byte-identical."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_08075_b200 as fp  # noqa: E402
from synth import configs  # noqa: E402
from synth.gen import arrivals_host, generate_host, generate_raw_host  # noqa: E402
from synth.shapes import CAT_TRUE_RATIO  # noqa: E402

N = 1_000_000_000


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else a).cuda()


def test_next1_full_size():
    cfg = configs.c5()
    body, mo, cat, tp = generate_raw_host(cfg.shape, cfg.seed, 0, N)
    cats = [(c * 0.98, 0.1 * c) for c in CAT_TRUE_RATIO]           # bench.py's snapshot
    db, dm, dc, dt = _dev(body), _dev(mo), _dev(cat), _dev(tp)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    res = fp.sweep_thresholds_raw(plan, db, dm, dc, cats, cfg.rate_rps, want_results=True)
    L = oracle.estimate(body, mo, cat, cats, 1.0, 0.5)
    allc, obest = oracle.sweep(cfg, L)
    assert res.tobytes() == allc.tobytes()
    assert fp.best_split(plan).tobytes() == obest.tobytes()
    counts, mis = fp.route_batch_raw(plan, db, dm, dc, cats, 8192, 8192, 65536, true_prompt=dt)
    _, _, oc, omis = oracle.route_batch_est(body, mo, cat, tp, cats, 1.0, 0.5, 8192, 8192, 65536)
    assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == [int(x) for x in oc]
    assert mis == [int(x) for x in omis]


def test_next3_full_size():
    cfg = configs.c5()
    body, _, cat, tp = generate_raw_host(cfg.shape, cfg.seed, 0, N)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    g = fp.calibrate_replay(plan, _dev(body), _dev(tp), _dev(cat), [(4.0, 0.5)] * 4)   # bench.py's call
    o = oracle.calibrate(body, tp, cat, 4, beta=0.95, c0=4.0, s0=0.5, snap_at=50)
    assert [int(x) for x in g["n_obs"]] == [int(x) for x in o["n_obs"]]
    for key in ("c_hat", "sigma", "snap_c", "snap_sigma"):
        assert np.allclose(g[key], o[key], rtol=1e-12, atol=0, equal_nan=True), key


def test_next4_full_size():
    cfg = configs.c5()
    L = generate_host(cfg.shape, cfg.seed, 0, N)
    arr = arrivals_host(cfg.seed, N, cfg.rate_rps)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    res, best = fp.sweep_peak_windows(plan, _dev(L), torch.from_numpy(arr.view(np.int64)).cuda(), 60 * 10**9,
                                      want_results=True)
    oall, obest = oracle.sweep_peak(cfg, L, arr, 60 * 10**9)
    assert res.tobytes() == oall.tobytes()
    assert best.tobytes() == obest.tobytes()
