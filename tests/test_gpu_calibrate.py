"""GPU calibration replay (NEXT-3) against the sequential oracle.

The GPU composes the EMA's affine maps in a parallel scan, so the result is
the sequential replay up to fp64 reassociation: asserted within 1e-12
relative (the north-star FP64 tolerance is 1e-9); counts are exact and the
snapshots at n = snap_at agree to the same tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_08075_b200 as fp  # noqa: E402
from synth import configs  # noqa: E402
from synth.gen import generate_raw_host  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else a).cuda()


def _close(a, b, rel=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    both_nan = np.isnan(a) & np.isnan(b)
    return np.all(both_nan | (np.abs(a - b) <= rel * np.maximum(np.abs(b), 1e-300)))


@pytest.mark.parametrize("stream", [False, True])
@pytest.mark.parametrize("n,ncat,snap", [(1, 4, 1), (37, 4, 5), (100_003, 4, 50), (5_000_000, 4, 1000),
                                         (2_000_001, 3, 50), (300_000, 16, 7),
                                         (3_000_001, 4, 400_000), (1_000_003, 16, 30_000),
                                         (1_062_400, 4, 1), (2_124_801, 2, 500_000)])
def test_replay_matches_sequential(n, ncat, snap, stream, monkeypatch):
    """The two-pass kernels (the default) and the streaming kernel
    (FP_CALIB_STREAM=1: one rank, <= 4 categories; sizes at and around whole
    chunks of 296 x 3,584 records) against the sequential oracle."""
    if stream:
        monkeypatch.setenv("FP_CALIB_STREAM", "1")
    body, mo, cat, tp = generate_raw_host("MIX", 13, 0, n)
    if ncat == 16:
        cat = (np.arange(n) * 7 % 20).astype(np.uint8)       # categories >= 16 -> last (R23)
    tp[::97] = 0                                             # invalid feedback is dropped
    init = [(4.0, 0.5)] * ncat
    plan = fp.fleet_plan_create(**fp.desc_from_config(configs.c1()))
    g = fp.calibrate_replay(plan, _dev(body), _dev(tp), _dev(cat), init, beta=0.95, snap_at=snap)
    o = oracle.calibrate(body, tp, cat, ncat, beta=0.95, c0=4.0, s0=0.5, snap_at=snap)
    assert np.array_equal(g["n_obs"], o["n_obs"])
    assert _close(g["c_hat"], o["c_hat"]) and _close(g["sigma"], o["sigma"])
    assert _close(g["snap_c"], o["snap_c"]) and _close(g["snap_sigma"], o["snap_sigma"])


def test_replay_feeds_the_estimator():
    # calibrate on feedback, then route with the snapshot: the loop of Fig. 5
    n = 1_000_000
    body, mo, cat, tp = generate_raw_host("AZ", 17, 0, n)
    plan = fp.fleet_plan_create(**fp.desc_from_config(configs.c1()))
    g = fp.calibrate_replay(plan, _dev(body), _dev(tp), _dev(cat), [(4.0, 0.5)] * 4)
    cats = list(zip(g["c_hat"], g["sigma"]))
    counts, mis = fp.route_batch_raw(plan, _dev(body), _dev(mo), _dev(cat), cats, 8192, 8192, 65536,
                                     true_prompt=_dev(tp))
    _, _, oc, omis = oracle.route_batch_est(body, mo, cat, tp, cats, 1.0, 0.5, 8192, 8192, 65536)
    assert mis == [int(x) for x in omis]
    static = fp.route_batch_raw(plan, _dev(body), _dev(mo), _dev(cat), [(4.0, 0.0)] * 4, 8192, 8192, 65536,
                                true_prompt=_dev(tp))[1]
    assert mis[0] <= static[0]       # calibration reduces short-pool mis-routes (Table 5)


@pytest.mark.parametrize("shift", [1, 3])
def test_replay_misaligned_columns(shift):
    """Columns that start mid-vector take the scalar staging path for their pieces."""
    n = 777_777
    body, mo, cat, tp = generate_raw_host("MIX", 21, 0, n)
    pad = lambda a: np.concatenate([np.zeros(shift, a.dtype), a])   # noqa: E731
    plan = fp.fleet_plan_create(**fp.desc_from_config(configs.c1()))
    g = fp.calibrate_replay(plan, _dev(pad(body))[shift:], _dev(pad(tp))[shift:], _dev(pad(cat))[shift:],
                            [(4.0, 0.5)] * 4, beta=0.9, snap_at=50)
    o = oracle.calibrate(body, tp, cat, 4, beta=0.9, c0=4.0, s0=0.5, snap_at=50)
    assert np.array_equal(g["n_obs"], o["n_obs"])
    assert _close(g["c_hat"], o["c_hat"]) and _close(g["sigma"], o["sigma"])
    assert _close(g["snap_c"], o["snap_c"]) and _close(g["snap_sigma"], o["snap_sigma"])


@pytest.mark.parametrize("stream", [False, True])
@pytest.mark.parametrize("mode", ["skew", "dropped", "empty", "one_cat", "mixed", "one_sided"])
def test_replay_edge_cases(mode, stream, monkeypatch):
    """A 99%-one-category mix, a stream whose feedback is all dropped, an empty
    stream, one category, a plain mix, a stream whose first half is one
    category and second half another -- through the two-pass kernels (the
    default) and the streaming kernel (FP_CALIB_STREAM=1: its category runs,
    empty lanes and empty categories)."""
    n = 0 if mode == "empty" else 777_777
    body, mo, cat, tp = generate_raw_host("MIX", 29, 0, max(n, 1))
    body, cat, tp = body[:n], cat[:n], tp[:n]
    ncat = 1 if mode == "one_cat" else 4
    if mode == "skew":
        cat = np.where(np.arange(n) % 101 == 0, cat, 2).astype(np.uint8)
    if mode == "dropped":
        tp = np.zeros_like(tp)
    if mode == "one_sided":
        cat = np.where(np.arange(n) < n // 2, 1, 3).astype(np.uint8)
    if stream:
        monkeypatch.setenv("FP_CALIB_STREAM", "1")
    init = [(4.0, 0.5)] * ncat
    plan = fp.fleet_plan_create(**fp.desc_from_config(configs.c1()))
    g = fp.calibrate_replay(plan, _dev(body), _dev(tp), _dev(cat), init, beta=0.95, snap_at=50)
    o = oracle.calibrate(body, tp, cat, ncat, beta=0.95, c0=4.0, s0=0.5, snap_at=50)
    assert np.array_equal(g["n_obs"], o["n_obs"])
    assert _close(g["c_hat"], o["c_hat"]) and _close(g["sigma"], o["sigma"])
    assert _close(g["snap_c"], o["snap_c"]) and _close(g["snap_sigma"], o["snap_sigma"])
