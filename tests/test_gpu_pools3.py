"""GPU parity of the three-pool sweep (NEXT-2) against the oracle (bit-exact)."""
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


@pytest.mark.parametrize("name,n", [("C2", 500_003), ("C5", 300_007), ("C1", 1000), ("C3", 20_011)])
def test_three_pools_match_oracle(name, n):
    cfg = configs.CONFIGS[name]().with_n(n)
    if name == "C3":   # keep the oracle's grid small: 64 thresholds
        from dataclasses import replace
        cfg = replace(cfg, b_short=cfg.b_short[::4])
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps)
    oall, obest = oracle.sweep3(cfg, L)
    if len(cfg.b_short) < 2:
        with pytest.raises(fp.FleetPlanError):
            fp.sweep_three_pools(plan, cfg.rate_rps)
        return
    res, best = fp.sweep_three_pools(plan, cfg.rate_rps, want_results=True, n_results=oall.size)
    assert res.tobytes() == oall.tobytes()
    assert best.tobytes() == obest.tobytes()


def test_three_pools_need_windows():
    cfg = configs.c4().with_n(10_000)           # independent C_S grid: B values are not windows
    L = generate_host(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    fp.sweep_thresholds(plan, _dev(L), cfg.rate_rps)
    with pytest.raises(fp.FleetPlanError):
        fp.sweep_three_pools(plan, cfg.rate_rps)
