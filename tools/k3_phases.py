"""K3 phase timeline (env FP_K3_PHASES=1: %globaltimer stamps of block (0, 0)
in the library, printed at plan destroy) for the step of several configs."""
import os, sys
os.environ["FP_K3_PHASES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device
for name, n in [("C5", 100_000_000), ("C2", 10_300_000), ("C3", 10_000_000), ("C4", 10_000_000), ("C1", 1000)]:
    cfg = configs.CONFIGS[name]().with_n(n)
    d = generate_device(cfg.shape, cfg.seed, 0, n)
    dec = torch.empty(n, dtype=torch.uint8, device="cuda")
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    for _ in range(20):
        fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False)
        fp.best_split(plan)
    print(name, fp.fleet_plan_info(plan)["k3_shape"], fp.fleet_plan_info(plan)["k3_blocks_per_model"], file=sys.stderr, flush=True)
    fp.fleet_plan_destroy(plan)
