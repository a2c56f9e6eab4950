"""Runs the C5 step a few times on a 1e8-request trace (for ncu captures of the K3 cluster shape)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = configs.CONFIGS[name]().with_n(int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000)
d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
dec = torch.empty(cfg.n_requests, dtype=torch.uint8, device="cuda")
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
for _ in range(4):
    fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False)
torch.cuda.synchronize()
print(fp.best_split(plan)["index"], fp.fleet_plan_info(plan))
