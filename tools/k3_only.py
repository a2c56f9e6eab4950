"""Runs the K3L (2^24 candidates) sweep a few times (for ncu captures of k3_eval)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device
cfg = configs.k3_large()
d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
for _ in range(4):
    fp.sweep_thresholds(plan, d, cfg.rate_rps)
torch.cuda.synchronize()
print(fp.best_split(plan)["index"])
