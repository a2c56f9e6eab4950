"""The README usage example, runnable (one B200)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device

cfg = configs.c5()                                   # 1e9 requests, 4 models x 2 GPUs x 64 B x 8 C_L
lens = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)   # u32 L_total column on the device
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_SPECULATE)
dec = torch.empty(cfg.n_requests, dtype=torch.uint8, device="cuda")
best, counts = fp.sweep_and_route(plan, lens, cfg.rate_rps, route_model=0, decision=dec)
#   best: one fp_candidate record per model (cheapest feasible split); dec: Alg. 1's decision bytes
fp.sweep_and_route_graph(plan, lens, cfg.rate_rps, dec)          # the same step as a captured graph
best = fp.best_split(plan)
fp.fleet_plan_destroy(plan)

print('best', best['index'].tolist(), counts)
