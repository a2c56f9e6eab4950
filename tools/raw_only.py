"""Runs the NEXT-1 raw sweep on C5 a few times (for ncu captures of the raw K1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_raw_device
from synth.shapes import CAT_TRUE_RATIO
cfg = configs.c5()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 250_000_000
body, mo, cat, tp = generate_raw_device(cfg.shape, cfg.seed, 0, n)
cats = [(c * 0.98, 0.1 * c) for c in CAT_TRUE_RATIO]
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg.with_n(n)))
dec = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    fp.sweep_thresholds_raw(plan, body, mo, cat, cats, cfg.rate_rps)
    fp.route_batch_raw(plan, body, mo, cat, cats, 8192, 8192, 65536, true_prompt=tp, decision=dec)
torch.cuda.synchronize()
