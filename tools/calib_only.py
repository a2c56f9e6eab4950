"""NEXT-3 alone: calibrate_replay over a C5-sized raw feedback stream (profiling driver)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_raw_device

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000_000)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = configs.c5()
body, mo, cat, tp = generate_raw_device(cfg.shape, cfg.seed, 0, args.n)
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
fp.calibrate_replay(plan, body, tp, cat, [(4.0, 0.5)] * 4)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    fp.calibrate_replay(plan, body, tp, cat, [(4.0, 0.5)] * 4)
e1.record()
torch.cuda.synchronize()
print("calibrate_replay ms", e0.elapsed_time(e1) / args.reps)
