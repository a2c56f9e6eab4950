"""NEXT-4 alone: sweep_peak_windows over a C5-sized trace with arrivals (profiling driver)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import arrivals_device, generate_device

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000_000)
ap.add_argument("--window-s", type=float, nargs="+", default=[60, 1])
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = configs.c5()
d = generate_device(cfg.shape, cfg.seed, 0, args.n)
arr = arrivals_device(cfg.seed, args.n, cfg.rate_rps)
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
for ws in args.window_s:
    w = int(ws * 1e9)
    fp.sweep_peak_windows(plan, d, arr, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fp.sweep_peak_windows(plan, d, arr, w)
    e1.record()
    torch.cuda.synchronize()
    print(f"window {ws} s: sweep_peak_windows {e0.elapsed_time(e1) / args.reps:.3f} ms")
