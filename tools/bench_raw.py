"""Measurement tool: the NEXT-1 fused-estimation kernels on the C5 raw columns."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_raw_device
from synth.shapes import CAT_TRUE_RATIO
cfg = configs.c5()
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_requests
body, mo, cat, tp = generate_raw_device(cfg.shape, cfg.seed, 0, n)
cats = [(c * 0.98, 0.1 * c) for c in CAT_TRUE_RATIO]
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg.with_n(n)), flags=fp.FP_FLAG_KERNEL_TIMING)
dec = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    fp.sweep_thresholds_raw(plan, body, mo, cat, cats, cfg.rate_rps)
    fp.route_batch_raw(plan, body, mo, cat, cats, 8192, 8192, 65536, true_prompt=tp, decision=dec)
torch.cuda.synchronize(); fp.fp_kernel_time_reset(plan)
for _ in range(10):
    fp.sweep_thresholds_raw(plan, body, mo, cat, cats, cfg.rate_rps)
    c, mis = fp.route_batch_raw(plan, body, mo, cat, cats, 8192, 8192, 65536, true_prompt=tp, decision=dec)
k1 = fp.fp_kernel_time(plan, fp.FP_KERNEL_TRACE); k4 = fp.fp_kernel_time(plan, fp.FP_KERNEL_ROUTE)
r = {"n": n, "k1_raw_ms": k1[0] / k1[1], "k1_raw_GBps": 9 * n / (k1[0] / k1[1] / 1e3) / 1e9,
     "k4_raw_ms": k4[0] / k4[1], "k4_raw_GBps": 14 * n / (k4[0] / k4[1] / 1e3) / 1e9, "misroute": mis}
print(json.dumps(r))
