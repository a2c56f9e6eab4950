"""route_batch alone (K4: 4 B in + 1 B decision per request) on the C5 trace, device-timed."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device
cfg = configs.c5()
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_requests
d = generate_device(cfg.shape, cfg.seed, 0, n)
dec = torch.empty(n, dtype=torch.uint8, device="cuda")
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg.with_n(n)), flags=fp.FP_FLAG_KERNEL_TIMING)
for _ in range(3):
    fp.route_batch(plan, d, 8192, 8192, 65536, decision=dec, want_counts=False)
torch.cuda.synchronize(); fp.fp_kernel_time_reset(plan)
for _ in range(20):
    fp.route_batch(plan, d, 8192, 8192, 65536, decision=dec, want_counts=False)
ms, k = fp.fp_kernel_time(plan, fp.FP_KERNEL_ROUTE)
print(json.dumps({"n": n, "k4_ms": ms / k, "k4_GBps": 5.0 * n / (ms / k / 1e3) / 1e9}))
