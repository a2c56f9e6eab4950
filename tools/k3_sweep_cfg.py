"""K3 launch-shape sweep on the bench's C5 step (device-timed kernel events).
Run once per FP_K3_BLOCK / FP_K3_GRID setting (read at plan creation)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device
cfg = configs.c5().with_n(int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000)
d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_KERNEL_TIMING)
for _ in range(3):
    fp.sweep_thresholds(plan, d, cfg.rate_rps)
torch.cuda.synchronize(); fp.fp_kernel_time_reset(plan)
for _ in range(50):
    fp.sweep_thresholds(plan, d, cfg.rate_rps)
ms, k = fp.fp_kernel_time(plan, fp.FP_KERNEL_EVAL)
info = fp.fleet_plan_info(plan)
print(json.dumps({"block": os.environ.get("FP_K3_BLOCK"), "grid": os.environ.get("FP_K3_GRID"),
                  "eval_us": 1e3 * ms / k, "best": [int(x) for x in fp.best_split(plan)["index"]]}))
