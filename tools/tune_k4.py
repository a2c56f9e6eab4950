"""K4 launch sweep (measurement tool): FP_K4_BLOCK x FP_K4_BLOCKS_PER_SM."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device
cfg = configs.c5()
n = cfg.n_requests
d = generate_device(cfg.shape, cfg.seed, 0, n)
dec = torch.empty(n, dtype=torch.uint8, device="cuda")
for blk, bps in [(512, 2), (512, 3), (512, 4), (256, 4), (256, 6), (256, 8)]:
    os.environ["FP_K4_BLOCK"] = str(blk); os.environ["FP_K4_BLOCKS_PER_SM"] = str(bps)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_KERNEL_TIMING)
    for _ in range(3):
        fp.route_batch(plan, d, 8192, 8192, 65536, decision=dec, want_counts=False)
    torch.cuda.synchronize(); fp.fp_kernel_time_reset(plan)
    for _ in range(10):
        fp.route_batch(plan, d, 8192, 8192, 65536, decision=dec, want_counts=False)
    ms, k = fp.fp_kernel_time(plan, fp.FP_KERNEL_ROUTE)
    print(json.dumps({"lib": os.environ.get("FLEETPLAN_LIB", "default"), "block": blk, "bps": bps,
                      "k4_ms": ms / k, "GBps": 5 * n / (ms / k / 1e3) / 1e9}), flush=True)
    fp.fleet_plan_destroy(plan)
