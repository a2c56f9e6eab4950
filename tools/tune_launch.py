"""Launch-configuration sweep for K1 (trace pass) and K4 (route_batch) on the
C5 trace (1e9 requests). Measurement tool: prints GB/s per configuration."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_08075_b200 as fp  # noqa: E402
from synth import configs  # noqa: E402
from synth.gen import generate_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    cfg = configs.CONFIGS[name]()
    n = cfg.n_requests
    d = generate_device(cfg.shape, cfg.seed, 0, n)
    dec = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = []
    for blk, bps in itertools.product([256, 512], [1, 2, 3, 4, 6, 8]):
        if blk * bps > 2048:
            continue
        os.environ["FP_K1_BLOCK"] = str(blk)
        os.environ["FP_K1_BLOCKS_PER_SM"] = str(bps)
        os.environ["FP_K4_BLOCK"] = str(blk)
        os.environ["FP_K4_BLOCKS_PER_SM"] = str(bps)
        plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_KERNEL_TIMING)
        for _ in range(3):
            fp.sweep_thresholds(plan, d, cfg.rate_rps)
            fp.route_batch(plan, d, 8192, 8192, 65536, decision=dec, want_counts=False)
        torch.cuda.synchronize()
        fp.fp_kernel_time_reset(plan)
        for _ in range(10):
            fp.sweep_thresholds(plan, d, cfg.rate_rps)
            fp.route_batch(plan, d, 8192, 8192, 65536, decision=dec, want_counts=False)
        torch.cuda.synchronize()
        k1 = fp.fp_kernel_time(plan, fp.FP_KERNEL_TRACE)
        k4 = fp.fp_kernel_time(plan, fp.FP_KERNEL_ROUTE)
        info = fp.fleet_plan_info(plan)
        r = {"block": blk, "bps": bps, "k1_grid": info["k1_grid"],
             "k1_ms": k1[0] / k1[1], "k1_GBps": 4 * n / (k1[0] / k1[1] / 1e3) / 1e9,
             "k4_ms": k4[0] / k4[1], "k4_GBps": 5 * n / (k4[0] / k4[1] / 1e3) / 1e9}
        print(json.dumps(r), flush=True)
        out.append(r)
        fp.fleet_plan_destroy(plan)


if __name__ == "__main__":
    main()
