"""sweep_and_route_graph vs the eager asynchronous step (device-timed, back to
back, an L2 flush between steps for traces that fit in L2), per configuration."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="+", default=["C1", "C2", "C3", "C4"])
ap.add_argument("--steps", type=int, default=50)
args = ap.parse_args()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(2 * l2 // 4, dtype=torch.int32, device="cuda")
out = {}
for name in args.configs:
    cfg = configs.CONFIGS[name]()
    n = cfg.n_requests
    d = generate_device(cfg.shape, cfg.seed, 0, n)
    dec = torch.empty(n, dtype=torch.uint8, device="cuda")
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_SPECULATE)
    do_flush = 4 * n < 2 * l2
    res = {}
    for mode in ("eager", "graph", "eager", "graph"):
        for _ in range(3):
            if mode == "graph":
                fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec)
            else:
                fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            if do_flush:
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if mode == "graph":
                fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec)
            else:
                fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False)
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ts)
        res.setdefault(mode, []).append(ms[len(ms) // 2])
    out[name] = {"n": n, "eager_ms_p50": res["eager"], "graph_ms_p50": res["graph"], "l2_flush": do_flush}
    print(name, json.dumps(out[name]), flush=True)
    fp.fleet_plan_destroy(plan)
print(json.dumps(out))
