"""The step (sweep_and_route, asynchronous device form) captured in a CUDA graph
and replayed, against the same step issued call by call, on C2 (10.3M requests:
launch-bound) and C5 (1e9: HBM-bound). Prints one JSON line per config."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device


def run(cfg, reps=200):
    d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
    dec = torch.empty(cfg.n_requests, dtype=torch.uint8, device="cuda")
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):           # allocations (bins) happen here, outside the capture
            fp.sweep_and_route(plan, d, cfg.rate_rps, decision=dec, stream=s, want_best=False)
    torch.cuda.synchronize()
    ref = fp.best_split(plan).tobytes()
    dref = dec.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # call by call
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            fp.sweep_and_route(plan, d, cfg.rate_rps, decision=dec, stream=s, want_best=False)
    e1.record(s)
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / reps
    # captured
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fp.sweep_and_route(plan, d, cfg.rate_rps, decision=dec, stream=s, want_best=False)
    torch.cuda.synchronize()
    dec.zero_()
    g.replay()
    torch.cuda.synchronize()
    ok = fp.best_split(plan).tobytes() == ref and torch.equal(dec, dref)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    graph_ms = e0.elapsed_time(e1) / reps
    fp.fleet_plan_destroy(plan)
    return {"config": cfg.name, "n": cfg.n_requests, "eager_ms": eager_ms, "graph_ms": graph_ms,
            "graph_requests_per_s": cfg.n_requests / (graph_ms / 1e3), "graph_equals_eager": ok}


if __name__ == "__main__":
    for cfg in (configs.c2(), configs.c5()):
        print(json.dumps(run(cfg, reps=200 if cfg.n_requests < 1e8 else 20)), flush=True)
