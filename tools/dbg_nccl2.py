import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import oracle, paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_device, generate_host
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
cfg = configs.c5().with_n(1_000_003)
n = cfg.n_requests
L = generate_host(cfg.shape, cfg.seed, 0, n); d = generate_device(cfg.shape, cfg.seed, 0, n)
uid = fp.fp_nccl_get_unique_id()
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0, rank=0, world=1, nccl_unique_id=uid,
                            flags=fp.FP_FLAG_COLLECTIVES | flags)
allc, obest = oracle.sweep(cfg, L)
edges = np.array(sorted(set(cfg.b_short) | set(cfg.c_long)), np.uint32)
ocnt, _ = oracle.count_le(L, edges)
dec = torch.empty(n, dtype=torch.uint8, device="cuda")
def chk(tag):
    e, cnt, mass = fp.sweep_histogram(plan)
    b = fp.best_split(plan)
    print(tag, "hist_ok", np.array_equal(np.cumsum(cnt)[:-1], ocnt), int(cnt.sum()), "best_ok", b.tobytes() == obest.tobytes(), flush=True)
for i in range(3):
    fp.sweep_thresholds(plan, d, cfg.rate_rps); chk(f"sweep{i}")
for i in range(3):
    fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec); chk(f"sar_sync{i}")
for i in range(3):
    fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec, want_best=False); chk(f"sar_async{i}")
