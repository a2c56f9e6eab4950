import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, paper_2604_08075_b200 as fp
from synth import configs
from synth.gen import generate_raw_host
import test_gpu_speculate as T
N = T.N
cfg = configs.c5().with_n(N)
body, mo, cat, _ = generate_raw_host(cfg.shape, cfg.seed, 0, N)
body, mo = body.copy(), mo.copy()
plan = T._plan(cfg)
st = T._sampled_stripes(plan, N, per_thread=2)
print("stripes", st[:3], len(st))
for lo, hi in st:
    body[lo:hi] = 10; mo[lo:hi] = 1
L = oracle.estimate(body, mo, cat, T.CALIB, 1.0, 0.5)
_, obest = oracle.sweep(cfg, L, want_all=False)
b = obest[0]
odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
for rep in range(3):
    dec = torch.full((N,), 0xEE, dtype=torch.uint8, device="cuda")
    best, counts = fp.sweep_and_route_raw(plan, T._raw_dev(body), T._raw_dev(mo), T._raw_dev(cat), T.CALIB, cfg.rate_rps, route_model=0, decision=dec)
    got = dec.cpu().numpy()
    bad = np.nonzero(got != odec)[0]
    info = fp.fleet_plan_info(plan)
    print("rep", rep, "bad", bad.size, bad[:10], got[bad[:10]], odec[bad[:10]], "L", L[bad[:10]], info["spec_calls"], info["spec_misses"], "best", b["b_short"], b["c_short"], b["c_long"])
