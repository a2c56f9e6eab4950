"""Benchmark of the fleet-sizing sweep (the north-star hot path) on B200.

One step = the whole hot path of SURVEY.md §8(a) over one batch (the trace):
  sweep_thresholds  (K1 trace pass + histogram, [C1 all-reduce], K3 scan +
                     candidate evaluation + argmin, [C2 all-gather])
  best_split        (per-model best split -> host)
  route_batch       (K4: Alg. 1 for model 0's best split, decision byte per
                     request + global counts -> host)
issued as the single ABI call sweep_and_route.
Default workload: C5 (1e9-request MIX trace per GPU, 4,096 candidates) --
the configuration BASELINE.json's "at 1/2/4/8 B200" metric is quoted on and
the largest single-GPU one. Multi-GPU (torchrun): weak scaling, 1e9 requests
per rank (global index shards of one trace), NCCL inside the library.

`--impl reference` times the CPU oracle (oracle/, as it stands) on bounded
samples of the same workload (the reference arm of this tier).

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace requests routed/s and fleet-sizing candidates/s at 1/2/4/8 B200"
UNIT = "requests/s"
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(workload, kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(workload, {}).get(kernel)
        return float(e["dram_bytes_per_launch"]) if e else None
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index, period_s=0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _l2_bytes(dev=None):
    import torch
    try:
        return int(torch.cuda.get_device_properties(dev or 0).L2_cache_size)
    except Exception:
        return 126 * 2 ** 20


def _l2_label(trace_bytes, l2, flushed):
    if flushed:
        return (f"L2 flushed before every timed step (a {2 * l2 / 1e6:.0f} MB write = 2 x L2) -- the trace "
                f"({trace_bytes / 1e6:.3g} MB) would otherwise stay in the {l2 / 1e6:.0f} MB L2")
    return (f"inputs larger than L2: {trace_bytes / 1e9:.3g} GB trace per GPU > 2 x {l2 / 1e6:.0f} MB L2 "
            f"(no flush needed)")


def _workload(cfg, n_per_rank, world, l2_label=None):
    return {"workload": f"{cfg.name}: {cfg.description}", "name": cfg.name,
            "trace": cfg.shape, "seed": cfg.seed, "n_requests_per_gpu": n_per_rank,
            "n_requests_total": n_per_rank * world, "n_candidates": cfg.n_candidates(),
            "rate_rps": cfg.rate_rps,
            "l2": l2_label or f"inputs larger than L2 (4 B x {n_per_rank:.3g} = {4 * n_per_rank / 1e9:.3g} GB per GPU)",
            "parallelism": f"dp{world} (trace sharded by global request index)"}


def _host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


# ------------------------------------------------------------------ CPU oracle ----
def oracle_step(cfg, L):
    """The hot path on the CPU oracle: sweep + argmin + Alg. 1 route of the
    sample with model 0's best split (same work as one GPU step)."""
    import oracle
    _, best = oracle.sweep(cfg, L, want_all=False)
    b = best[0]
    if b["index"] != 0xFFFFFFFF:
        oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    return best


def _time_oracle(cfg, target_s, n0=1 << 20):
    from synth.gen import generate_host
    L = generate_host(cfg.shape, cfg.seed, 0, n0)
    t = time.perf_counter()
    oracle_step(cfg.with_n(n0), L)
    dt = max(time.perf_counter() - t, 1e-3)
    n = int(min(cfg.n_requests, max(n0, n0 * target_s / dt)))
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    t = time.perf_counter()
    oracle_step(cfg.with_n(n), L)
    return n, time.perf_counter() - t


def cpu_baseline(cfg, target_s=10.0, target_1t_s=8.0):
    """The oracle as it stands on this host: all cores (OpenMP over requests)
    and one thread, each on a bounded sample of the same workload."""
    import oracle
    cores = oracle.num_threads()
    n, dt = _time_oracle(cfg, target_s)
    oracle.set_num_threads(1)
    try:
        n1, dt1 = _time_oracle(cfg, target_1t_s, n0=1 << 18)
    finally:
        oracle.set_num_threads(cores)
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {n:,} requests of the {cfg.name} trace (one oracle step: sweep of all "
                      f"{cfg.n_candidates()} candidates + argmin + Alg. 1 route), {dt:.1f} s on {cores} threads",
            "single_thread": {"value": n1 / dt1, "unit": UNIT, "cores": 1,
                              "sample": f"first {n1:,} requests, {dt1:.1f} s on 1 thread"},
            "host_cpu": _host_cpu()}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from synth.gen import generate_host
    n = args.ref_sample
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    c = cfg.with_n(n)
    for _ in range(args.warmup):
        oracle_step(c, L)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle_step(c, L)
        times.append(time.perf_counter() - t)
    ms = 1e3 * sum(times) / len(times)
    value = n / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
            "config": _workload(cfg, cfg.n_requests, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"each step: first {n:,} requests of the {cfg.name} trace"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ------------------------------------------------------------------ GPU path ----
def next1_fused_estimation(fp, cfg, n, reps=5):
    """NEXT-1: sweep_thresholds_raw / route_batch_raw on raw request columns
    (body bytes, max_output, category, true prompt tokens) of the same trace."""
    import torch
    from synth.gen import generate_raw_device
    from synth.shapes import CAT_TRUE_RATIO
    body, mo, cat, tp = generate_raw_device(cfg.shape, cfg.seed, 0, n)
    cats = [(c * 0.98, 0.1 * c) for c in CAT_TRUE_RATIO]     # a calibrated snapshot (stated)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_KERNEL_TIMING)
    dec = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        fp.sweep_thresholds_raw(plan, body, mo, cat, cats, cfg.rate_rps)
        fp.route_batch_raw(plan, body, mo, cat, cats, 8192, 8192, 65536, true_prompt=tp, decision=dec)
    torch.cuda.synchronize()
    fp.fp_kernel_time_reset(plan)
    for _ in range(reps):
        fp.sweep_thresholds_raw(plan, body, mo, cat, cats, cfg.rate_rps)
        counts, mis = fp.route_batch_raw(plan, body, mo, cat, cats, 8192, 8192, 65536, true_prompt=tp,
                                         decision=dec)
    k1 = fp.fp_kernel_time(plan, fp.FP_KERNEL_TRACE)
    k4 = fp.fp_kernel_time(plan, fp.FP_KERNEL_ROUTE)
    # the whole NEXT-1 workflow in one call (sweep_and_route_raw): speculative
    # (sample, full raw pass writing decisions, verify) vs the three calls
    step_raw = {}
    for mode, flags in (("speculative", fp.FP_FLAG_SPECULATE), ("sequential", 0)):
        pl = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=flags)
        for _ in range(2):
            fp.sweep_and_route_raw(pl, body, mo, cat, cats, cfg.rate_rps, decision=dec, want_best=(flags == 0))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fp.sweep_and_route_raw(pl, body, mo, cat, cats, cfg.rate_rps, decision=dec, want_best=(flags == 0))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        info = fp.fleet_plan_info(pl)
        step_raw[mode] = {"ms": ms, "requests_per_s": n / (ms / 1e3), "spec_calls": info["spec_calls"],
                          "spec_misses": info["spec_misses"]}
        fp.fleet_plan_destroy(pl)
    # NEXT-3: calibration replay of the same stream as feedback (|r|, usage.prompt_tokens, category)
    cal = fp.calibrate_replay(plan, body, tp, cat, [(4.0, 0.5)] * 4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        cal = fp.calibrate_replay(plan, body, tp, cat, [(4.0, 0.5)] * 4)
    e1.record()
    torch.cuda.synchronize()
    cal_ms = e0.elapsed_time(e1) / reps
    fp.fleet_plan_destroy(plan)
    del body, mo, cat, tp, dec
    torch.cuda.empty_cache()
    k1ms, k4ms = k1[0] / k1[1], k4[0] / k4[1]
    return {"n_requests": n, "k1_raw_ms": k1ms, "k1_raw_GBps": 9.0 * n / (k1ms / 1e3) / 1e9,
            "k1_raw_requests_per_s": n / (k1ms / 1e3),
            "k4_raw_ms": k4ms, "k4_raw_GBps": 14.0 * n / (k4ms / 1e3) / 1e9,
            "misroute_short_long_at_8K": mis,
            "step_raw": dict(step_raw, note="sweep_and_route_raw (estimate -> sweep -> argmin -> route) on the raw "
                             "columns: speculative = 9 B read + 1 B written per request in one full pass (+ ~1% "
                             "sample); sequential = sweep_thresholds_raw + host argmin + route_batch_raw"),
            "next3_calibration_replay": {"records": n, "ms": cal_ms, "records_per_s": n / (cal_ms / 1e3),
                                         "GBps": 18.0 * n / (cal_ms / 1e3) / 1e9,
                                         "c_hat": [float(x) for x in cal["c_hat"]],
                                         "note": "two passes (C1 maps, C3 replay) over 9 B/record = 18 B/record; "
                                                 "issue-bound (~60 instructions/record/pass), not HBM-bound"},
            "note": "algorithmic bytes: sweep 9 B/request (bytes u32, max_output u32, category u8); "
                    "route 13 B in + 1 B decision"}


def next4_peak_windows(fp, cfg, n, d_len, reps=3):
    """NEXT-4: peak-window provisioning over the same trace with arrival times
    (windowed 2-D histogram K1w + scan K2w, K3 peak mode)."""
    import torch
    from synth.gen import arrivals_device
    arr = arrivals_device(cfg.seed, n, cfg.rate_rps)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_KERNEL_TIMING)
    out = {"n_requests": n, "span_s": float(arr[-1].item()) / 1e9}
    for wsec in (60, 1):
        w = wsec * 10**9
        fp.sweep_peak_windows(plan, d_len, arr, w)
        torch.cuda.synchronize()
        fp.fp_kernel_time_reset(plan)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            _, best = fp.sweep_peak_windows(plan, d_len, arr, w)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        # per call: the trace timer records two launches per call (K0w+K1w, then K2w)
        kh, nh = fp.fp_kernel_time(plan, fp.FP_KERNEL_TRACE)
        ke, ne = fp.fp_kernel_time(plan, fp.FP_KERNEL_EVAL)
        hist_ms = kh / reps
        out[f"window_{wsec}s"] = {
            "windows": int(out["span_s"] // wsec) + 1, "ms": ms, "requests_per_s": n / (ms / 1e3),
            "hist_ms": hist_ms, "hist_GBps": 4.0 * n / (hist_ms / 1e3) / 1e9,
            "hist_frac": 4.0 * n / (hist_ms / 1e3) / 1e9 / _peaks()[0], "eval_ms": ke / reps,
            "timed_launches_per_call": {"hist": nh / reps, "eval": ne / reps},
            "best_savings_peak": [float(x) for x in best["savings"]],
            "best_gpus_dual_peak": [int(x) for x in best["gpus_dual"]]}
    out["note"] = ("hist = K0w window bounds + K1w 2-D histogram + K2w scan/maxima; algorithmic bytes "
                   "4 B/request (L_total; arrivals are read only at window boundaries, the trace being in "
                   "arrival order); K3 peak reads the per-(B, C_L) window maxima")
    fp.fleet_plan_destroy(plan)
    del arr
    torch.cuda.empty_cache()
    return out


def k3_large_grid(fp, generate_device, reps=5):
    """K3 alone on a 2^24-candidate grid (SURVEY §8(d) ALU regime)."""
    import torch
    from synth import configs
    cfg = configs.k3_large()
    d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_KERNEL_TIMING)
    fp.sweep_thresholds(plan, d, cfg.rate_rps)
    torch.cuda.synchronize()
    fp.fp_kernel_time_reset(plan)
    for _ in range(reps):
        fp.sweep_thresholds(plan, d, cfg.rate_rps)
    ms, k = fp.fp_kernel_time(plan, fp.FP_KERNEL_EVAL)
    best = fp.best_split(plan)
    fp.fleet_plan_destroy(plan)
    per = ms / k
    return {"candidates": cfg.n_candidates(), "k3_ms": per,
            "candidates_per_s": cfg.n_candidates() / (per / 1e3),
            "note": "K3 only (scan + capacity table + fp64 sizing + argmin), results not copied out",
            "best_index_model0": int(best[0]["index"])}


def _bcast_uid(fp, dist, rank):
    """A fresh ncclUniqueId from rank 0 for the library's communicator."""
    obj = [fp.fp_nccl_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def _timed_steps(step, steps, stream, flush=None):
    """Device time of `steps` calls of step() on `stream` (ms, list per step when
    flushing). With `flush` (a tensor of 2 x L2) the L2 is overwritten before
    every step, outside the timed events."""
    import torch
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(k)
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    ev[-1][1].synchronize()
    per = [a.elapsed_time(b) for a, b in ev]
    return sum(per), per


def config_results(fp, names, steps, warmup):
    """BASELINE.json's other configurations (C1-C4) at their full sizes on this
    GPU, the same step (sweep_and_route, asynchronous, FP_FLAG_SPECULATE like
    the main step: speculative where its preconditions hold) timed per step
    with CUDA events, the L2 flushed before every step when the trace would fit
    in it; then the same step replayed as the plan's captured CUDA graph."""
    import torch
    from synth import configs
    from synth.gen import generate_device
    l2 = _l2_bytes()
    peak = _peaks()[0]
    stream = torch.cuda.current_stream()
    flush = torch.empty(2 * l2 // 4, dtype=torch.int32, device="cuda")
    out = {}
    for name in names:
        cfg = configs.CONFIGS[name]()
        n = cfg.n_requests
        d = generate_device(cfg.shape, cfg.seed, 0, n)
        dec = torch.empty(n, dtype=torch.uint8, device="cuda")
        plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), flags=fp.FP_FLAG_SPECULATE)
        step = lambda: fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec,  # noqa: E731
                                          stream=stream, want_best=False)
        for _ in range(warmup):
            step()
        needs_flush = 4 * n < 2 * l2
        l0 = fp.fp_kernel_launches(plan)
        total, per = _timed_steps(step, steps, stream, flush if needs_flush else None)
        launches = fp.fp_kernel_launches(plan) - l0
        best = fp.best_split(plan)
        info = fp.fleet_plan_info(plan)
        # the same step as the plan's captured CUDA graph (sweep_and_route_graph):
        # one graph launch per step instead of the kernel launches
        gstep = lambda: fp.sweep_and_route_graph(plan, d, cfg.rate_rps, dec, stream=stream)  # noqa: E731
        for _ in range(max(warmup, 2)):
            gstep()
        gtotal, gper = _timed_steps(gstep, steps, stream, flush if needs_flush else None)
        gbest = fp.best_split(plan)
        assert gbest.tobytes() == best.tobytes(), f"{name}: graph replay differs from the eager step"
        fp.fleet_plan_destroy(plan)
        if per is None:
            per = [total / steps] * steps
        if gper is None:
            gper = [gtotal / steps] * steps
        per = sorted(per)
        gper = sorted(gper)
        med = per[len(per) // 2]
        ms = total / steps
        # the bytes the step must move at least: the trace read once, one decision byte written
        out[name] = {
            "workload": f"{cfg.name}: {cfg.description}", "n_requests": n, "n_candidates": cfg.n_candidates(),
            "ms_per_step": ms, "ms_p10_p50_p90": [per[int(0.1 * (steps - 1))], med, per[int(0.9 * (steps - 1))]],
            "requests_per_s": n / (ms / 1e3), "candidates_per_s_step": cfg.n_candidates() / (ms / 1e3),
            "step_min_bytes_per_request": 5.0,
            "step_frac_min_bytes": 5.0 * n / (ms / 1e3) / 1e9 / peak,
            "l2": _l2_label(4 * n, l2, needs_flush), "gpu_launches_per_step": launches / steps,
            "speculative": bool(info["spec_calls"]),
            "graph": {"ms_per_step": gtotal / steps,
                      "ms_p10_p50_p90": [gper[int(0.1 * (steps - 1))], gper[len(gper) // 2],
                                         gper[int(0.9 * (steps - 1))]],
                      "requests_per_s": n / (gtotal / steps / 1e3),
                      "note": "sweep_and_route_graph: the same step replayed as the plan's captured CUDA graph"},
            "k3_shape": ["cluster", "factored", "grid"][info["k3_shape"]],
            "best_model0": {"index": int(best[0]["index"]), "b_short": int(best[0]["b_short"]),
                            "c_short": int(best[0]["c_short"]), "c_long": int(best[0]["c_long"]),
                            "savings": float(best[0]["savings"])}}
        del d, dec
        torch.cuda.empty_cache()
    del flush
    torch.cuda.empty_cache()
    return out


def multi_variants(fp, dist, cfg, n_weak, rank, world, local, steps, warmup, spec_flag=0):
    """The multi-GPU step under each exchange / grid mode, weak (n_weak
    requests per rank) and strong (the config's trace split over the ranks):
    NCCL all-reduce with the grid replicated or sliced across ranks (+ the
    all-gather of best records), and the peer-memory exchange (FP_FLAG_P2P,
    grid replicated). Device time, max over ranks."""
    import torch
    from synth.gen import generate_device
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    out = []
    for strong in (False, True):
        if strong:
            first, n = fp.fp_shard_range(cfg.n_requests, rank, world)
        else:
            first, n = rank * n_weak, n_weak
        c = cfg.with_n(n)
        d = generate_device(c.shape, c.seed, first, n)
        dec = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        for mode in ("nccl-replicated", "nccl-sliced", "p2p"):
            flags = fp.FP_FLAG_COLLECTIVES | spec_flag
            if mode != "nccl-sliced":
                flags |= fp.FP_FLAG_REPLICATED_GRID
            if mode == "p2p":
                flags |= fp.FP_FLAG_P2P
            plan = fp.fleet_plan_create(**fp.desc_from_config(c), device=local, rank=rank, world=world,
                                        nccl_unique_id=_bcast_uid(fp, dist, rank), flags=flags)
            if mode == "p2p":
                handles = [None] * world
                dist.all_gather_object(handles, fp.fp_p2p_export(plan))
                fp.fp_p2p_import(plan, handles)
            step = lambda: fp.sweep_and_route(plan, d, c.rate_rps, route_model=0, decision=dec,  # noqa: E731
                                              stream=stream, want_best=False)
            for _ in range(warmup):
                step()
            dist.barrier(device_ids=[local])
            torch.cuda.synchronize(dev)
            ms, _ = _timed_steps(step, steps, stream)
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_step = float(t.item()) / steps
            best = fp.best_split(plan)
            dist.barrier(device_ids=[local])       # peers may still read a P2P buffer
            fp.fleet_plan_destroy(plan)
            total = cfg.n_requests if strong else n_weak * world
            spec = fp.fleet_plan_info(plan)["spec_calls"] > 0
            out.append({"scaling": "strong" if strong else "weak", "exchange": mode, "n_gpus": world,
                        "ms_per_step": ms_step, "requests_per_s": total / (ms_step / 1e3),
                        "best_index_model0": int(best[0]["index"]), "speculative": spec})
        del d, dec
        torch.cuda.empty_cache()
    return out


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2604_08075_b200 as fp
    from synth.gen import generate_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # --collectives: the multi-GPU code path at world 1 (process group, NCCL
    # unique-id broadcast, the library's one-rank communicator, max-over-ranks)
    multi = world > 1 or args.collectives
    if multi:
        dist.init_process_group("nccl", device_id=dev)
    n = args.n or cfg.n_requests
    if args.strong:
        # strong scaling: the config's trace split over the ranks (global-index
        # shards, fp_shard_range's rounding), instead of n requests per rank
        first, n = fp.fp_shard_range(n, rank, world)
    else:
        first = rank * n
    n_weak = args.n or cfg.n_requests
    cfg = cfg.with_n(n)

    uid = _bcast_uid(fp, dist, rank) if multi else None
    # the timed loop's plan records CUDA events around the trace pass (the
    # dominant kernel, for the roofline) only: an event pair costs a few us of
    # stream time, and timing K3 and K4 too would add ~16 us to every step
    # (1.5% of C5's, a third of C2's); the per-kernel breakdown is a second loop
    coll = fp.FP_FLAG_COLLECTIVES if multi else 0
    # speculative routing (FP_FLAG_SPECULATE, fleet_plan.h): the library applies
    # it where it can (one rank, device trace, |E| < 127, >= 2^26 requests) and
    # falls back otherwise; results are identical either way
    spec_flag = fp.FP_FLAG_SPECULATE if args.speculate else 0
    if multi and args.p2p:
        coll |= fp.FP_FLAG_P2P
    # the north star's split: the candidate grid is sliced over the ranks and
    # the per-model winners are gathered (argmin reduce). --replicated-grid
    # evaluates the whole (small) grid on every rank instead -- K3 is latency-
    # bound at C5's 4,096 candidates, so that skips the all-gather and the
    # pick kernel; the variants block times both
    if multi and args.replicated_grid:
        coll |= fp.FP_FLAG_REPLICATED_GRID

    def p2p_setup(pl):
        # FP_FLAG_P2P: all-gather the ranks' IPC handles, open the peers' buffers
        if coll & fp.FP_FLAG_P2P:
            handles = [None] * world
            dist.all_gather_object(handles, fp.fp_p2p_export(pl))
            fp.fp_p2p_import(pl, handles)
    plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=local, rank=rank, world=world,
                                nccl_unique_id=uid,
                                flags=(0 if args.no_kernel_events else fp.FP_FLAG_TIME_TRACE) | coll | spec_flag)
    p2p_setup(plan)
    info = fp.fleet_plan_info(plan)
    if multi:
        print(f"[bench] rank {rank}/{world}: NCCL communicator of {info['nccl_comm_size']} ranks "
              f"(device {local})", file=sys.stderr, flush=True)
    # this rank's shard of the global trace: requests [rank*n, (rank+1)*n)
    d_len = generate_device(cfg.shape, cfg.seed, first, n)
    d_dec = torch.empty(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    l2 = _l2_bytes(local)
    needs_flush = 4 * n < 2 * l2
    flush = torch.empty(2 * l2 // 4, dtype=torch.int32, device=dev) if needs_flush else None

    def step(lengths, want_best=False, pl=None):
        # sweep_thresholds -> per-model argmin -> route_batch(model 0's best split), one ABI call;
        # the device-timed steps leave the best records on the device (asynchronous call)
        return fp.sweep_and_route(pl or plan, lengths, cfg.rate_rps, route_model=0, decision=d_dec, stream=stream,
                                  want_best=want_best)

    def barrier():
        if multi:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step(d_len)
    barrier()
    if not args.no_kernel_events:
        fp.fp_kernel_time_reset(plan)
    l0 = fp.fp_kernel_launches(plan)
    with ClockSampler(local) as clk:
        barrier()
        ms_local, _ = _timed_steps(lambda: step(d_len), args.steps, stream, flush)
        torch.cuda.synchronize(dev)
    barrier()
    best = fp.best_split(plan)                  # the records of the last timed step
    launches = fp.fp_kernel_launches(plan) - l0
    info = fp.fleet_plan_info(plan)             # (+ the speculation counters of the timed steps)
    k1_time = (0.0, 0) if args.no_kernel_events else fp.fp_kernel_time(plan, fp.FP_KERNEL_TRACE)

    # ---- per-kernel breakdown and per-step spread: a second loop on a plan that
    # times every kernel (not part of the headline value) ----
    plan_b = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=local, rank=rank, world=world,
                                  nccl_unique_id=_bcast_uid(fp, dist, rank) if multi else None,
                                  flags=fp.FP_FLAG_KERNEL_TIMING | coll | spec_flag)
    p2p_setup(plan_b)
    for _ in range(2):
        step(d_len, pl=plan_b)
    barrier()
    fp.fp_kernel_time_reset(plan_b)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record(stream)
    for k in range(args.steps):
        step(d_len, pl=plan_b)
        ev[k + 1].record(stream)
    torch.cuda.synchronize(dev)
    per_step = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps))
    pct = lambda q: per_step[min(len(per_step) - 1, int(q * len(per_step)))]   # noqa: E731
    ktime = {k: fp.fp_kernel_time(plan_b, kind) for k, kind in
             (("trace", fp.FP_KERNEL_TRACE), ("eval", fp.FP_KERNEL_EVAL), ("route", fp.FP_KERNEL_ROUTE))}
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if multi:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    total_requests = (args.n or cfg.n_requests) if args.strong else n * world
    value = total_requests / (ms_step / 1e3)

    # ---- NEXT-2: three pools over the same histogram (rank-local, no collective) ----
    next2 = None
    if args.next2:
        fp.fp_kernel_time_reset(plan_b)        # (its last sweep's histogram)
        for _ in range(3):
            _, best3 = fp.sweep_three_pools(plan_b, cfg.rate_rps)
        ms3, k3n = fp.fp_kernel_time(plan_b, fp.FP_KERNEL_EVAL)
        nb = len(cfg.b_short)
        n3 = len(cfg.models) * len(cfg.gpus) * len(cfg.c_long) * nb * (nb - 1) // 2
        next2 = {"candidates": n3, "k3_three_pool_ms": ms3 / k3n,
                 "candidates_per_s": n3 / (ms3 / k3n / 1e3),
                 "best_savings_two_pools": [float(x) for x in best["savings"]],
                 "best_savings_three_pools": [float(x) for x in best3["savings"]],
                 "note": "P:1099-1100 claims ~2% marginal savings for a third pool; under the stated "
                         "uncapped pow23 mu the gain is larger (it depends on mu saturation, not stated)"}
    if multi:
        barrier()
    fp.fleet_plan_destroy(plan_b)

    # ---- e2e: the same step through the C ABI with HOST (pinned) buffers ----
    e2e = None
    if args.e2e_steps > 0:
        h_len = d_len.cpu().pin_memory()
        step(h_len, want_best=True)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            step(h_len, want_best=True)
        barrier()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if multi:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e_value = total_requests * args.e2e_steps / float(dt.item())
        # the link's own rate: a plain pinned H2D copy of 1 GB of this trace (device-timed)
        hb = h_len[: min(n, 1 << 28)]
        db = torch.empty_like(hb, device=dev)
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            db.copy_(hb, non_blocking=True)
            e1.record()
            e1.synchronize()
        h2d_gbps = 4 * hb.numel() / (e0.elapsed_time(e1) * 1e6)
        del db, hb
        e2e = {"value": e2e_value, "unit": UNIT,
               "h2d_bytes_per_step": 4 * n,   # the pinned trace crosses PCIe once per step
               "d2h_bytes_per_step": best.nbytes + 5 * 8,
               "h2d_GBps_step": 4 * n * e2e_value / total_requests / 1e9,
               "h2d_GBps_copy": h2d_gbps,
               "frac_of_h2d_copy": 4 * n * e2e_value / total_requests / 1e9 / h2d_gbps,
               "note": "sweep_and_route on a pinned host trace: 128 MB chunks DMA'd into the device while K1 "
                       "consumes them (bins written on the device), K4 routes from the bins; best records + "
                       "route counts to host every step"}
        del h_len

    # ---- the multi-GPU exchange / grid variants (N > 1, or --collectives at N = 1) ----
    variants = None
    if multi and args.variants:
        barrier()
        variants = multi_variants(fp, dist, cfg, n_weak, rank, world, local, steps=max(5, args.steps // 2),
                                  warmup=3, spec_flag=spec_flag)

    if rank != 0:
        barrier()
        fp.fleet_plan_destroy(plan)
        if multi:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    peak, peak_src = _peaks()
    shares = {k: v[0] for k, v in ktime.items()}
    dom = max(shares, key=shares.get)
    # bytes each kernel moves per step as designed: with the bin
    # pass (a fine-cell LUT and a device trace: u8 bins for |E| < 256, clamped
    # bytes above) the trace pass reads 4 B and writes a bin per request
    # (6-bit packed: 0.75 B; else 1 B) and the routing pass maps the bins to
    # 1-B decisions; otherwise the routing pass re-reads L_total.
    bin_pass = info["lut_cells"] > 0
    speculative = info["spec_calls"] > 0
    packed = bin_pass and info["n_edges"] + 1 <= 64 and not speculative
    bin_bytes = 0.75 if packed else 1.0
    moved = ({"trace": (4.0 + bin_bytes) * n, "route": (bin_bytes + 1.0) * n, "eval": 0.0} if bin_pass
             else {"trace": 4.0 * n, "route": 5.0 * n, "eval": 0.0})
    if speculative:
        # the full trace pass reads L_total and writes the decision byte; the
        # verify kernel reads two 16-B splits (re-routing only on a miss)
        moved = {"trace": 5.0 * n, "route": 0.0, "eval": 0.0}
    # SURVEY §8(d)'s algorithmic bytes: the sweep pass reads 4 B per request;
    # route_batch reads 4 B and writes 1 B (the bins are this design's, not the method's)
    algo = {"trace": 4.0 * n, "route": 5.0 * n, "eval": 0.0}
    algo_note = "SURVEY §8(d): the sweep's trace pass reads 4 B per request"
    if speculative:
        # the speculative full pass does both §8(d) passes at once: the sweep's
        # 4-B read and route_batch's 1-B decision write (its 4-B read is the same read)
        algo = {"trace": 5.0 * n, "route": 0.0, "eval": 0.0}
        algo_note = ("SURVEY §8(d): the sweep reads 4 B per request and route_batch writes a 1-B decision; the "
                     "speculative full trace pass does both, so its minimum is 5 B per request (the verify kernel "
                     "reads 32 B per step)")
    kms, kcount = k1_time if dom == "trace" else ktime[dom]
    per_launch_ms = kms / max(kcount, 1)
    per_launch_bytes = algo[dom] / max(1.0, kcount / args.steps)   # bytes per step / launches per step
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else float("nan")
    moved_gbs = moved[dom] / max(1.0, kcount / args.steps) / (per_launch_ms / 1e3) / 1e9 if per_launch_ms else None
    k_gbs = {k: (moved[k] * args.steps / (ktime[k][0] / 1e3) / 1e9 if ktime[k][0] and moved[k] else None)
             for k in ktime}
    kname = {"trace": "K1 k1_trace" + ((" (6-bit packed bin pass)" if packed else " (bin pass)") if bin_pass else ""),
             "route": ("K4p k4_route_packed" if packed else "K4b k4_route_bins") if bin_pass else "K4 k4_route"}
    if speculative:
        kname = {"trace": "K1 k1_trace (decision-writing pass for the sampled split)", "route": "K4v k4_route_verify"}
    # the step's DRAM traffic as ncu measured it (profiles/ncu_traffic.json, --set full)
    step_dram = None
    tkey = cfg.name + ("-spec" if speculative else "")     # ncu_traffic.json workload key
    if all(_traffic(tkey, k) for k in ("trace", "route")):
        step_dram = sum(_traffic(tkey, k) or 0.0 for k in ("trace", "route", "eval", "sample", "sample_eval"))
    roof = {"bound": "hbm", "kernel": kname.get(dom, dom),
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": _traffic(tkey, dom), "peak_source": peak_src,
            "algorithmic_bytes_per_launch": per_launch_bytes,
            "algorithmic_bytes_per_request": algo[dom] / n,
            "algorithmic_bytes_note": algo_note,
            "bytes_moved_per_request": moved[dom] / n,
            "achieved_bytes_moved": moved_gbs, "frac_bytes_moved": moved_gbs / peak if moved_gbs else None,
            "frac_of_nominal_7700": achieved / 7700.0,
            "per_kernel_GBps_bytes_moved": k_gbs,
            "step_share": {k: v / sum(per_step) for k, v in shares.items()},   # breakdown loop
            "step_dram_bytes_per_request_ncu": step_dram / 1e9 if step_dram and cfg.n_requests == 10**9 else None,
            "step_frac_dram_ncu": (step_dram / (ms_step / 1e3) / 1e9 / peak
                                   if step_dram and n == 10**9 else None)}
    cand_per_s = cfg.n_candidates() * args.steps / (ktime["eval"][0] / 1e3) if ktime["eval"][0] else None

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "ms_per_step_p10_p50_p90": [pct(0.1), pct(0.5), pct(0.9)],
            "vs_baseline": None, "dtype": "u32/f64",
            "data": "synthetic (seeded Philox MIX trace, generated on device; not timed)",
            "step": (("sweep_and_route with speculative routing (FP_FLAG_SPECULATE): K1s sample pass (~2% of the "
                      "trace in grid-wide stripes) -> K3s sampled split -> K1 full trace pass writing the decision "
                      "bytes for it -> K3 sweep + per-model argmin -> K4v verify (re-routes every request from "
                      "L_total if the split differs); results identical to the non-speculative step"
                      if speculative else
                      "sweep_and_route: K1 trace pass (+6-bit packed bins) -> K3 sweep + per-model argmin -> "
                      "device split pick -> K4p routing pass")
                     + ", stream-ordered with no host round trip; the best records stay on the device and are "
                       "read once after the timed loop (e2e reads them every step)"),
            "speculation": ({"calls": info["spec_calls"], "misses": info["spec_misses"]}
                            if speculative else None),
            "config": dict(_workload(cfg, n, world, _l2_label(4 * n, l2, needs_flush)),
                           n_requests_total=total_requests),
            "candidates_per_s": cand_per_s,
            "candidates_per_s_step": cfg.n_candidates() / (ms_step / 1e3),
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in ktime.items()},
            "kernel_timing": ("timed loop: CUDA events around the trace pass only (value, roofline); "
                              "kernel_ms_per_step, step_share and the p10/p50/p90 from a second loop of "
                              "the same steps on a plan that times every kernel (~16 us of event overhead "
                              "per step)"),
            "roofline": roof,
            "gpu_launches": launches,
            "k3_shape": ["cluster", "factored", "grid"][info["k3_shape"]],
            "next2_three_pools": next2,
            "clocks": clk.summary(),
            "e2e": e2e,
            "variants": variants,
            "configs": None,
            "best_split_model0": {k: (int(best[0][k]) if k not in ("cost_dual", "savings", "predicted_savings")
                                      else float(best[0][k]))
                                  for k in ("index", "b_short", "c_short", "c_long", "gpus_dual", "gpus_homo",
                                            "cost_dual", "savings", "predicted_savings")},
            "plan": {k: info[k] for k in ("n_edges", "lut_shift", "lut_cells", "k1_grid", "k1_block", "sm_count",
                                          "nccl_comm_size", "k3_blocks_per_model")}}
    if multi and world == 1:
        line["config"]["parallelism"] += "; --collectives: one-rank NCCL communicator in the step"
    if coll & fp.FP_FLAG_P2P:
        line["config"]["parallelism"] += "; --p2p: histogram sum over peer memory in K3 (no all-reduce)"
    if coll & fp.FP_FLAG_REPLICATED_GRID:
        line["config"]["parallelism"] += "; candidate grid replicated on every rank (no all-gather)"
    if multi:
        barrier()
    fp.fleet_plan_destroy(plan)
    del d_dec
    if world == 1 and args.k3_grid:
        line["k3_large_grid"] = k3_large_grid(fp, generate_device)
    if world == 1 and args.next4:
        line["next4_peak_windows"] = next4_peak_windows(fp, cfg, n, d_len)
    if world == 1 and args.configs:
        del d_len
        torch.cuda.empty_cache()
        line["configs"] = config_results(fp, [c for c in ("C1", "C2", "C3", "C4") if c != cfg.name],
                                         steps=max(10, args.steps), warmup=args.warmup)
    if world == 1 and args.next1:
        d_len = None
        torch.cuda.empty_cache()
        line["next1_fused_estimation"] = next1_fused_estimation(fp, cfg, n)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    emit(line)
    if multi:
        dist.destroy_process_group()


_JSON_OUT = None


def emit(line):
    """The one JSON line on stdout. Everything else that writes to fd 1 (NCCL's
    version banner at communicator init, library diagnostics) is sent to
    stderr by main(), so stdout carries exactly this line."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def _spawn_ranks(gpus):
    """`bench.py --gpus N` (N > 1) without a launcher: re-run this command as N
    ranks under torch.distributed.run (127.0.0.1 rendezvous); rank 0 prints the
    line. Returns the launcher's exit code."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print("[bench] spawning: " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def run_plumbing_check(args):
    """CPU check of the multi-rank plumbing the GPU arm uses (launcher, env,
    process group on 127.0.0.1, max over ranks, rank-0-only output) with gloo."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ranks = [None] * world
    dist.all_gather_object(ranks, {"rank": rank, "local_rank": int(os.environ.get("LOCAL_RANK", "0"))})
    if rank == 0:
        emit({"plumbing": "ok", "n_gpus": world, "max_over_ranks": float(t.item()), "ranks": ranks})
    dist.destroy_process_group()


def main():
    global _JSON_OUT
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=0, help="requests per GPU (default: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="diagnostic: no per-kernel CUDA events in the timed loop (no roofline)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the config's trace over the ranks (default: weak, n per rank)")
    ap.add_argument("--collectives", action="store_true",
                    help="take the multi-GPU code path even at world 1 (NCCL group of one; for testing)")
    ap.add_argument("--no-speculate", dest="speculate", action="store_false",
                    help="no speculative routing (FP_FLAG_SPECULATE) in the step: the bin-pass step instead")
    ap.add_argument("--replicated-grid", action="store_true",
                    help="multi-rank: evaluate the whole candidate grid on every rank (no all-gather) "
                         "instead of the default split + argmin gather")
    ap.add_argument("--sliced-grid", action="store_true",
                    help="(the default at N > 1; kept for compatibility)")
    ap.add_argument("--p2p", action="store_true",
                    help="multi-rank: the histogram exchange through peer memory (FP_FLAG_P2P) instead of NCCL")
    ap.add_argument("--no-variants", dest="variants", action="store_false",
                    help="multi-rank: skip the NCCL/P2P x replicated/sliced x weak/strong variant timings")
    ap.add_argument("--no-configs", dest="configs", action="store_false",
                    help="skip the C1-C4 per-configuration results")
    ap.add_argument("--no-next2", dest="next2", action="store_false",
                    help="skip the three-pool (NEXT-2) measurement")
    ap.add_argument("--no-next1", dest="next1", action="store_false",
                    help="skip the fused token-budget estimation measurement (NEXT-1)")
    ap.add_argument("--no-next4", dest="next4", action="store_false",
                    help="skip the peak-window provisioning measurement (NEXT-4)")
    ap.add_argument("--no-k3-grid", dest="k3_grid", action="store_false",
                    help="skip the 2^24-candidate K3 measurement")
    ap.add_argument("--ref-sample", type=int, default=10_000_000,
                    help="requests per reference (oracle) step")
    ap.add_argument("--plumbing-check", action="store_true",
                    help="CPU: exercise the multi-rank launch / gloo / rank-0 output path only")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(_spawn_ranks(args.gpus))
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.plumbing_check:
        run_plumbing_check(args)
        return
    from synth import configs
    cfg = configs.CONFIGS[args.config]()
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
