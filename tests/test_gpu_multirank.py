"""Multi-rank parity on ONE GPU: two (or four) processes, each a rank of a world-2 (or 4) plan
on cuda:0, with the library's host-collective hooks carried by a gloo process
group (127.0.0.1) instead of NCCL (which refuses two ranks on one device).
This runs the whole world > 1 path of libfleetplan.so -- shard-local K1,
cross-rank histogram sum, candidate slicing, per-rank argmin, all-gather of
best records, rank-order merge, route count sum -- and compares with the CPU
oracle on the whole trace. Only the NCCL calls themselves are not covered.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class GlooCollectives:
    def __init__(self, world):
        self.world = world

    def allreduce_sum_u64(self, a):
        import torch.distributed as dist
        t = torch.from_numpy(a.view(np.int64))
        dist.all_reduce(t)

    def allgather_bytes(self, data):
        import torch.distributed as dist
        arr = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = [torch.empty_like(arr) for _ in range(self.world)]
        dist.all_gather(out, arr)
        return b"".join(o.numpy().tobytes() for o in out)


def _rank(rank, world, port, name, n, flags, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2604_08075_b200 as fp
        from synth import configs
        from synth.gen import generate_device
        cfg = configs.CONFIGS[name]().with_n(n)
        first, count = fp.fp_shard_range(n, rank, world)
        d = generate_device(cfg.shape, cfg.seed, first, count) if count else \
            torch.zeros(0, dtype=torch.int32, device="cuda")
        plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0, rank=rank, world=world,
                                    flags=flags, collectives=GlooCollectives(world))
        if flags & fp.FP_FLAG_P2P:
            # exchange the IPC handles of the K1 accumulators (any host transport)
            handles = [None] * world
            dist.all_gather_object(handles, fp.fp_p2p_export(plan))
            fp.fp_p2p_import(plan, handles)
        res = fp.sweep_thresholds(plan, d, cfg.rate_rps, want_results=True)
        best = fp.best_split(plan)
        edges, cnt, mass = fp.sweep_histogram(plan)
        counts = fp.route_batch(plan, d, 8192, 16384, 65536)
        info = fp.fleet_plan_info(plan)
        # the bench's step on this rank's shard: split picked across ranks on the
        # device (sliced grid: all-gather + k_pick_route), packed or byte bins
        dec = torch.zeros(count, dtype=torch.uint8, device="cuda")
        sbest, _ = fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec)
        q.put((rank, res.tobytes(), best.tobytes(), cnt.tobytes(), mass.tobytes(), counts,
               info["cand_first"], info["cand_count"], None,
               (first, dec.cpu().numpy().tobytes(), sbest.tobytes() if sbest is not None else None)))
        fp.fleet_plan_destroy(plan)
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, None, None, None, None, None, 0, 0, traceback.format_exc(), None))


@pytest.mark.parametrize("name,n,replicated,world", [("C5", 2_000_003, False, 2), ("C3", 300_001, False, 2),
                                                     ("C4", 500_000, True, 2), ("C1", 1000, False, 2),
                                                     ("C5", 1_500_001, "p2p", 2), ("C1", 1000, "p2p", 2),
                                                     ("C5", 1_000_003, False, 4), ("C5", 1_000_003, "p2p", 4),
                                                     ("K3F", 200_003, False, 2), ("K3F", 200_003, "p2p", 2)])
def test_two_ranks_one_gpu_match_oracle(name, n, replicated, world):
    """replicated="p2p": the histogram sum goes through peer memory (FP_FLAG_P2P,
    CUDA IPC between the two processes sharing cuda:0), grid replicated."""
    import oracle
    import paper_2604_08075_b200 as fp
    from synth import configs
    from synth.gen import generate_host
    flags = fp.FP_FLAG_REPLICATED_GRID if replicated else 0
    if replicated == "p2p":
        flags |= fp.FP_FLAG_P2P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, name, n, flags, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert o[8] is None, o[8]
    cfg = configs.CONFIGS[name]().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    allc, obest = oracle.sweep(cfg, L)
    # candidate slices concatenate to the oracle's grid (or each is the whole grid)
    recs = [np.frombuffer(o[1], dtype=fp.FP_CANDIDATE) for o in out]
    if replicated:
        for r in recs:
            assert r.tobytes() == allc.tobytes()
    else:
        assert out[0][6] == 0 and sum(o[7] for o in out) == cfg.n_candidates()
        assert all(out[r][6] + out[r][7] == out[r + 1][6] for r in range(world - 1))
        assert np.concatenate(recs).tobytes() == allc.tobytes()
    for o in out:
        assert o[2] == obest.tobytes()                      # same best split on every rank
        cnt = np.frombuffer(o[3], dtype=np.uint64)
        mass = np.frombuffer(o[4], dtype=np.uint64)
        edges = np.array(sorted(set(cfg.b_short) | set(cfg.c_short) | set(cfg.c_long)), dtype=np.uint32)
        ocnt, omass = oracle.count_le(L, edges)
        assert np.array_equal(np.cumsum(cnt)[:-1], ocnt) and int(cnt.sum()) == n
        assert np.array_equal(np.cumsum(mass)[:-1], omass)
        _, oc = oracle.route_batch(L, 8192, 16384, 65536, want_decisions=False)
        assert [o[5][k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == \
            [int(x) for x in oc]
    # sweep_and_route: every rank routes its shard with the global best split
    b = obest[0]
    odec, _ = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    for o in out:
        first, dec, sbest = o[9]
        if sbest is not None:
            assert sbest == obest.tobytes()
        got = np.frombuffer(dec, dtype=np.uint8)
        assert np.array_equal(got, odec[first:first + got.size])


def _spec_rank(rank, world, port, n, flags, q):
    """FP_FLAG_SPECULATE on a world-2 plan: this rank's shard (>= 2^26 requests)
    is sampled and routed speculatively; the decisions must be those of the
    global best split."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2604_08075_b200 as fp
        from synth import configs
        from synth.gen import generate_device
        cfg = configs.c5().with_n(n)
        first, count = fp.fp_shard_range(n, rank, world)
        d = generate_device(cfg.shape, cfg.seed, first, count)
        plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0, rank=rank, world=world,
                                    flags=flags | fp.FP_FLAG_SPECULATE, collectives=GlooCollectives(world))
        if flags & fp.FP_FLAG_P2P:
            handles = [None] * world
            dist.all_gather_object(handles, fp.fp_p2p_export(plan))
            fp.fp_p2p_import(plan, handles)
        dec = torch.full((count,), 0xEE, dtype=torch.uint8, device="cuda")
        sbest, counts = fp.sweep_and_route(plan, d, cfg.rate_rps, route_model=0, decision=dec)
        info = fp.fleet_plan_info(plan)
        q.put((rank, first, dec.cpu().numpy().tobytes(), sbest.tobytes(), counts, info["spec_calls"], None))
        dist.barrier()
        fp.fleet_plan_destroy(plan)
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, 0, None, None, None, 0, traceback.format_exc()))


@pytest.mark.parametrize("mode", ["sliced", "replicated", "p2p"])
def test_ranks_speculative_match_oracle(mode):
    import oracle
    import paper_2604_08075_b200 as fp
    from synth import configs
    from synth.gen import generate_host
    world, n = 2, 2 * ((1 << 26) + 4_099)
    flags = {"sliced": 0, "replicated": fp.FP_FLAG_REPLICATED_GRID, "p2p": fp.FP_FLAG_P2P}[mode]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spec_rank, args=(r, world, port, n, flags, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert o[6] is None, o[6]
    cfg = configs.c5().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    _, obest = oracle.sweep(cfg, L, want_all=False)
    b = obest[0]
    odec, oc = oracle.route_batch(L, int(b["b_short"]), int(b["c_short"]), int(b["c_long"]))
    for rank, first, dec, sbest, counts, calls, _ in out:
        assert sbest == obest.tobytes()
        assert calls == 1, "the speculative path must have run on every rank"
        got = np.frombuffer(dec, dtype=np.uint8)
        assert np.array_equal(got, odec[first:first + got.size]), f"rank {rank}"
        assert [counts[k] for k in ("n_short", "n_long", "n_reject", "mass_short", "mass_long")] == \
            [int(x) for x in oc]


def _silent_peer(rank, world, port, q):
    """Rank 1 opens the exchange but never sweeps; rank 0's K3 must give up
    waiting (FP_P2P_TIMEOUT_MS) and report FP_ERR_NCCL instead of hanging."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        os.environ["FP_P2P_TIMEOUT_MS"] = "1500"
        import time
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2604_08075_b200 as fp
        from synth import configs
        from synth.gen import generate_device
        cfg = configs.c5().with_n(100_000)
        plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0, rank=rank, world=world,
                                    flags=fp.FP_FLAG_P2P, collectives=GlooCollectives(world))
        handles = [None] * world
        dist.all_gather_object(handles, fp.fp_p2p_export(plan))
        fp.fp_p2p_import(plan, handles)
        status = None
        if rank == 0:
            d = generate_device(cfg.shape, cfg.seed, 0, cfg.n_requests)
            t0 = time.time()
            fp.sweep_thresholds(plan, d, cfg.rate_rps)
            try:
                fp.best_split(plan)
                status = "no error"
            except fp.FleetPlanError as e:
                status = (e.status, time.time() - t0)
            # the error word is cleared: the plan reports it once
        dist.barrier()
        fp.fleet_plan_destroy(plan)
        dist.destroy_process_group()
        q.put((rank, status, None))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_p2p_wait_is_bounded():
    import paper_2604_08075_b200 as fp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_silent_peer, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for o in out:
        assert o[2] is None, o[2]
    status, dt = out[0][1]
    assert status == 7 and 1.0 < dt < 60.0       # FP_ERR_NCCL
