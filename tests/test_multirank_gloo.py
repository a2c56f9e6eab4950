"""World-size-2 CPU test of the multi-GPU decomposition (gloo, 127.0.0.1).

On B200s the library shards the trace by global request index
(fp_shard_range), sums per-rank histograms with one NCCL all-reduce, splits
the candidate grid (fp_candidate_range), and merges per-rank best records in
rank order (fp_merge_best). Here each rank plays that protocol with the
oracle standing in for the kernels and gloo for NCCL, and the product's host
helpers doing the partitioning and the merge; the result must equal the
single-process oracle on the whole trace.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n_total, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_2604_08075_b200 as fp
        from synth import configs
        from synth.gen import generate_host

        cfg = configs.CONFIGS[name]().with_n(n_total)
        first, count = fp.fp_shard_range(n_total, rank, world)
        shard = generate_host(cfg.shape, cfg.seed, first, count)
        edges = np.array(sorted(set(cfg.b_short) | set(cfg.c_long)), dtype=np.uint32)
        cnt, mass = oracle.count_le(shard, edges) if count else (np.zeros(len(edges), np.uint64),) * 2
        t = torch.from_numpy(np.concatenate([cnt, mass]).astype(np.int64))
        dist.all_reduce(t)                                   # C1: histogram all-reduce
        full = generate_host(cfg.shape, cfg.seed, 0, n_total)
        fc, fm = oracle.count_le(full, edges)
        ok_hist = np.array_equal(t.numpy(), np.concatenate([fc, fm]).astype(np.int64))

        allc, obest = oracle.sweep(cfg, full)                # candidate records from the global CDF
        allc = allc.view(fp.FP_CANDIDATE)
        c0, cn = fp.fp_candidate_range(cfg.n_candidates(), rank, world)
        mine = allc[c0:c0 + cn]
        local = np.zeros(len(cfg.models), dtype=fp.FP_CANDIDATE)
        for m in range(len(cfg.models)):                     # this rank's per-model argmin (K3)
            sel = mine[(mine["model"] == m) & ((mine["flags"] & fp.FP_CAND_FEASIBLE) != 0)]
            if sel.size:
                j = np.lexsort((sel["index"], sel["cost_dual"]))[0]
                local[m] = sel[j]
            else:
                local[m]["index"] = 0xFFFFFFFF
                local[m]["model"] = m
        gathered = [None] * world
        dist.all_gather_object(gathered, local.tobytes())    # C2: best-record all-gather
        recs = np.frombuffer(b"".join(gathered), dtype=fp.FP_CANDIDATE)
        merged = fp.fp_merge_best(recs, world, len(cfg.models))
        ok_best = merged.tobytes() == obest.view(fp.FP_CANDIDATE).tobytes()
        q.put((rank, bool(ok_hist), bool(ok_best), int(count)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, False, False, repr(e)))


@pytest.mark.parametrize("name,n,world", [("C5", 100_003, 2), ("C3", 50_001, 2), ("C4", 64, 2), ("C5", 100_003, 4),
                                          ("C4", 7, 4), ("C5", 100_003, 8), ("C1", 1000, 8)])
def test_two_rank_protocol_equals_single_process(name, n, world):
    """World 2, 4 and 8 -- the 8-GPU box of SURVEY §8(e) -- (shard invariance;
    C4 with 7 requests leaves ranks empty)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    assert all(r[1] for r in res), res
    assert all(r[2] for r in res), res
    assert sum(r[3] for r in res) == n
