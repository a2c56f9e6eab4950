"""World-2 parity of the NEXT rows on ONE GPU (gloo host-collective hooks, as
tests/test_gpu_multirank.py): calibration replay (the feedback stream sharded
in order; ranks exchange their composed EMA maps) and peak-window
provisioning (the trace and its arrival times sharded; ranks sum their
window x bin histograms). Each rank's result must equal the oracle's on the
whole stream."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

from test_gpu_multirank import GlooCollectives, _free_port  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else a).cuda()


def _rank(rank, world, port, job, n, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2604_08075_b200 as fp
        from synth import configs
        from synth.gen import arrivals_host, generate_host, generate_raw_host
        first, count = fp.fp_shard_range(n, rank, world)
        if job == "calib":
            cfg = configs.c1()
            body, mo, cat, tp = generate_raw_host("MIX", 31, 0, n)
            tp[::89] = 0
            sl = slice(first, first + count)
            plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0, rank=rank, world=world,
                                        collectives=GlooCollectives(world))
            g = fp.calibrate_replay(plan, _dev(body[sl]), _dev(tp[sl]), _dev(cat[sl]), [(4.0, 0.5)] * 4,
                                    beta=0.95, snap_at=50)
            out = {k: np.asarray(v).tolist() for k, v in g.items()}
        else:
            cfg = configs.c5().with_n(n)
            L = generate_host(cfg.shape, cfg.seed, 0, n)
            arr = arrivals_host(cfg.seed, n, cfg.rate_rps)
            sl = slice(first, first + count)
            plan = fp.fleet_plan_create(**fp.desc_from_config(cfg), device=0, rank=rank, world=world,
                                        collectives=GlooCollectives(world))
            res, best = fp.sweep_peak_windows(plan, _dev(L[sl]), torch.from_numpy(arr[sl].view(np.int64)).cuda(),
                                              10**9, want_results=True)
            out = (res.tobytes(), best.tobytes())
        q.put((rank, out, None))
        fp.fleet_plan_destroy(plan)
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, None, traceback.format_exc()))


def _run(job, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, job, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=600) for _ in procs), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert o[2] is None, o[2]
    return [o[1] for o in out]


@pytest.mark.parametrize("n", [2_000_003, 1_001])
def test_calibration_two_ranks(n):
    import oracle
    from synth.gen import generate_raw_host
    body, mo, cat, tp = generate_raw_host("MIX", 31, 0, n)
    tp[::89] = 0
    o = oracle.calibrate(body, tp, cat, 4, beta=0.95, c0=4.0, s0=0.5, snap_at=50)
    for g in _run("calib", n):
        assert g["n_obs"] == [int(x) for x in o["n_obs"]]
        for key in ("c_hat", "sigma", "snap_c", "snap_sigma"):
            assert np.allclose(g[key], o[key], rtol=1e-12, atol=0, equal_nan=True), key


def test_peak_windows_two_ranks():
    import oracle
    import paper_2604_08075_b200 as fp
    from synth import configs
    from synth.gen import arrivals_host, generate_host
    n = 3_000_001
    cfg = configs.c5().with_n(n)
    L = generate_host(cfg.shape, cfg.seed, 0, n)
    arr = arrivals_host(cfg.seed, n, cfg.rate_rps)
    oall, obest = oracle.sweep_peak(cfg, L, arr, 10**9)
    for res, best in _run("peak", n):
        assert np.frombuffer(res, dtype=fp.FP_PEAK).tobytes() == oall.tobytes()
        assert best == obest.tobytes()
