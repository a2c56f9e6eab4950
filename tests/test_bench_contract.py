"""bench.py's JSON contract on CPU: the reference arm (the oracle, this tier's
reference) prints one line with the keys the driver reads, and the argument
checks reject runs the timing rules forbid. The GPU arm's line is checked on
the B200 by the round-end bench itself."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout)


def test_reference_arm_line():
    r = _bench("--impl", "reference", "--steps", "2", "--warmup", "3", "--ref-sample", "100000")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1                     # exactly one JSON line on stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["unit"] == "requests/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"].startswith("C5")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and "100,000" in cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_warmup_below_three_is_rejected():
    r = _bench("--impl", "reference", "--steps", "1", "--warmup", "1", "--ref-sample", "1000", timeout=120)
    assert r.returncode != 0
    assert "warmup" in r.stderr


def test_self_spawn_two_ranks_gloo():
    """`bench.py --gpus 2` without torchrun re-launches itself as two ranks
    (torch.distributed.run, 127.0.0.1); the plumbing check runs the same launch,
    process group, max-over-ranks and rank-0-only output path on gloo."""
    r = _bench("--gpus", "2", "--plumbing-check", timeout=240)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["plumbing"] == "ok" and d["n_gpus"] == 2 and d["max_over_ranks"] == 2.0
    assert sorted(x["rank"] for x in d["ranks"]) == [0, 1]
