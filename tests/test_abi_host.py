"""C-ABI checks that need no GPU: the library loads, exports every function
include/fleet_plan.h declares, and its host-only partition helpers behave."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2604_08075_b200 as fp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fleet_plan.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"\{[^{}]*\}", "", src)          # drop struct bodies (function-pointer fields)
    return sorted(set(re.findall(r"\b([a-z_][a-z0-9_]*)\s*\([^;{]*\)\s*;", src)))


def test_every_declared_symbol_is_exported():
    names = _declared()
    assert "sweep_thresholds" in names and "fleet_plan_create" in names and len(names) >= 14
    lib = ctypes.CDLL(fp.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(fp.EXPORTED) == names


def test_candidate_record_layout_matches_header():
    # 8 x u32 + 12 x u64 + 8 x f64 (fleet_plan.h fp_candidate)
    assert fp.FP_CANDIDATE.itemsize == 192
    assert fp.FP_CANDIDATE.fields["nseq_short"][1] == 32
    assert fp.FP_CANDIDATE.fields["alpha"][1] == 128


@pytest.mark.parametrize("n", [0, 1, 31, 32, 1000, 10**9 + 7])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(n, world):
    got = [fp.fp_shard_range(n, r, world) for r in range(world)]
    pos = 0
    for first, count in got:
        assert first == pos or count == 0
        if count:
            assert first % 32 == 0                      # 128-byte aligned shard starts
        pos = first + count if count else pos
    assert sum(c for _, c in got) == n


@pytest.mark.parametrize("n,world", [(1, 1), (7, 2), (4096, 8), (30720, 3), (5, 8)])
def test_candidate_range_partitions(n, world):
    got = [fp.fp_candidate_range(n, r, world) for r in range(world)]
    assert sum(c for _, c in got) == n
    flat = np.concatenate([np.arange(f, f + c) for f, c in got])
    assert np.array_equal(flat, np.arange(n))


def test_merge_best_is_deterministic_lowest_index():
    recs = np.zeros(6, dtype=fp.FP_CANDIDATE)        # world 3 x 2 models
    recs["model"] = [0, 1, 0, 1, 0, 1]
    recs["index"] = [5, 100, 9, 120, 2, 130]
    recs["flags"] = [7, 7, 7, 1, 7, 7]
    recs["cost_dual"] = [10.0, 3.0, 10.0, 1.0, 11.0, 3.0]
    out = fp.fp_merge_best(recs, 3, 2)
    assert out["index"].tolist() == [5, 100]          # tie on cost -> lowest index; infeasible skipped
    recs["flags"] = 0
    out = fp.fp_merge_best(recs, 3, 2)
    assert out["index"].tolist() == [0xFFFFFFFF] * 2 and np.all(np.isinf(out["cost_dual"]))


def test_create_without_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from synth import configs
    with pytest.raises(fp.FleetPlanError) as e:
        fp.fleet_plan_create(**fp.desc_from_config(configs.c1()))
    assert e.value.status == 6           # FP_ERR_CUDA: no CPU fallback
