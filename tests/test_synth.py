"""Input module checks: the three Philox/trace generators agree word for word,
traces are shard-independent, and the synthetic shapes hit the paper's stated
trace statistics."""
import numpy as np
import pytest

from synth import configs
from synth.gen import generate_host, generate_np
from synth.philox import philox4x32_10


def test_philox_known_answers():
    # Random123 known-answer vectors for Philox4x32-10
    assert [int(x) for x in philox4x32_10(0, 0, 0, 0, 0, 0)] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    f = 0xFFFFFFFF
    assert [int(x) for x in philox4x32_10(f, f, f, f, f, f)] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert [int(x) for x in philox4x32_10(0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344,
                                          0xA4093822, 0x299F31D0)] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


@pytest.mark.parametrize("shape", ["AZ", "LM", "SG", "MIX"])
def test_host_c_matches_numpy(shape):
    for first in (0, 12345, (1 << 32) - 100):
        a = generate_np(shape, 99, first, 5000)
        b = generate_host(shape, 99, first, 5000)
        assert np.array_equal(a, b)


def test_shard_independence():
    full = generate_host("MIX", 7, 0, 100_000)
    parts = [generate_host("MIX", 7, s, 25_000) for s in range(0, 100_000, 25_000)]
    assert np.array_equal(full, np.concatenate(parts))


def test_shape_targets():
    az = generate_host("AZ", configs.SEED0, 0, 2_000_000)
    assert abs((az <= 1024).mean() - 0.35) < 0.01
    assert abs((az <= 8192).mean() - 0.80) < 0.01
    assert (az > 65536).mean() < 0.005                    # tail to 64K, rare rejections
    lm = generate_host("LM", configs.SEED0, 0, 2_000_000)
    assert abs((lm <= 8192).mean() - 0.68) < 0.01
    sg = generate_host("SG", configs.SEED0, 0, 2_000_000)
    assert (sg <= 2048).mean() > 0.75                     # "heavily concentrated below 2K"
    assert sg.max() > 131072                              # rejections exercised at C_L <= 128K


def test_az_prompt_quantiles():
    # 80% of prompts fit in 2K and 95% in 8K (L_in alone)
    from synth.gen import _sample
    from synth.philox import philox_words
    from synth.shapes import shape_az
    w0, _, _, _ = philox_words(3, 0, 1_000_000)
    lin = _sample(shape_az().t_in, w0)
    assert abs((lin <= 2048).mean() - 0.80) < 0.005
    assert abs((lin <= 8192).mean() - 0.95) < 0.005
    assert lin.max() <= 65536


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["AZ", "LM", "SG", "MIX"])
def test_cuda_generator_matches_host(shape):
    import torch
    from synth.gen import generate_device
    n = 1_000_003
    d = generate_device(shape, 11, 5, n).cpu().numpy().view(np.uint32)
    h = generate_host(shape, 11, 5, n)
    assert np.array_equal(d, h)


@pytest.mark.parametrize("shape", ["AZ", "MIX"])
def test_raw_columns_host_matches_numpy_and_trace(shape):
    from synth.gen import generate_raw_host, generate_raw_np
    a = generate_raw_np(shape, 5, 1000, 20000)
    b = generate_raw_host(shape, 5, 1000, 20000)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    # the true total of the raw columns is the L_total trace
    L = generate_host(shape, 5, 1000, 20000)
    assert np.array_equal(a[3].astype(np.uint64) + a[1], L)


def test_raw_columns_category_ratios():
    # Table 5 "True c_k": per-category mean bytes/token within 1%
    from synth.gen import generate_raw_host
    from synth.shapes import CAT_TRUE_RATIO, CAT_WEIGHTS
    body, _, cat, lin = generate_raw_host("AZ", 9, 0, 1_000_000)
    for k, c in enumerate(CAT_TRUE_RATIO):
        m = (cat == k) & (lin >= 64)
        assert abs(body[m].sum() / lin[m].sum() - c) / c < 0.01
        assert abs(np.mean(cat == k) - CAT_WEIGHTS[k]) < 0.005


@pytest.mark.gpu
def test_raw_columns_cuda_matches_host():
    from synth.gen import generate_raw_device, generate_raw_host
    d = generate_raw_device("MIX", 3, 7, 500_001)
    h = generate_raw_host("MIX", 3, 7, 500_001)
    for x, y in zip(d, h):
        xv = x.cpu().numpy()
        assert np.array_equal(xv.view(y.dtype) if xv.dtype != y.dtype else xv, y)
