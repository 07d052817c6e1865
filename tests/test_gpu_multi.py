"""Single-process multi-GPU bws_sort (csrc/multi.cpp):
the drop-in call on a host array with G logical ranks. Only one GPU is
available to this build, so the G ranks share device 0 (bws_gpu_set_devices
with a repeated device): every rank has its own shard, bitset, stream and
slice, and the exchange is the P2P fused scan reading all G bitsets (NCCL
needs distinct devices). Results are pinned to the reference's sorted
hashes (tests/golden/anchors.json) for C1, C2 and C5 at G = 2, 4, 8."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import bitwise_sort

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi(cuda):
    from paper_1312_0138_b200 import capi as c

    cuda.cuda.set_device(0)
    return c


@pytest.fixture
def ranks(capi):
    old = os.environ.get("BITSORT_MULTI_MIN_KEYS")
    os.environ["BITSORT_MULTI_MIN_KEYS"] = "0"  # small inputs take the multi-GPU path too
    yield capi
    capi.set_device_count(1)
    if old is None:
        os.environ.pop("BITSORT_MULTI_MIN_KEYS", None)
    else:
        os.environ["BITSORT_MULTI_MIN_KEYS"] = old


def _pinned(keys):
    import torch

    t = torch.empty(keys.size, dtype=torch.int32, pin_memory=True)
    a = t.numpy().view(np.uint32)
    a[:] = keys
    return t, a


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("n,key_range", [(1, 1 << 10), (7, 1 << 10), (5000, 1 << 20), (300_001, (1 << 22) - 5),
                                         (1 << 21, 1 << 23), (3 << 20, 1 << 32)])
def test_multi_rank_sort_vs_oracle(ranks, G, n, key_range):
    capi = ranks
    capi.set_devices([0] * G)
    assert capi.device_count() == G
    rng = np.random.default_rng(G * 1000 + n)
    keys = rng.choice(key_range, size=n, replace=False).astype(np.uint32) if key_range < (1 << 32) else \
        np.unique(rng.integers(0, 1 << 32, size=n + n // 8, dtype=np.uint64)).astype(np.uint32)[:n]
    rng.shuffle(keys)
    expected = np.sort(keys)
    a = keys.copy()
    capi.sort(a)  # pageable host array, no hint
    assert np.array_equal(a, expected)
    t, p = _pinned(keys)
    capi.sort(p)  # pinned host array
    assert np.array_equal(p, expected)
    b = keys.copy()
    capi.sort_u32_range(b, key_range)  # with the hint
    assert np.array_equal(b, expected)
    if n <= 5000:
        assert np.array_equal(expected, bitwise_sort(keys))


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_multi_rank_configs_vs_reference_hash(ranks, anchors, G, name):
    from paper_1312_0138_b200.configs import CONFIGS
    from paper_1312_0138_b200.datagen import fnv1a64

    capi = ranks
    capi.set_devices([0] * G)
    keys = CONFIGS[name].generate()
    assert fnv1a64(keys) == anchors[name]["fnv1a64_input"]
    t, p = _pinned(keys)
    del keys
    capi.sort(p)
    assert fnv1a64(p) == anchors[name]["fnv1a64_sorted"]


@pytest.mark.parametrize("G", [2, 5])
def test_multi_rank_repeats_and_errors(ranks, G):
    capi = ranks
    capi.set_devices([0] * G)
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 1 << 12, size=200_000).astype(np.uint32)  # many repeats
    a = keys.copy()
    capi.sort(a)  # bws_sort: repeats are sorted too (single-GPU counting pass)
    assert np.array_equal(a, np.sort(keys))
    u = rng.choice(1 << 24, size=100_000, replace=False).astype(np.uint32)
    u[10] = u[99_000]  # one cross-shard duplicate
    b = u.copy()
    with pytest.raises(capi.BitsortError) as e:
        capi.sort_u32_range(b, 1 << 24)  # the distinct-key extension
    assert e.value.status == capi.Status.ERROR_DATA
    assert np.array_equal(b, u)  # untouched
    c = rng.choice(1 << 20, size=100_000, replace=False).astype(np.uint32)
    c[5] = 1 << 20  # out of the hinted range
    d = c.copy()
    with pytest.raises(capi.BitsortError) as e:
        capi.sort_u32_range(d, 1 << 20)
    assert e.value.status == capi.Status.ERROR_DATA and "key range" in capi.last_error()
    assert np.array_equal(d, c)


def test_multi_rank_other_widths_stay_single(ranks):
    capi = ranks
    capi.set_devices([0, 0])
    s = np.random.default_rng(3).integers(-(1 << 20), 1 << 20, size=100_000).astype(np.int32)
    a = s.copy()
    assert capi.sort_raw(a.ctypes.data, a.size, 32, 0) == capi.Status.OK  # signed: single GPU
    assert np.array_equal(a, np.sort(s))
    w = np.random.default_rng(4).integers(0, 1 << 60, size=50_000, dtype=np.uint64)
    b = w.copy()
    assert capi.sort_raw(b.ctypes.data, b.size, 64, 1) == capi.Status.OK
    assert np.array_equal(b, np.sort(w))


def test_multi_rank_bad_device(capi):
    import torch

    with pytest.raises(capi.BitsortError) as e:
        capi.set_devices([0, torch.cuda.device_count()])
    assert e.value.status == capi.Status.ERROR_CONFIG
    assert capi.device_count() == 1
