"""GPU parity of the single-launch sorts (KF / KD, csrc/fused.cu; KS,
csrc/small.cu) through the C ABI: ring laps across many launches, both pass counts, ragged and
misaligned arrays, skewed owners, out-of-range keys and repeats, against the
oracle / np.sort (distinct keys have one ascending order, bitsort.hpp:84-136).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import bitwise_sort, fnv1a64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi(cuda):
    from paper_1312_0138_b200 import capi as c

    cuda.cuda.set_device(0)
    return c


@pytest.fixture(autouse=True, params=["FUSED", "FUSED_DIRECT", "SMALL"])
def _fused(capi, request):
    """KF (ring mode), KD (direct mode) and KS (small sorts, bitset words in
    registers); ranges a mode cannot hold take AUTO's pipeline."""
    capi.set_path(getattr(capi.Path, request.param))
    yield
    capi.set_path(capi.Path.AUTO)


def _device_sort(capi, torch, keys: np.ndarray, key_range: int, offset: int = 0, key_lo: int = 0):
    buf = torch.zeros(keys.size + offset + 4, dtype=torch.int32, device="cuda")
    src = buf[offset: offset + keys.size]
    src.copy_(torch.from_numpy(keys.view(np.int32)))
    out = torch.full((keys.size + 4,), -1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    if key_lo:
        capi.sort_range_device_async(src.data_ptr(), keys.size, out.data_ptr(), key_lo, key_range, s)
    else:
        capi.sort_device_async(src.data_ptr(), keys.size, out.data_ptr(), key_range, s)
    total = capi.sort_check(s)
    got = out.cpu().numpy().view(np.uint32)
    assert got[keys.size:].tolist() == [0xFFFFFFFF] * 4, "wrote past the output"
    return total, got[: keys.size]


def _distinct(rng, n, key_range):
    if n >= key_range:
        return rng.permutation(key_range).astype(np.uint32)
    return rng.choice(key_range, size=n, replace=False).astype(np.uint32)


@pytest.mark.parametrize("key_range", [1 << 12, 1 << 20, 1 << 24, (1 << 27) + 12345, 1 << 28])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 33, 1000, 4097, 65537, 300_001])
def test_random_vs_oracle(capi, cuda, n, key_range):
    if n > key_range:
        pytest.skip("n > key_range")
    rng = np.random.default_rng(n * 31 + key_range % 9973)
    keys = _distinct(rng, n, key_range)
    expected = bitwise_sort(keys) if n <= 100_000 else np.sort(keys)
    for off in (0, 1, 3):
        total, got = _device_sort(capi, cuda, keys, key_range, off)
        assert total == n
        assert np.array_equal(got, expected), (n, key_range, off)


def test_host_array_and_no_hint(capi):
    """bws_sort on a host array (no range hint: K0 then the fused plan)."""
    rng = np.random.default_rng(7)
    keys = _distinct(rng, 1 << 20, 1 << 26)
    a = keys.copy()
    capi.sort(a)
    assert np.array_equal(a, np.sort(keys))


def test_ring_laps_many_launches(capi, cuda):
    """Hundreds of launches of different sizes: ring positions run through
    many laps and wrap mid-run; every result must stay exact."""
    rng = np.random.default_rng(11)
    for i in range(300):
        n = int(rng.integers(1, 400_000))
        key_range = int(rng.choice([1 << 20, 1 << 24, 1 << 28]))
        n = min(n, key_range)
        keys = _distinct(rng, n, key_range) if key_range <= 1 << 24 else \
            np.unique(rng.integers(0, key_range, size=n + n // 8, dtype=np.int64).astype(np.uint32))[:n]
        rng.shuffle(keys)
        total, got = _device_sort(capi, cuda, keys, key_range, offset=int(rng.integers(0, 4)))
        assert total == keys.size, i
        assert np.array_equal(got, np.sort(keys)), i


@pytest.mark.parametrize("layout", ["sorted", "reverse", "one_slice", "two_slices", "blocks"])
def test_skewed_layouts(capi, cuda, layout):
    """Inputs whose keys all go to one or a few owners (one consumer drains
    most of the keys; producers wait on ring space)."""
    rng = np.random.default_rng(3)
    key_range = 1 << 28
    if layout == "sorted":
        keys = np.arange(1 << 22, dtype=np.uint32) * 3
    elif layout == "reverse":
        keys = (np.arange(1 << 22, dtype=np.uint32) * 3)[::-1].copy()
    elif layout == "one_slice":  # every key inside one owner's slice
        keys = rng.permutation(1 << 19).astype(np.uint32) + (5 << 20)
    elif layout == "two_slices":  # both passes' first slice
        keys = np.concatenate([rng.permutation(1 << 18).astype(np.uint32),
                               rng.permutation(1 << 18).astype(np.uint32) + (1 << 27) + 7])
        rng.shuffle(keys)
    else:  # sorted blocks of consecutive keys, blocks shuffled
        blocks = rng.permutation(1 << 12)
        keys = (blocks[:, None] * (1 << 14) + np.arange(1 << 10)[None, :]).astype(np.uint32).ravel()
    total, got = _device_sort(capi, cuda, keys, key_range)
    assert total == keys.size
    assert np.array_equal(got, np.sort(keys))


def test_dense_identity(capi, cuda):
    """n == M (every bit set): the output is the identity."""
    keys = np.random.default_rng(5).permutation(1 << 24).astype(np.uint32)
    total, got = _device_sort(capi, cuda, keys, 1 << 24)
    assert total == keys.size
    assert np.array_equal(got, np.arange(1 << 24, dtype=np.uint32))


def test_out_of_range_and_repeats(capi, cuda):
    """Keys >= the hint are counted, not sorted (BWS_ERROR_DATA); repeats
    give fewer set bits than keys (BWS_ERROR_DATA for the distinct-key
    extension, a full sort for bws_sort)."""
    keys = np.array([5, 1 << 20, 3, 7], dtype=np.uint32)
    with pytest.raises(capi.BitsortError) as e:
        _device_sort(capi, cuda, keys, 1 << 20)
    assert e.value.status == capi.Status.ERROR_DATA
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 1 << 16, size=200_000).astype(np.uint32)
    with pytest.raises(capi.BitsortError) as e:
        _device_sort(capi, cuda, keys, 1 << 16)
    assert e.value.status == capi.Status.ERROR_DATA
    a = keys.copy()
    capi.sort(a)
    assert np.array_equal(a, np.sort(keys))
    # the ring state is intact afterwards
    k2 = _distinct(rng, 100_000, 1 << 24)
    total, got = _device_sort(capi, cuda, k2, 1 << 24)
    assert total == k2.size and np.array_equal(got, np.sort(k2))


def test_range_sort_key_lo(capi, cuda):
    """bws_gpu_sort_range_device_async: keys in [lo, lo + range)."""
    rng = np.random.default_rng(13)
    lo, key_range = 3_000_000_000, 1 << 26
    keys = (_distinct(rng, 1 << 20, key_range).astype(np.uint64) + lo).astype(np.uint32)
    total, got = _device_sort(capi, cuda, keys, key_range, key_lo=lo)
    assert total == keys.size
    assert np.array_equal(got, np.sort(keys))


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_configs_vs_reference_anchors(capi, cuda, anchors, name):
    """C1 (one pass) and C2 (two passes) at full size, pinned to the FNV-1a
    anchors of the reference's own sorted output (tests/golden/anchors.json)."""
    from paper_1312_0138_b200 import configs

    cfg = configs.CONFIGS[name]
    keys = cfg.generate()
    assert fnv1a64(keys) == anchors[name]["fnv1a64_input"]
    for rep in range(3):
        total, got = _device_sort(capi, cuda, keys, cfg.key_range)
        assert total == cfg.n
        assert fnv1a64(got) == anchors[name]["fnv1a64_sorted"], rep


@pytest.mark.parametrize("count", [10_240, 10_241, 50_000, 131_072])
def test_one_slice_small_range(capi, cuda, count):
    """Every key inside one 2^17-key slice of a 2^24 range (KS: one CTA holds
    all the keys; at most 10240 leave through the SMEM stage, more by direct
    stores), the slice full at 131072 keys; then a spread-out sort to show the
    cached bitset was left all-zero."""
    rng = np.random.default_rng(count)
    keys = (rng.permutation(1 << 17)[:count].astype(np.uint32) + (5 << 17)).astype(np.uint32)
    for off in (0, 1):
        total, got = _device_sort(capi, cuda, keys, 1 << 24, off)
        assert total == count
        assert np.array_equal(got, np.sort(keys))
    k2 = _distinct(rng, 200_000, 1 << 24)
    total, got = _device_sort(capi, cuda, k2, 1 << 24)
    assert total == k2.size and np.array_equal(got, np.sort(k2))


def test_small_sort_graph_replay(capi, cuda):
    """A hinted small sort captured in a CUDA graph and replayed with new keys
    in the same buffers, interleaved with direct calls: the KS grid barrier
    takes its generation from the device-side arrival counter, so nothing
    launch-specific is baked into the captured kernel node."""
    n, key_range = 300_000, 1 << 24
    rng = np.random.default_rng(41)
    t = cuda.empty(n, dtype=cuda.int32, device="cuda")
    out = cuda.empty_like(t)
    s = cuda.cuda.Stream()
    k0 = _distinct(rng, n, key_range)
    t.copy_(cuda.from_numpy(k0.view(np.int32)))
    with cuda.cuda.stream(s):
        capi.sort_device_async(t.data_ptr(), n, out.data_ptr(), key_range, s.cuda_stream)  # warm-up
    s.synchronize()
    g = cuda.cuda.CUDAGraph()
    with cuda.cuda.graph(g, stream=s):
        capi.sort_device_async(t.data_ptr(), n, out.data_ptr(), key_range, s.cuda_stream)
    for rep in range(7):
        keys = _distinct(rng, n, key_range)
        t.copy_(cuda.from_numpy(keys.view(np.int32)))
        out.zero_()
        cuda.cuda.synchronize()
        g.replay()
        s.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys)), rep
        if rep % 3 == 1:  # a direct call between replays
            total, got = _device_sort(capi, cuda, k0, key_range)
            assert total == n and np.array_equal(got, np.sort(k0))
