"""GPU parity for inputs with repeated keys (bws_sort's full uint32/int32
contract).

The reference's bws_sort sorts any input (bitsort.hpp:84-136 is a radix sort).
The B200 build's bitset pass detects repeats (fewer set bits than keys) and
redoes the sort from the untouched input with the counting-sort pass (KB1-KB3
packed layout + KB4m, bucket.cu). Checked bit-exact against the oracle (C
restatement of the reference's bitwise sort) and, where it was built, the
reference's own bws_sort.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import bitwise_sort

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi(cuda):
    from paper_1312_0138_b200 import capi as c

    cuda.cuda.set_device(0)
    return c


@pytest.fixture(autouse=True)
def _auto_mode(capi):
    yield
    capi.set_path(capi.Path.AUTO)


def _reference(keys: np.ndarray, is_unsigned: int = 1) -> np.ndarray:
    a = keys.copy()
    if oracle.REFERENCE is not None:  # the reference's own bws_sort
        assert oracle.REFERENCE.bws_sort(a.ctypes.data, a.size, 32, is_unsigned, 0) == 0
        return a
    return bitwise_sort(a)  # the oracle's restatement (signed split included)


def _sort_host(capi, keys, is_unsigned=1):
    a = keys.copy()
    assert capi.sort_raw(a.ctypes.data, a.size, 32, is_unsigned, capi.Algorithm.BITWISE) == capi.Status.OK, \
        capi.last_error()
    return a


def _sort_device(capi, torch, keys, is_unsigned=1, offset=0):
    buf = torch.zeros(keys.size + offset + 4, dtype=torch.int32, device="cuda")
    view = buf[offset: offset + keys.size]
    view.copy_(torch.from_numpy(keys.view(np.int32)))
    assert capi.sort_raw(view.data_ptr(), keys.size, 32, is_unsigned, 0) == capi.Status.OK, capi.last_error()
    torch.cuda.synchronize()
    assert int(buf[offset + keys.size:].abs().sum()) == 0  # nothing written past the array
    return view.cpu().numpy().view(keys.dtype)


@pytest.mark.parametrize("path", ["AUTO", "DIRECT", "BUCKETED"])
@pytest.mark.parametrize("n", [2, 3, 100, 1000, 65537, (1 << 21) - 1, (1 << 21) + 5])
@pytest.mark.parametrize("key_range", [1, 2, 17, 1000, 1 << 20, 1 << 32])
def test_repeats_vs_oracle(capi, cuda, path, n, key_range):
    capi.set_path(getattr(capi.Path, path))
    rng = np.random.default_rng(n * 31 + key_range % 1000)
    keys = rng.integers(0, key_range, size=n, dtype=np.uint64).astype(np.uint32)
    expected = bitwise_sort(keys)
    assert np.array_equal(_sort_host(capi, keys), expected)
    assert np.array_equal(_sort_device(capi, cuda, keys, offset=n % 3), expected)


@pytest.mark.parametrize("n", [1000, 1 << 20])
def test_reference_generator_inputs(capi, n):
    """The reference's own uint32 input generator (generator.hpp:91-103, seeded
    like acceptance.cpp) draws with repeats: bit-exact vs its bws_sort."""
    for trial in range(3):
        keys = oracle.generate_uniform_u32(n, seed=1337, trial=trial)
        assert np.array_equal(_sort_host(capi, keys), _reference(keys))


@pytest.mark.parametrize("value", [0, 123456789, 0xFFFFFFFF])
@pytest.mark.parametrize("n", [5, 1 << 22])
def test_all_equal(capi, cuda, value, n):
    """One key repeated n times: the counting pass expands a single counter."""
    keys = np.full(n, value, dtype=np.uint32)
    assert np.array_equal(_sort_host(capi, keys), keys)
    assert np.array_equal(_sort_device(capi, cuda, keys), keys)


def test_few_values_many_times(capi, cuda):
    rng = np.random.default_rng(7)
    vals = rng.integers(0, 1 << 32, size=37, dtype=np.uint64).astype(np.uint32)
    keys = vals[rng.integers(0, vals.size, size=(1 << 22) + 3)]
    expected = np.sort(keys)
    assert np.array_equal(_sort_host(capi, keys), expected)
    assert np.array_equal(_sort_device(capi, cuda, keys, offset=1), expected)


@pytest.mark.parametrize("n", [3, 1000, 1 << 21])
def test_signed_repeats(capi, cuda, n):
    rng = np.random.default_rng(n)
    keys = rng.integers(-(1 << 31), 1 << 31, size=n, dtype=np.int64).astype(np.int32)
    keys[: n // 2] = keys[n // 2: 2 * (n // 2)]  # every key of the first half repeats
    if n >= 4:
        keys[:4] = [-(1 << 31), -(1 << 31), (1 << 31) - 1, (1 << 31) - 1]
    rng.shuffle(keys)
    expected = _reference(keys, is_unsigned=0)
    assert np.array_equal(expected, np.sort(keys))
    assert np.array_equal(_sort_host(capi, keys, 0), expected)
    assert np.array_equal(_sort_device(capi, cuda, keys, 0), expected)


def test_pinned_host_repeats(capi, cuda):
    keys = np.random.default_rng(11).integers(0, 1 << 16, size=1 << 21, dtype=np.uint32)
    t = cuda.from_numpy(keys.view(np.int32).copy()).pin_memory()
    assert capi.sort_raw(t.data_ptr(), keys.size, 32, 1, 0) == capi.Status.OK, capi.last_error()
    assert np.array_equal(t.numpy().view(np.uint32), np.sort(keys))


def test_repeats_then_distinct(capi, cuda):
    """A repeat-sorting call leaves nothing behind for the next distinct sort
    (cached bitset, slab counters, control block)."""
    rng = np.random.default_rng(2)
    for _ in range(2):
        rep = rng.integers(0, 1 << 24, size=1 << 22, dtype=np.uint32)
        assert np.array_equal(_sort_host(capi, rep), np.sort(rep))
        dis = rng.choice(1 << 24, size=1 << 22, replace=False).astype(np.uint32)
        assert np.array_equal(_sort_host(capi, dis), np.sort(dis))
        small = rng.choice(1 << 20, size=5000, replace=False).astype(np.uint32)
        assert np.array_equal(_sort_host(capi, small), np.sort(small))


@pytest.mark.slow
def test_c2_shape_with_repeats(capi, cuda):
    """C2's size (2^26 keys) drawn WITH replacement from [0, 2^24): every value
    about four times. Device array, in place."""
    keys = np.random.default_rng(42).integers(0, 1 << 24, size=1 << 26, dtype=np.uint32)
    t = cuda.from_numpy(keys.view(np.int32).copy()).cuda()
    assert capi.sort_raw(t.data_ptr(), keys.size, 32, 1, 0) == capi.Status.OK, capi.last_error()
    got = t.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, np.sort(keys))


@pytest.mark.parametrize("case", ["distinct", "repeats_no_overflow", "overflow", "signed_repeats",
                                  "distinct_then_repeats"])
@pytest.mark.parametrize("offset", [0, 1])
def test_device_array_in_place(capi, cuda, case, offset):
    """bws_sort on device arrays of >= 2^21 keys sorts in place through the
    slab pipeline: distinct keys need no copy; repeats without a dropped slab
    run are redone from the slabs (KB4m over the slab layout, padding dropped);
    a bucket that overflowed makes KB4 write nothing, so the counting pass
    starts from the intact keys. Every case against the reference's sort."""
    rng = np.random.default_rng(31 + offset)
    n = (1 << 22) + 3
    is_unsigned = 1
    if case == "distinct":
        keys = rng.choice(1 << 23, size=n, replace=False).astype(np.uint32)
    elif case == "repeats_no_overflow":  # ~2^21 repeated values over 8 slab buckets
        keys = rng.integers(0, 1 << 23, size=n, dtype=np.uint64).astype(np.uint32)
    elif case == "overflow":  # one 2^20-key bucket receives 4x its capacity
        keys = rng.integers(0, 1 << 20, size=n, dtype=np.uint64).astype(np.uint32)
    elif case == "signed_repeats":
        keys = rng.integers(-(1 << 22), 1 << 22, size=n, dtype=np.int64).astype(np.int32)
        is_unsigned = 0
    else:  # a distinct sort, then repeats over the same buffers
        d = rng.choice(1 << 23, size=n, replace=False).astype(np.uint32)
        assert np.array_equal(_sort_device(capi, cuda, d, 1, offset), np.sort(d))
        keys = rng.integers(0, 1 << 23, size=n, dtype=np.uint64).astype(np.uint32)
    got = _sort_device(capi, cuda, keys, is_unsigned, offset)
    assert np.array_equal(got, np.sort(keys)), case
    if case != "distinct" and oracle.REFERENCE is not None:
        assert np.array_equal(got, _reference(keys, is_unsigned))


def test_device_array_speculated_range(capi, cuda):
    """An in-place device-array bws_sort without a hint plans for the range the
    previous such sort's keys had instead of running K0 (KB3 folds the largest
    key). Sequences that grow, shrink and repeat the range, with repeats and
    signed keys in between: every result against numpy; a sort whose keys
    outgrow the speculated range is redone from the intact keys."""
    rng = np.random.default_rng(77)
    n = (1 << 22) + 1
    def distinct(m):
        return rng.choice(m, size=n, replace=False).astype(np.uint32)
    seq = [
        ("first", distinct(1 << 23), 1),
        ("same range", distinct(1 << 23), 1),
        ("grown 2x", distinct(1 << 24), 1),           # beyond the speculated range: redone in place
        ("grown 16x", distinct(1 << 27), 1),          # beyond it again, and too wide for the slab
        ("shrunk", distinct(1 << 23), 1),             # inside it: sorted on the wide plan
        ("shrunk again", distinct(1 << 23), 1),       # now planned for 2^23
        ("one key above", np.concatenate([distinct(1 << 23)[:-1], [np.uint32((1 << 30) + 5)]]).astype(np.uint32), 1),
        ("repeats", rng.integers(0, 1 << 23, size=n, dtype=np.uint64).astype(np.uint32), 1),
        ("signed", rng.integers(-(1 << 22), 1 << 22, size=n, dtype=np.int64).astype(np.int32), 0),
        ("unsigned after signed", distinct(1 << 24), 1),
        ("top of the range", (np.uint32(0xffffffff) - distinct(1 << 23)).astype(np.uint32), 1),
        ("small after top", distinct(1 << 23), 1),
    ]
    for name, keys, is_unsigned in seq:
        for offset in (0, 1):
            got = _sort_device(capi, cuda, keys, is_unsigned, offset)
            assert np.array_equal(got, np.sort(keys)), name


def test_small_unhinted_speculation(capi, cuda):
    """bws_sort on arrays below 2^21 keys: the first sort runs K2 + K3 and
    reports the keys' range; the next ones run the single-launch KS planned
    for it. Host and device arrays through sequences that keep, outgrow
    (redo with K2 + K3) and shrink the range, with repeats and a range above
    KS's limit in between."""
    rng = np.random.default_rng(91)
    def distinct(n, m):
        return rng.choice(m, size=n, replace=False).astype(np.uint32)
    seq = [
        distinct(100_000, 1 << 20),
        distinct(100_000, 1 << 20),                       # same range: KS
        distinct(300_001, 1 << 24),                       # outgrown: redone
        distinct(300_001, 1 << 24),                       # KS
        distinct(5, 1 << 10),                             # shrunk
        distinct(5, 1 << 10),
        rng.integers(0, 1 << 12, size=50_000, dtype=np.uint64).astype(np.uint32),   # repeats on the KS pass
        distinct(70_000, 1 << 18),
        (distinct(1000, 1 << 16).astype(np.uint64) + (1 << 31)).astype(np.uint32),  # beyond KS's AUTO range
        distinct(70_000, 1 << 18),
        np.array([7], dtype=np.uint32),
        np.array([0xffffffff, 0, 5], dtype=np.uint32),
        distinct((1 << 21) - 1, 1 << 22),
    ]
    for i, keys in enumerate(seq):
        expected = np.sort(keys)
        assert np.array_equal(_sort_host(capi, keys), expected), ("host", i)
        assert np.array_equal(_sort_device(capi, cuda, keys, offset=i % 3), expected), ("device", i)
    t = cuda.from_numpy(seq[3].view(np.int32).copy()).pin_memory()  # pinned host array
    assert capi.sort_raw(t.data_ptr(), seq[3].size, 32, 1, 0) == capi.Status.OK, capi.last_error()
    assert np.array_equal(t.numpy().view(np.uint32), np.sort(seq[3]))


def test_device_array_alternating_ranges(capi, cuda):
    """A caller alternating between a narrow and a wide key range on one
    device: every second sort outgrows the speculated range; after two misses
    in a row the library stops speculating for a while. All results exact."""
    rng = np.random.default_rng(5)
    n = (1 << 22) + 7
    narrow = rng.choice(1 << 23, size=n, replace=False).astype(np.uint32)
    wide = rng.choice(1 << 24, size=n, replace=False).astype(np.uint32)
    for i in range(24):
        keys = wide if i % 2 else narrow
        assert np.array_equal(_sort_device(capi, cuda, keys, 1, i % 2), np.sort(keys)), i
