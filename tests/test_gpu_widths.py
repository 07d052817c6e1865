"""GPU parity for the other key widths of bws_sort (dispatch.hpp:17-40's
with_width arms): 8/16-bit keys by the GPU counting sort over the type's range
(widths.cu KW1-KW3), 64-bit keys whose span is below 2^32 narrowed to the
32-bit pipeline and widened back. Checked bit-exact against the oracle (C
restatement of the reference's bitwise sort per width) and, for signed keys,
the reference's own bws_sort where it was built.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import bitwise_sort

pytestmark = pytest.mark.gpu

WIDTH = {np.dtype(np.uint8): 8, np.dtype(np.int8): 8, np.dtype(np.uint16): 16, np.dtype(np.int16): 16,
         np.dtype(np.uint64): 64, np.dtype(np.int64): 64, np.dtype(np.uint32): 32, np.dtype(np.int32): 32}


@pytest.fixture(scope="module")
def capi(cuda):
    from paper_1312_0138_b200 import capi as c

    cuda.cuda.set_device(0)
    return c


def _expected(keys: np.ndarray) -> np.ndarray:
    unsigned = keys.dtype.kind == "u"
    a = keys.copy()
    if oracle.REFERENCE is not None:  # the reference's own bws_sort at this width
        assert oracle.REFERENCE.bws_sort(a.ctypes.data, a.size, WIDTH[a.dtype], int(unsigned), 0) == 0
        return a
    return bitwise_sort(a)  # the oracle's restatement (signed split included)


def _host(capi, keys):
    a = keys.copy()
    st = capi.sort_raw(a.ctypes.data, a.size, WIDTH[a.dtype], int(a.dtype.kind == "u"), capi.Algorithm.BITWISE)
    assert st == capi.Status.OK, capi.last_error()
    return a


def _device(capi, torch, keys, offset=0):
    offset *= keys.itemsize  # keys stay naturally aligned (bitsort.h:86-88)
    nb = keys.nbytes
    buf = torch.zeros(nb + 64, dtype=torch.uint8, device="cuda")
    view = buf[offset: offset + nb]
    view.copy_(torch.from_numpy(keys.view(np.uint8).copy()))
    st = capi.sort_raw(view.data_ptr(), keys.size, WIDTH[keys.dtype], int(keys.dtype.kind == "u"), 0)
    assert st == capi.Status.OK, capi.last_error()
    torch.cuda.synchronize()
    assert int(buf[:offset].sum()) == 0 and int(buf[offset + nb:].sum()) == 0  # nothing outside the array
    return view.cpu().numpy().view(keys.dtype).copy()


@pytest.mark.parametrize("width", [8, 16, 32, 64])
def test_width_golden_vectors(capi, cuda, width_records, width):
    """The reference's own bws_sort outputs for its generator's distributions
    at this width, signed and unsigned (tests/golden/widths.bin): bit-exact,
    host and device arrays."""
    recs = [r for r in width_records if r["width"] == width]
    assert recs
    for rec in recs:
        assert np.array_equal(_host(capi, rec["input"]), rec["output"]), (rec["unsigned"], rec["dist"], rec["n"])
        assert np.array_equal(_device(capi, cuda, rec["input"], offset=1), rec["output"])


def test_capi_uint8_vector(capi):
    """test_capi.cpp:78-82 exactly as the reference tests it: width 8, unsigned."""
    a = np.array([200, 3, 255, 0], dtype=np.uint8)
    assert capi.sort_raw(a.ctypes.data, 4, 8, 1, capi.Algorithm.BITWISE) == capi.Status.OK, capi.last_error()
    assert a.tolist() == [0, 3, 200, 255]


@pytest.mark.parametrize("dtype", [np.uint8, np.int8, np.uint16, np.int16])
@pytest.mark.parametrize("n", [1, 2, 3, 17, 1000, 65537, (1 << 20) + 3])
def test_small_widths_random(capi, cuda, dtype, n):
    info = np.iinfo(dtype)
    keys = np.random.default_rng(n + info.bits).integers(info.min, info.max + 1, size=n, dtype=np.int64).astype(dtype)
    expected = _expected(keys)
    assert np.array_equal(expected, np.sort(keys))
    assert np.array_equal(_host(capi, keys), expected)
    assert np.array_equal(_device(capi, cuda, keys, offset=n % 7), expected)


@pytest.mark.parametrize("dtype", [np.uint8, np.int16])
@pytest.mark.parametrize("kind", ["constant", "sorted", "reverse", "extremes", "sparse_values"])
def test_small_widths_layouts(capi, cuda, dtype, kind):
    info = np.iinfo(dtype)
    n = (1 << 22) + 1
    rng = np.random.default_rng(3)
    if kind == "constant":
        keys = np.full(n, info.max, dtype=dtype)
    elif kind == "extremes":
        keys = rng.choice(np.array([info.min, info.max], dtype=dtype), size=n)
    elif kind == "sparse_values":  # few distinct values spread over the range: long zero runs in the prefix
        keys = rng.choice(np.linspace(info.min, info.max, 7).astype(dtype), size=n)
    else:
        keys = np.sort(rng.integers(info.min, info.max + 1, size=n, dtype=np.int64).astype(dtype))
        if kind == "reverse":
            keys = keys[::-1].copy()
    expected = np.sort(keys)
    assert np.array_equal(_host(capi, keys), expected)
    assert np.array_equal(_device(capi, cuda, keys, offset=3), expected)


@pytest.mark.parametrize("signed", [False, True])
@pytest.mark.parametrize("n", [1, 5, 1000, (1 << 21) + 9])
@pytest.mark.parametrize("span_log2", [1, 20, 32])
def test_64bit_narrow_span(capi, cuda, signed, n, span_log2):
    """64-bit keys spanning fewer than 2^32 values, placed far from zero (and
    across zero for signed keys), with repeats in the small spans."""
    rng = np.random.default_rng(n + span_log2)
    span = (1 << span_log2) - 1
    if signed:
        base = -(1 << 62) if span_log2 < 32 else -(1 << 31)
        keys = (base + rng.integers(0, span + 1, size=n, dtype=np.int64)).astype(np.int64)
    else:
        base = (1 << 63) + (1 << 40)
        keys = (np.uint64(base) + rng.integers(0, span + 1, size=n, dtype=np.int64).astype(np.uint64))
    expected = _expected(keys)
    assert np.array_equal(expected, np.sort(keys))
    assert np.array_equal(_host(capi, keys), expected)
    assert np.array_equal(_device(capi, cuda, keys, offset=8), expected)


@pytest.mark.parametrize("signed", [False, True])
@pytest.mark.parametrize("n", [2, 3, 255, 1000, 65537, (1 << 20) + 7])
@pytest.mark.parametrize("kind", ["full_range", "high_bits", "repeats"])
def test_64bit_wide_span_radix(capi, cuda, signed, n, kind):
    """Spans of 2^32 values or more: the stable LSD radix path (8-bit digits,
    constant digits skipped)."""
    rng = np.random.default_rng(n * 3 + len(kind))
    dt = np.int64 if signed else np.uint64
    info = np.iinfo(dt)
    if kind == "full_range":
        keys = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
    elif kind == "high_bits":  # only bits 40-47 and 0-3 vary: most digits are skipped
        keys = ((rng.integers(0, 256, size=n).astype(np.uint64) << np.uint64(40)) |
                rng.integers(0, 16, size=n).astype(np.uint64)).astype(dt)
    else:
        vals = rng.integers(info.min, info.max, size=max(2, n // 50), dtype=dt, endpoint=True)
        keys = vals[rng.integers(0, vals.size, size=n)]
    keys[0], keys[-1] = info.min, info.max
    expected = _expected(keys)
    assert np.array_equal(expected, np.sort(keys))
    assert np.array_equal(_host(capi, keys), expected)
    assert np.array_equal(_device(capi, cuda, keys, offset=1), expected)


def test_64bit_edges(capi):
    c = np.array([np.iinfo(np.int64).min, np.iinfo(np.int64).min + 5, np.iinfo(np.int64).min], dtype=np.int64)
    assert capi.sort_raw(c.ctypes.data, 3, 64, 0, 0) == capi.Status.OK, capi.last_error()
    assert c.tolist() == sorted(c.tolist())
    d = np.full(1000, 1 << 63, dtype=np.uint64)  # all equal: no radix pass at all
    assert capi.sort_raw(d.ctypes.data, d.size, 64, 1, 0) == capi.Status.OK
    assert bool((d == np.uint64(1 << 63)).all())
    e = np.array([5, 1 << 40, 3], dtype=np.uint64)  # 3 keys, span > 2^32
    assert capi.sort_raw(e.ctypes.data, 3, 64, 1, 0) == capi.Status.OK
    assert e.tolist() == [3, 5, 1 << 40]


def test_misaligned_data_rejected(capi):
    a = np.zeros(9, dtype=np.uint8)
    for width in (16, 32, 64):
        assert capi.sort_raw(a.ctypes.data + 1, 2, width, 1, 0) == capi.Status.ERROR_DATA
        assert "aligned" in capi.last_error()


def test_widths_interleaved_with_32bit(capi):
    """Width switches between calls leave no state behind."""
    rng = np.random.default_rng(9)
    for _ in range(2):
        for dt in (np.uint8, np.uint32, np.int16, np.uint64, np.int32):
            keys = rng.integers(0, 200, size=5000).astype(dt)
            assert np.array_equal(_host(capi, keys), np.sort(keys))


def test_concurrent_mixed_widths_and_shutdown(capi):
    """Host threads sorting different widths (counting sort, bitset sort with
    and without repeats, 64-bit narrowing and radix) at the same time share one
    device context safely; bws_gpu_shutdown releases it and the next call
    re-initialises."""
    import threading

    rng = np.random.default_rng(77)
    inputs = [rng.integers(0, 256, size=300_000, dtype=np.uint8),
              rng.integers(-(1 << 15), 1 << 15, size=300_000, dtype=np.int64).astype(np.int16),
              rng.choice(1 << 26, size=1 << 21, replace=False).astype(np.uint32),
              rng.integers(0, 1 << 20, size=1 << 21, dtype=np.uint32),
              rng.integers(0, 1 << 30, size=300_000).astype(np.uint64) + np.uint64(7 << 40),
              rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, size=300_000, dtype=np.int64)]
    expected = [np.sort(a) for a in inputs]
    errors = []

    def work(i):
        try:
            for _ in range(3):
                assert np.array_equal(_host(capi, inputs[i]), expected[i])
        except Exception as e:  # noqa: BLE001
            errors.append((i, e))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(inputs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    capi.lib.bws_gpu_shutdown()
    for a, e in zip(inputs, expected):
        assert np.array_equal(_host(capi, a), e)
