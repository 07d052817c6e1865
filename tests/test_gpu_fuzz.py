"""Randomised GPU parity sweep: sizes, key ranges, layouts, pipelines,
pointer alignments and signedness drawn from a seeded generator, each sort
compared with numpy (a correct sort of distinct keys has exactly one answer).
Bounded to about a minute on a B200.
"""
from __future__ import annotations

import time

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _keys(rng, n, key_range, layout):
    if key_range <= 1 << 26:
        keys = rng.choice(key_range, size=n, replace=False).astype(np.uint64)
    else:
        keys = np.unique(rng.integers(0, key_range, size=n + n // 4 + 16, dtype=np.uint64))
        keys = rng.permutation(keys)[:n]
    if layout == "sorted":
        keys.sort()
    elif layout == "reverse":
        keys = np.sort(keys)[::-1]
    elif layout == "blocks":  # sorted runs in random order
        keys.sort()
        parts = np.array_split(keys, max(1, n // 4096))
        keys = np.concatenate([parts[i] for i in rng.permutation(len(parts))]) if parts else keys
    return keys.astype(np.uint32)


def test_random_sweep(cuda):
    from paper_1312_0138_b200 import capi

    rng = np.random.default_rng(20261019)
    deadline = time.time() + 60
    done = 0
    try:
        while time.time() < deadline and done < 400:
            n = int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 1 << 20), rng.integers(1 << 20, 1 << 23)]))
            lo_bits = max(1, int(np.ceil(np.log2(max(n, 2)))))
            key_range = int(min(1 << 32, (1 << int(rng.integers(lo_bits, 33))) - int(rng.integers(0, 3))))
            key_range = max(key_range, n)
            layout = str(rng.choice(["uniform", "sorted", "reverse", "blocks"]))
            path = str(rng.choice(["AUTO", "DIRECT", "BUCKETED", "FUSED", "FUSED_DIRECT", "SMALL"]))
            offset = int(rng.integers(0, 4))
            signed = bool(rng.random() < 0.2) and key_range == 1 << 32
            keys = _keys(rng, n, key_range, layout)
            capi.set_path(getattr(capi.Path, path))
            ctx = f"n={n} range={key_range} layout={layout} path={path} off={offset} signed={signed}"
            if signed:
                a = keys.view(np.int32).copy()
                assert capi.sort_raw(a.ctypes.data, a.size, 32, 0, 0) == capi.Status.OK, ctx + capi.last_error()
                assert np.array_equal(a, np.sort(keys.view(np.int32))), ctx
            else:
                buf = cuda.zeros(n + offset + 4, dtype=cuda.int32, device="cuda")
                view = buf[offset: offset + n]
                view.copy_(cuda.from_numpy(keys.view(np.int32)))
                stream = cuda.cuda.current_stream().cuda_stream
                hint = key_range if rng.random() < 0.7 else 0
                capi.sort_device_async(view.data_ptr(), n, view.data_ptr(), hint, stream)
                assert capi.sort_check(stream) == n, ctx
                assert np.array_equal(view.cpu().numpy().view(np.uint32), np.sort(keys)), ctx
            done += 1
    finally:
        capi.set_path(capi.Path.AUTO)
    assert done >= 50


def test_random_sweep_full_contract(cuda):
    """The rest of bws_sort's contract under the same kind of sweep: every
    width and signedness, draws WITH replacement (repeats), host and device
    arrays, the three pipelines. About thirty seconds."""
    from paper_1312_0138_b200 import capi

    dtypes = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64]
    rng = np.random.default_rng(20261020)
    deadline = time.time() + 30
    done = 0
    try:
        while time.time() < deadline and done < 300:
            dt = np.dtype(dtypes[int(rng.integers(0, len(dtypes)))])
            info = np.iinfo(dt)
            n = int(rng.choice([rng.integers(1, 3000), rng.integers(3000, 1 << 19), rng.integers(1 << 19, 1 << 22)]))
            span_bits = int(rng.integers(1, info.bits + 1))
            # base + (random & mask) modulo 2^bits: spans of 2^span_bits values
            # anywhere in the type, wrapping across its ends
            r = np.frombuffer(rng.bytes(8 * n), dtype=np.uint64)
            base = np.frombuffer(rng.bytes(8), dtype=np.uint64)[0]
            mask = np.uint64((1 << span_bits) - 1)
            udt = np.dtype(f"uint{info.bits}")
            keys = (base + (r & mask)).astype(udt).view(dt)
            lo, hi = int(base), span_bits
            path = str(rng.choice(["AUTO", "DIRECT", "BUCKETED", "FUSED", "FUSED_DIRECT", "SMALL"]))
            capi.set_path(getattr(capi.Path, path))
            ctx = f"{dt} n={n} base={lo} span=2^{hi} path={path}"
            if rng.random() < 0.5:
                a = keys.copy()
                assert capi.sort_raw(a.ctypes.data, n, info.bits, int(info.min == 0), 0) == capi.Status.OK, \
                    ctx + capi.last_error()
            else:
                t = cuda.from_numpy(keys.view(np.uint8).copy()).cuda()
                assert capi.sort_raw(t.data_ptr(), n, info.bits, int(info.min == 0), 0) == capi.Status.OK, \
                    ctx + capi.last_error()
                a = t.cpu().numpy().view(dt)
            assert np.array_equal(a, np.sort(keys)), ctx
            done += 1
    finally:
        capi.set_path(capi.Path.AUTO)
    assert done >= 30
