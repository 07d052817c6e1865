"""GPU parity: the sm_100a bitset sort through the C ABI vs the reference.

Golden vectors come from the reference's own bws_sort (tests/golden/); small
random cases are checked against the oracle (C restatement of
bitsort.hpp:84-136); full-size configs against reference-generated hashes
(tests/golden/anchors.json) and size-independent properties.
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


@pytest.fixture(autouse=True)
def _auto_mode(capi):
    yield
    capi.set_scatter_mode(capi.ScatterMode.AUTO)
    capi.set_path(capi.Path.AUTO)


PATHS = ["DIRECT", "BUCKETED"]


def gpu_sort_host(capi, keys: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(keys, dtype=np.uint32).copy()
    capi.sort(a)
    return a


def gpu_sort_device(capi, torch, keys: np.ndarray, offset: int = 0) -> np.ndarray:
    buf = torch.zeros(keys.size + offset + 4, dtype=torch.int32, device="cuda")
    view = buf[offset: offset + keys.size]
    view.copy_(torch.from_numpy(keys.view(np.int32)))
    capi.sort(view)
    torch.cuda.synchronize()
    return view.cpu().numpy().view(np.uint32)


# --- golden vectors from the reference ------------------------------------

@pytest.mark.parametrize("path", PATHS)
def test_acceptance_golden_vectors(capi, acceptance_records, path):
    """acceptance.cpp:65-95 criterion-2 inputs (uint32 arm) vs the reference's
    bws_sort output, bit-exact."""
    capi.set_path(getattr(capi.Path, path))
    checked = 0
    for rec in acceptance_records:
        a = rec["input"].copy()
        status = capi.sort_raw(a.ctypes.data, a.size, 32, 1, capi.Algorithm.BITWISE)
        assert status == capi.Status.OK, capi.last_error()
        assert np.array_equal(a, rec["output"]), (rec["n"], rec["trial"])
        checked += 1
    assert checked >= 60


@pytest.mark.parametrize("path", PATHS)
def test_repeats_golden_vectors(capi, cuda, repeats_records, path):
    """Inputs with repeated keys from the reference's own generator (small
    range, constant) vs the reference's bws_sort output, host and device
    arrays: the bitset pass detects the repeats, the counting pass sorts."""
    capi.set_path(getattr(capi.Path, path))
    for rec in repeats_records:
        assert np.array_equal(gpu_sort_host(capi, rec["input"]), rec["output"]), (rec["n"], rec["trial"])
        assert np.array_equal(gpu_sort_device(capi, cuda, rec["input"]), rec["output"])


@pytest.mark.parametrize("path", PATHS)
def test_edge_golden_vectors(capi, cuda, edge_records, path):
    capi.set_path(getattr(capi.Path, path))
    for rec in edge_records:
        assert np.array_equal(gpu_sort_host(capi, rec["input"]), rec["output"])
        assert np.array_equal(gpu_sort_device(capi, cuda, rec["input"]), rec["output"])


def test_capi_uint8_vector_widened(capi):
    """test_capi.cpp:78-82 {200,3,255,0} -> {0,3,200,255}, at width 32."""
    a = np.array([200, 3, 255, 0], dtype=np.uint32)
    capi.sort(a)
    assert a.tolist() == [0, 3, 200, 255]


# --- the ABI conventions on a GPU ----------------------------------------

@pytest.mark.parametrize("path", PATHS)
def test_status_conventions(capi, path):
    capi.set_path(getattr(capi.Path, path))
    a = np.array([5, 1, 5], dtype=np.uint32)
    assert capi.sort_raw(a.ctypes.data, 3, 32, 1, 0) == capi.Status.OK  # repeats sort like the reference
    assert a.tolist() == [1, 5, 5]
    a = np.array([5, 1, 5], dtype=np.uint32)
    assert capi.lib.bws_sort_u32_range(a.ctypes.data, 3, 16) == capi.Status.ERROR_DATA  # distinct-only extension
    assert "distinct" in capi.last_error()
    assert a.tolist() == [5, 1, 5]  # rejected input left unmodified
    b = np.array([3, 1, 2], dtype=np.uint32)
    assert capi.sort_raw(b.ctypes.data, 3, 32, 1, 0) == capi.Status.OK
    assert capi.last_error() == ""
    assert b.tolist() == [1, 2, 3]
    assert capi.sort_raw(b.ctypes.data, 3, 32, 1, capi.Algorithm.BITWISE_SKIP_EMPTY) == capi.Status.OK
    assert capi.sort_raw(b.ctypes.data, 3, 24, 1, 0) == capi.Status.ERROR_CONFIG
    assert capi.sort_raw(b.ctypes.data, 3, 32, 1, capi.Algorithm.PLATFORM) == capi.Status.OK


@pytest.mark.parametrize("path", PATHS)
def test_every_algorithm_id(capi, path):
    """Every algorithm id sorts on the GPU to the reference's bytes
    (run_algorithm, dispatch.hpp:42-55; test_capi.cpp:83-93 "int64 with every
    algorithm"), and COUNTING keeps the reference's span limit: a span >= 2^26
    is BWS_ERROR_RANGE naming the span (test_capi.cpp:98-101), data untouched."""
    import oracle

    capi.set_path(getattr(capi.Path, path))
    cases = [(np.array([5, -9, 0, 5, -9, 123456789], dtype=np.int64), 64, 0),
             (np.array([3, -1, 0, -7, 2], dtype=np.int16), 16, 0),
             (np.array([200, 3, 255, 0], dtype=np.uint8), 8, 1),
             (np.random.default_rng(4).integers(0, 1 << 25, 5000).astype(np.uint32), 32, 1),
             (np.random.default_rng(5).integers(-(1 << 24), 1 << 24, 5000).astype(np.int32), 32, 0)]
    for alg in capi.Algorithm:
        for keys, width, uns in cases:
            a = keys.copy()
            span = int(keys.astype(np.int64).max()) - int(keys.astype(np.int64).min())
            if alg == capi.Algorithm.COUNTING and span >= 1 << 26:  # baselines.hpp:95-110 span limit
                assert capi.sort_raw(a.ctypes.data, a.size, width, uns, alg) == capi.Status.ERROR_RANGE
                assert np.array_equal(a, keys)
                if oracle.REFERENCE is not None:
                    r = keys.copy()
                    assert oracle.REFERENCE.bws_sort(r.ctypes.data, r.size, width, uns, int(alg)) == 4
                continue
            assert capi.sort_raw(a.ctypes.data, a.size, width, uns, alg) == capi.Status.OK, capi.last_error()
            assert np.array_equal(a, np.sort(keys)), (alg, keys.dtype)
            if oracle.REFERENCE is not None:
                r = keys.copy()
                assert oracle.REFERENCE.bws_sort(r.ctypes.data, r.size, width, uns, int(alg)) == 0
                assert np.array_equal(a, r)
    for keys, width, uns in [(np.array([0, 1 << 30], dtype=np.int32), 32, 0),
                             (np.array([7, 7 + (1 << 26)], dtype=np.uint32), 32, 1),
                             (np.array([-5, (1 << 26) - 5], dtype=np.int64), 64, 0)]:
        a = keys.copy()
        assert capi.sort_raw(a.ctypes.data, a.size, width, uns, capi.Algorithm.COUNTING) == capi.Status.ERROR_RANGE
        assert "span" in capi.last_error()
        assert np.array_equal(a, keys)
        if oracle.REFERENCE is not None:
            r = keys.copy()
            assert oracle.REFERENCE.bws_sort(r.ctypes.data, r.size, width, uns, 4) == 4  # BWS_ERROR_RANGE
    # a span just under the limit sorts
    a = np.array([7 + (1 << 26) - 1, 7], dtype=np.uint32)
    assert capi.sort_raw(a.ctypes.data, 2, 32, 1, capi.Algorithm.COUNTING) == capi.Status.OK
    assert a.tolist() == [7, 7 + (1 << 26) - 1]


@pytest.mark.parametrize("path", PATHS)
def test_range_hint(capi, path):
    capi.set_path(getattr(capi.Path, path))
    keys = np.array([9, 0, 15, 3], dtype=np.uint32)
    a = keys.copy()
    capi.sort_u32_range(a, 16)
    assert a.tolist() == [0, 3, 9, 15]
    b = keys.copy()
    with pytest.raises(capi.BitsortError) as e:
        capi.sort_u32_range(b, 15)  # 15 is not below 15
    assert e.value.status == capi.Status.ERROR_DATA
    assert b.tolist() == keys.tolist()
    with pytest.raises(capi.BitsortError) as e:
        capi.sort_u32_range(b, (1 << 32) + 1)
    assert e.value.status == capi.Status.ERROR_RANGE
    # the bitset cache stays clean after rejected sorts
    c = np.array([2, 1], dtype=np.uint32)
    capi.sort_u32_range(c, 1 << 32)
    assert c.tolist() == [1, 2]


# --- random / ragged / aligned cases vs the oracle -------------------------

@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 31, 32, 33, 100, 1000, 4095, 4096, 4097, 65537])
@pytest.mark.parametrize("key_range", [1 << 12, 1 << 20, 1 << 32])
def test_random_distinct_vs_oracle(capi, cuda, n, key_range, path):
    capi.set_path(getattr(capi.Path, path))
    if n > key_range:
        pytest.skip("n > key_range")
    rng = np.random.default_rng(n * 7919 + key_range % 1000003)
    keys = rng.choice(key_range, size=n, replace=False).astype(np.uint32) if key_range <= 1 << 24 \
        else np.unique(rng.integers(0, key_range, size=2 * n, dtype=np.uint64).astype(np.uint32))[:n]
    rng.shuffle(keys)
    expected = bitwise_sort(keys)
    assert np.array_equal(gpu_sort_host(capi, keys), expected)
    for off in (0, 1, 2, 3):
        assert np.array_equal(gpu_sort_device(capi, cuda, keys, off), expected)
    a = keys.copy()
    capi.sort_u32_range(a, key_range)
    assert np.array_equal(a, expected)


@pytest.mark.parametrize("mode", ["AUTO", "PLAIN", "WARP_AGG", "SMEM", "BUCKETED"])
@pytest.mark.parametrize("layout", ["shuffled", "sorted", "reverse", "runs", "clustered"])
def test_scatter_modes(capi, mode, layout):
    """Warp aggregation and SMEM staging (K2 paths) and the bucketed pipeline
    give identical results on shuffled, sorted and cluster-ordered layouts."""
    if mode == "BUCKETED":
        capi.set_path(capi.Path.BUCKETED)
        mode = "AUTO"
    else:
        capi.set_path(capi.Path.DIRECT)
    rng = np.random.default_rng(5)
    n = 300_000
    if layout == "clustered":
        # cluster-ordered keys (sorted within each of 16 windows): the case the
        # SMEM staging path targets
        centres = rng.choice((1 << 32) - (1 << 17), size=16, replace=False) + (1 << 16)
        keys = np.unique(np.concatenate([
            (c + rng.integers(-(1 << 16), 1 << 16, size=n // 12)) for c in centres]).astype(np.uint32))
        keys = np.concatenate([np.sort(keys[i::16]) for i in range(16)])
    else:
        keys = rng.choice(1 << 26, size=n, replace=False).astype(np.uint32)
        if layout == "sorted":
            keys.sort()
        elif layout == "reverse":
            keys = np.sort(keys)[::-1].copy()
        elif layout == "runs":
            keys = np.arange(n, dtype=np.uint32) * 3 + 17
            rng.shuffle(keys.reshape(-1, 1000))
    capi.set_scatter_mode(getattr(capi.ScatterMode, mode))
    expected = np.sort(keys)
    assert np.array_equal(gpu_sort_host(capi, keys), expected)
    a = keys.copy()
    capi.sort_u32_range(a, 1 << 32)
    assert np.array_equal(a, expected)


@pytest.mark.parametrize("path", PATHS)
def test_dense_identity(capi, cuda, path):
    """n == M: every word full, output is the identity (dense extraction path)."""
    capi.set_path(getattr(capi.Path, path))
    n = 1 << 22
    keys = np.random.default_rng(1).permutation(n).astype(np.uint32)
    t = cuda.from_numpy(keys.view(np.int32)).cuda()
    capi.sort_u32_range(t, n)
    cuda.cuda.synchronize()
    assert cuda.equal(t.cpu(), cuda.arange(n, dtype=cuda.int32))


@pytest.mark.parametrize("path", PATHS)
def test_top_of_range(capi, path):
    capi.set_path(getattr(capi.Path, path))
    keys = (np.uint32(0xFFFFFFFF) - np.arange(5000, dtype=np.uint32) * np.uint32(7)).astype(np.uint32)
    a = keys[::-1].copy()
    capi.sort(a)
    assert np.array_equal(a, np.sort(keys))


@pytest.mark.parametrize("path", PATHS)
def test_one_repeat_at_scale(capi, cuda, path):
    """One repeated key among 2^20: bws_sort sorts it (host and device
    arrays); the distinct-only range extension rejects it untouched."""
    capi.set_path(getattr(capi.Path, path))
    keys = np.random.default_rng(3).choice(1 << 24, size=1 << 20, replace=False).astype(np.uint32)
    keys[777] = keys[123456]
    a = keys.copy()
    assert capi.sort_raw(a.ctypes.data, a.size, 32, 1, 0) == capi.Status.OK, capi.last_error()
    assert np.array_equal(a, np.sort(keys))
    assert np.array_equal(gpu_sort_device(capi, cuda, keys), np.sort(keys))
    b = keys.copy()
    assert capi.lib.bws_sort_u32_range(b.ctypes.data, b.size, 1 << 24) == capi.Status.ERROR_DATA
    assert np.array_equal(b, keys)


# --- signed int32 (x ^ 0x80000000 on load and store, bucketed pipeline) ----

def _reference_signed(keys: np.ndarray) -> np.ndarray:
    import oracle

    a = keys.copy()
    if oracle.REFERENCE is not None:  # the reference's own signed bitwise sort
        assert oracle.REFERENCE.bws_sort(a.ctypes.data, a.size, 32, 0, 0) == 0
        return a
    return oracle.bitwise_sort(a)  # the restatement's signed split


@pytest.mark.parametrize("n", [1, 2, 5, 1000, 65537, 1 << 21])
def test_signed_int32(capi, cuda, n):
    rng = np.random.default_rng(n + 99)
    keys = np.unique(rng.integers(-(1 << 31), 1 << 31, size=n + n // 4 + 8, dtype=np.int64)).astype(np.int32)
    keys = rng.permutation(keys)[:n]
    if n >= 5:
        keys[:4] = [-(1 << 31), -1, 0, (1 << 31) - 1]
        keys = np.unique(keys)
        rng.shuffle(keys)
    expected = _reference_signed(keys)
    assert np.array_equal(expected, np.sort(keys))
    a = keys.copy()
    assert capi.sort_raw(a.ctypes.data, a.size, 32, 0, capi.Algorithm.BITWISE) == capi.Status.OK, capi.last_error()
    assert np.array_equal(a, expected)
    t = cuda.from_numpy(keys.copy()).cuda()  # device pointer, in place
    assert capi.sort_raw(t.data_ptr(), t.numel(), 32, 0, capi.Algorithm.BITWISE) == capi.Status.OK
    assert np.array_equal(t.cpu().numpy(), expected)


@pytest.mark.parametrize("kind", ["all_negative", "dense_window", "duplicate"])
def test_signed_int32_layouts(capi, kind):
    rng = np.random.default_rng(5)
    if kind == "all_negative":
        keys = -(rng.choice(1 << 30, size=1 << 20, replace=False).astype(np.int64) + 1)
    else:  # a dense window straddling zero (both signs, consecutive keys)
        keys = np.arange(-(1 << 20), 1 << 20, dtype=np.int64)
    keys = rng.permutation(keys).astype(np.int32)
    if kind == "duplicate":
        keys[10] = keys[12345]
    a = keys.copy()
    assert capi.sort_raw(a.ctypes.data, a.size, 32, 0, 0) == capi.Status.OK
    assert np.array_equal(a, np.sort(keys))


# --- slab layout of the bucket buffer (KB3 fill counters, no KB1/KB2) -------
# Used when n >= key_range / 4 (kernels.h SlabArgs): n = 2^22 keys below 2^24
# gives 256 buckets of 2^16 slots.

SLAB_N = 1 << 22
SLAB_RANGE = 1 << 24


@pytest.mark.parametrize("extra", [0, 3])
@pytest.mark.parametrize("offset", [0, 1])
def test_slab_layout_vs_oracle(capi, cuda, extra, offset):
    capi.set_path(capi.Path.BUCKETED)
    n = SLAB_N + extra
    keys = np.random.default_rng(21 + extra).choice(SLAB_RANGE, size=n, replace=False).astype(np.uint32)
    expected = np.sort(keys)
    assert np.array_equal(gpu_sort_device(capi, cuda, keys, offset), expected)
    a = keys.copy()
    capi.sort_u32_range(a, SLAB_RANGE)
    assert np.array_equal(a, expected)
    # a non-power-of-two range: the last bucket is partial; a key at the limit is bad
    b = keys.copy()
    capi.sort_u32_range(b, int(keys.max()) + 1)
    assert np.array_equal(b, expected)
    c = keys.copy()
    with pytest.raises(capi.BitsortError) as e:
        capi.sort_u32_range(c, int(keys.max()))
    assert e.value.status == capi.Status.ERROR_DATA
    assert np.array_equal(c, keys)


def test_slab_layout_full_bucket(capi):
    """A bucket that holds every key of its range (2^16 slots exactly full)."""
    capi.set_path(capi.Path.BUCKETED)
    rng = np.random.default_rng(8)
    full = np.arange(5 << 16, 6 << 16, dtype=np.uint32)
    rest = rng.choice(np.setdiff1d(np.arange(SLAB_RANGE, dtype=np.uint32), full),
                      size=SLAB_N - full.size, replace=False).astype(np.uint32)
    keys = np.concatenate([full, rest])
    rng.shuffle(keys)
    a = keys.copy()
    capi.sort_u32_range(a, SLAB_RANGE)
    assert np.array_equal(a, np.sort(keys))


@pytest.mark.parametrize("kind", ["pair", "overflow"])
def test_slab_layout_duplicates(capi, kind):
    """Repeats in the slab layout, including ones that overflow a bucket's
    fixed slots (then that bucket sorts nothing and the popcount total drops):
    the distinct-only range extension rejects them untouched, bws_sort then
    sorts them by the counting-sort pass (from the untouched input)."""
    capi.set_path(capi.Path.BUCKETED)
    keys = np.random.default_rng(4).choice(SLAB_RANGE, size=SLAB_N, replace=False).astype(np.uint32)
    if kind == "pair":
        keys[5] = keys[SLAB_N - 9]
    else:  # 2^17 copies of 40 keys of bucket 7: far past its 2^16 slots
        keys[: 1 << 17] = (7 << 16) + (np.arange(1 << 17, dtype=np.uint32) % 40)
    for _ in range(2):  # and the next sort is unaffected
        a = keys.copy()
        assert capi.lib.bws_sort_u32_range(a.ctypes.data, a.size, SLAB_RANGE) == capi.Status.ERROR_DATA
        assert "distinct" in capi.last_error()
        assert np.array_equal(a, keys)
        assert capi.sort_raw(a.ctypes.data, a.size, 32, 1, 0) == capi.Status.OK, capi.last_error()
        assert np.array_equal(a, np.sort(keys))
    good = np.random.default_rng(5).choice(SLAB_RANGE, size=SLAB_N, replace=False).astype(np.uint32)
    a = good.copy()
    capi.sort_u32_range(a, SLAB_RANGE)
    assert np.array_equal(a, np.sort(good))


@pytest.mark.parametrize("n_log2,range_log2", [(26, 28), (20, 29), (22, 28)])
def test_non_power_of_two_bucket_width(capi, cuda, n_log2, range_log2):
    """Ranges >= 2^28 may use buckets of 7 * 2^17 keys (bucket = umulhi
    mapping; plan_buckets): slab layout (n = 2^26 below 2^28) and packed
    layout (fewer keys), sort and per-rank bitset build, plus duplicates."""
    capi.set_path(capi.Path.BUCKETED)
    n, m = 1 << n_log2, 1 << range_log2
    rng = np.random.default_rng(n_log2 * 31 + range_log2)
    step = m // n  # one key per stride of the range, jittered: distinct by construction
    keys = (np.arange(n, dtype=np.uint64) * step + rng.integers(0, step, size=n)).astype(np.uint32)
    # keys on both sides of the 7 * 2^17 boundaries near the top of the range
    w = 7 << 17
    edges = np.array([b * w + d for b in range(m // w - 2, m // w + 1) for d in (-1, 0, 1)
                      if 0 <= b * w + d < m], dtype=np.uint32)
    keys = np.concatenate([keys[~np.isin(keys, edges)], edges])
    expected = np.sort(keys)
    rng.shuffle(keys)
    t = cuda.from_numpy(keys.view(np.int32)).cuda()
    out = cuda.empty_like(t)
    stream = cuda.cuda.current_stream().cuda_stream
    capi.sort_device_async(t.data_ptr(), t.numel(), out.data_ptr(), m, stream)
    assert capi.sort_check(stream) == keys.size
    got = out.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, expected)
    # per-rank bitset build: bucketed (KB4b) == direct (K2 scatter)
    bits = {}
    for path in ("BUCKETED", "DIRECT"):
        capi.set_path(getattr(capi.Path, path))
        b = cuda.full((m // 32,), -1, dtype=cuda.int32, device="cuda")
        capi.bitset_build(t.data_ptr(), t.numel(), b.data_ptr(), m)
        cuda.cuda.synchronize()
        bits[path] = b
    assert cuda.equal(bits["BUCKETED"], bits["DIRECT"])
    capi.set_path(capi.Path.BUCKETED)
    dup = keys.copy()
    dup[1] = dup[keys.size - 2]
    expected = np.sort(dup)
    assert capi.sort_raw(dup.ctypes.data, dup.size, 32, 1, 0) == capi.Status.OK, capi.last_error()
    assert np.array_equal(dup, expected)


@pytest.mark.parametrize("kind", ["distinct", "overflow"])
def test_slab_layout_bitset_build(capi, cuda, kind):
    """The per-rank bitset build (KB4b) over the slab layout: exact bitset for
    distinct keys; fewer set bits than keys when duplicates overflow a bucket
    (how dist.py detects them)."""
    capi.set_path(capi.Path.BUCKETED)
    keys = np.random.default_rng(6).choice(SLAB_RANGE, size=SLAB_N, replace=False).astype(np.uint32)
    if kind == "overflow":
        keys[: 1 << 17] = (3 << 16) + (np.arange(1 << 17, dtype=np.uint32) % 5)
    src = cuda.from_numpy(keys.view(np.int32)).cuda()
    bits = cuda.full((SLAB_RANGE // 32,), -1, dtype=cuda.int32, device="cuda")
    capi.bitset_build(src.data_ptr(), SLAB_N, bits.data_ptr(), SLAB_RANGE)
    cuda.cuda.synchronize()
    got = np.unpackbits(bits.cpu().numpy().view(np.uint8), bitorder="little")
    if kind == "distinct":
        want = np.zeros(SLAB_RANGE, dtype=np.uint8)
        want[keys] = 1
        assert np.array_equal(got, want)
    else:
        assert int(got.sum()) < SLAB_N


# --- device-resident async API and the multi-rank building blocks ----------

@pytest.mark.parametrize("path", PATHS)
def test_device_async_and_check(capi, cuda, path):
    capi.set_path(getattr(capi.Path, path))
    keys = np.random.default_rng(11).choice(1 << 28, size=1 << 20, replace=False).astype(np.uint32)
    src = cuda.from_numpy(keys.view(np.int32)).cuda()
    out = cuda.empty_like(src)
    stream = cuda.cuda.current_stream().cuda_stream
    for _ in range(3):
        capi.sort_device_async(src.data_ptr(), src.numel(), out.data_ptr(), 1 << 28, stream)
    assert capi.sort_check(stream) == keys.size
    assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))
    # derived key range
    capi.sort_device_async(src.data_ptr(), src.numel(), out.data_ptr(), 0, stream)
    assert capi.sort_check(stream) == keys.size
    assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_rank_building_blocks_emulated(capi, cuda, world, path):
    """The per-rank K2/K3 calls of dist.py, with the reduce-scatter emulated by
    a sum on one GPU (ranks run one after another; nothing waits on anything)."""
    from paper_1312_0138_b200.dist import CudaRankOps, shard_bounds, slice_words

    capi.set_path(getattr(capi.Path, path))
    n, key_range = 200_000, (1 << 22) - 7  # not a multiple of 32: exercises the last-word mask
    keys = np.random.default_rng(world).choice(key_range, size=n, replace=False).astype(np.uint32)
    words, per = slice_words(key_range, world)
    ops = CudaRankOps()
    acc = cuda.zeros(words, dtype=cuda.int32, device="cuda")
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        shard = cuda.from_numpy(keys[lo:hi].view(np.int32)).cuda()
        acc += ops.bitset_build(shard, key_range, words)
    parts = []
    for r in range(world):
        out, cnt = ops.bitset_scan(acc[r * per:(r + 1) * per].contiguous(), r * per * 32, n)
        parts.append(out[: int(cnt.item())].cpu().numpy().view(np.uint32).copy())
    assert np.array_equal(np.concatenate(parts), np.sort(keys))


@pytest.mark.parametrize("world,key_range,n", [(2, (1 << 22) - 7, 200_000), (3, 1 << 32, 300_000),
                                               (8, 1 << 28, 1 << 22), (5, 1000, 1000)])
def test_a2a_building_blocks_emulated(capi, cuda, world, key_range, n):
    """dist.distributed_sort_a2a's per-rank calls on one GPU: range split of
    every input shard, the all-to-all emulated by concatenating each
    destination's groups, then each rank's range sort (keys offset by the
    rank's first key)."""
    from paper_1312_0138_b200.dist import CudaRankOps, part_width, shard_bounds

    rng = np.random.default_rng(world * 7 + n)
    if key_range <= 1 << 28:
        keys = rng.choice(key_range, size=n, replace=False).astype(np.uint32)
    else:
        keys = np.unique(rng.integers(0, key_range, size=2 * n, dtype=np.uint64).astype(np.uint32))[:n]
        rng.shuffle(keys)
    ops = CudaRankOps()
    inbox = [[] for _ in range(world)]
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        shard = cuda.from_numpy(keys[lo:hi].view(np.int32)).cuda()
        grouped, counts, w, ok = ops.range_split(shard, key_range, world)
        assert ok and w == part_width(key_range, world)
        c = counts.cpu().tolist()
        assert sum(c) == hi - lo
        g = grouped[: hi - lo].cpu().numpy().view(np.uint32)
        start = 0
        for d in range(world):
            part = g[start:start + c[d]]
            assert ((part.astype(np.uint64) >= d * w) & (part.astype(np.uint64) < (d + 1) * w)).all()
            inbox[d].append(part)
            start += c[d]
    parts = []
    for d in range(world):
        recv = np.concatenate(inbox[d])
        key_lo, key_hi = min(d * w, key_range), min((d + 1) * w, key_range)
        out, ok = ops.sort_range(cuda.from_numpy(recv.view(np.int32)).cuda(), key_lo, max(key_hi - key_lo, 1))
        assert ok
        parts.append(out.cpu().numpy().view(np.uint32))
    assert np.array_equal(np.concatenate(parts), np.sort(keys))


def test_range_sort_rejects(capi, cuda):
    """Range sort: keys below key_lo or at/after key_lo + key_range, and
    duplicates, are BWS_ERROR_DATA; a valid offset range sorts exactly."""
    from paper_1312_0138_b200.dist import CudaRankOps

    ops = CudaRankOps()
    lo, rng_ = 3 << 28, 1 << 24
    keys = (np.random.default_rng(2).choice(rng_, size=1 << 21, replace=False) + lo).astype(np.uint32)
    t = cuda.from_numpy(keys.view(np.int32)).cuda()
    out, ok = ops.sort_range(t, lo, rng_)
    assert ok and np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))
    for bad in (lo - 1, lo + rng_, int(keys[7])):
        k2 = keys.copy()
        k2[100] = bad
        _, ok = ops.sort_range(cuda.from_numpy(k2.view(np.int32)).cuda(), lo, rng_)
        assert not ok


# --- full-size BASELINE configs -------------------------------------------

def _config_sort(capi, cuda, name, path="AUTO"):
    from paper_1312_0138_b200.configs import CONFIGS

    capi.set_path(getattr(capi.Path, path))
    cfg = CONFIGS[name]
    keys = cfg.generate()
    t = cuda.from_numpy(keys.view(np.int32)).cuda()
    out = cuda.empty_like(t)
    stream = cuda.cuda.current_stream().cuda_stream
    capi.sort_device_async(t.data_ptr(), t.numel(), out.data_ptr(), cfg.key_range, stream)
    assert capi.sort_check(stream) == cfg.n
    return cfg, keys, out


@pytest.mark.parametrize("path", PATHS)
def test_c1_vs_reference(capi, cuda, anchors, path):
    from paper_1312_0138_b200.configs import CONFIGS

    capi.set_path(getattr(capi.Path, path))
    cfg = CONFIGS["C1"]
    keys = cfg.generate()
    assert fnv1a64(keys) == anchors["C1"]["fnv1a64_input"]
    a = keys.copy()
    capi.sort(a)  # the drop-in call, host array, no range hint
    assert fnv1a64(a) == anchors["C1"]["fnv1a64_sorted"]
    assert np.array_equal(a, bitwise_sort(keys))


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["C2", "C4"])
def test_config_vs_reference_hash(capi, cuda, anchors, name, path):
    cfg, keys, out = _config_sort(capi, cuda, name, path)
    assert fnv1a64(keys) == anchors[name]["fnv1a64_input"]
    got = out.cpu().numpy().view(np.uint32)
    assert fnv1a64(got) == anchors[name]["fnv1a64_sorted"]


@pytest.mark.parametrize("path", PATHS)
def test_c3_dense_permutation(capi, cuda, anchors, path):
    """C3 = a permutation of [0, 2^30): the output is the identity, and its
    hash equals the reference sort's output hash (gen_golden.cpp)."""
    cfg, keys, out = _config_sort(capi, cuda, "C3", path)
    assert fnv1a64(keys) == anchors["C3"]["fnv1a64_input"]
    del keys
    assert cuda.equal(out, cuda.arange(cfg.n, dtype=cuda.int32, device="cuda"))
    assert fnv1a64(out.cpu().numpy().view(np.uint32)) == anchors["C3"]["fnv1a64_sorted"]


@pytest.mark.slow
@pytest.mark.parametrize("path", PATHS)
def test_more_than_2_31_keys(capi, cuda, path):
    """n = 2^31 + 5 keys (a permutation of [0, n), n not a power of two): 64-bit
    sizes and offsets everywhere, 32-bit bucket slots still in range; the
    output must be the identity."""
    from paper_1312_0138_b200 import datagen

    capi.set_path(getattr(capi.Path, path))
    n = (1 << 31) + 5
    keys = datagen.permutation(n, seed=3)
    t = cuda.from_numpy(keys.view(np.int32)).cuda()
    del keys
    out = cuda.empty_like(t)
    stream = cuda.cuda.current_stream().cuda_stream
    capi.sort_device_async(t.data_ptr(), n, out.data_ptr(), n, stream)
    assert capi.sort_check(stream) == n
    del t
    ref = cuda.arange(n, dtype=cuda.int64, device="cuda").to(cuda.int32)  # wraps like uint32
    assert cuda.equal(out, ref)


@pytest.mark.parametrize("path", PATHS)
def test_c5_clustered_properties(capi, cuda, anchors, path):
    """Pinned to the reference: input and sorted-output hashes equal the ones
    gen_golden.cpp recorded from the reference bws_sort of the same C5 keys.
    Also the size-independent properties: strictly ascending, same count, and
    the same sum and sum-of-squares (mod 2^64) as the input."""
    cfg, keys, out = _config_sort(capi, cuda, "C5", path)
    assert fnv1a64(keys) == anchors["C5"]["fnv1a64_input"]
    assert fnv1a64(out.cpu().numpy().view(np.uint32)) == anchors["C5"]["fnv1a64_sorted"]
    u = out.to(cuda.int64) & 0xFFFFFFFF
    assert u.numel() == cfg.n
    assert bool((u[1:] > u[:-1]).all())
    k = cuda.from_numpy(keys.view(np.int32)).cuda().to(cuda.int64) & 0xFFFFFFFF
    assert int(u.sum()) == int(k.sum())
    assert int((u * u).sum()) == int((k * k).sum())
    assert int(u[0]) == int(keys.min()) and int(u[-1]) == int(keys.max())


@pytest.mark.parametrize("world,key_range,n", [(2, (1 << 22) - 7, 200_000), (8, 1 << 26, 1 << 22)])
def test_p2p_or_gather_emulated(capi, cuda, world, key_range, n):
    """dist.distributed_sort_p2p's per-rank calls on one GPU: every shard's
    full bitset in its own buffer (the ranks' exported bitsets), each rank's
    slice OR-gathered from all of them (bws_gpu_bitset_or_gather, here with
    local pointers instead of IPC-opened peer pointers), then scanned."""
    from paper_1312_0138_b200.dist import CudaRankOps, shard_bounds, slice_words

    keys = np.random.default_rng(world + 5).choice(key_range, size=n, replace=False).astype(np.uint32)
    words, per = slice_words(key_range, world)
    ops = CudaRankOps()
    bitsets = []
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        shard = cuda.from_numpy(keys[lo:hi].view(np.int32)).cuda()
        bitsets.append(ops.bitset_build(shard, key_range, words).clone())
    parts = []
    for r in range(world):
        sl = ops.or_gather(bitsets, r * per, per).clone()
        ref = bitsets[0][r * per:(r + 1) * per].clone()
        for b in bitsets[1:]:
            ref |= b[r * per:(r + 1) * per]
        assert cuda.equal(sl, ref)
        out, cnt = ops.bitset_scan(sl, r * per * 32, n)
        got = out[: int(cnt.item())].cpu().numpy().view(np.uint32).copy()
        parts.append(got)
        # the fused exchange + scan (bws_gpu_bitset_scan_sources, local source first)
        srcs = [bitsets[r]] + [b for q, b in enumerate(bitsets) if q != r]
        out2, cnt2 = ops.or_scan(srcs, r * per, per, r * per * 32, n)
        assert int(cnt2.item()) == got.size
        assert np.array_equal(out2[: got.size].cpu().numpy().view(np.uint32), got)
    assert np.array_equal(np.concatenate(parts), np.sort(keys))
    # odd word counts and misaligned pointers take the scalar path
    a = cuda.arange(1, 1000, dtype=cuda.int32, device="cuda")
    b = cuda.arange(1000, 1999, dtype=cuda.int32, device="cuda")
    dst = cuda.zeros(998, dtype=cuda.int32, device="cuda")
    capi.bitset_or_gather([a[1:].data_ptr(), b[1:].data_ptr()], 998, dst.data_ptr())
    cuda.cuda.synchronize()
    assert cuda.equal(dst, a[1:] | b[1:])


@pytest.mark.parametrize("nsrc", [1, 2, 3, 8])
@pytest.mark.parametrize("n_words,offset", [(1, 0), (8191, 0), (8192, 4), (8195, 4), (50_003, 0),
                                            (300_000, 4), (1000, 1), (77_777, 3)])
def test_scan_sources_vs_numpy(capi, cuda, nsrc, n_words, offset):
    """bws_gpu_bitset_scan_sources on random disjoint-bit slices: ragged tile
    tails, aligned (fused kernel) and misaligned (OR-gather + scan) sources,
    against numpy. offset shifts every source by that many words."""
    rng = np.random.default_rng(nsrc * 1000 + n_words + offset)
    owner = rng.integers(0, nsrc, size=n_words * 32)
    present = rng.random(n_words * 32) < 0.3
    bufs = []
    for s in range(nsrc):
        bits = np.zeros(n_words * 32, dtype=bool)
        bits[(owner == s) & present] = True
        words = np.packbits(bits.reshape(-1, 8)[:, ::-1]).view("<u4")
        t = cuda.zeros(n_words + offset, dtype=cuda.int32, device="cuda")
        t[offset:] = cuda.from_numpy(words.view(np.int32).copy()).cuda()
        bufs.append(t)
    expected = (np.flatnonzero(present).astype(np.uint64) + 12345).astype(np.uint32)
    out = cuda.full((expected.size + 7,), -1, dtype=cuda.int32, device="cuda")
    total = cuda.zeros(1, dtype=cuda.int64, device="cuda")
    capi.bitset_scan_sources([b.data_ptr() + 4 * offset for b in bufs], n_words, 12345, out.data_ptr(),
                             out.numel(), total.data_ptr())
    cuda.cuda.synchronize()
    assert int(total.item()) == expected.size
    assert np.array_equal(out[: expected.size].cpu().numpy().view(np.uint32), expected)
    assert bool((out[expected.size:] == -1).all())


@pytest.mark.parametrize("world,key_range,n", [(2, (1 << 22) - 7, 200_000), (8, 1 << 26, 1 << 22),
                                             (3, 1 << 32, 1 << 21), (8, 1 << 28, 1 << 24), (1, 5000, 3000)])
def test_push_build_emulated(capi, cuda, world, key_range, n):
    """dist.distributed_sort_push's per-rank calls on one GPU: every emulated
    rank ORs its shard's bucket bitsets into ALL ranks' slices
    (bws_gpu_bitset_push, local pointers here instead of IPC-opened peer
    pointers), then each slice is scanned; the concatenation is the sort."""
    from paper_1312_0138_b200.dist import CudaRankOps, push_slice_words, shard_bounds

    keys = np.random.default_rng(world + 11).choice(key_range, size=n, replace=False).astype(np.uint32)
    per = push_slice_words(key_range, world)
    ops = CudaRankOps()
    slices = [ops.alloc_slice(per) for _ in range(world)]
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        shard = cuda.from_numpy(keys[lo:hi].view(np.int32)).cuda()
        ops.bitset_push(shard, key_range, slices, per)
    cuda.cuda.synchronize()
    parts = []
    for r in range(world):
        out, cnt = ops.bitset_scan(slices[r], r * per * 32, n)
        parts.append(out[: int(cnt.item())].cpu().numpy().view(np.uint32).copy())
    assert np.array_equal(np.concatenate(parts), np.sort(keys))
    # the full bitset is the OR of the slices: equal to the direct build
    full = cuda.cat(slices)[: (key_range + 31) // 32]
    ref = cuda.full(((key_range + 31) // 32,), -1, dtype=cuda.int32, device="cuda")
    t = cuda.from_numpy(keys.view(np.int32)).cuda()
    capi.bitset_build(t.data_ptr(), t.numel(), ref.data_ptr(), key_range)
    cuda.cuda.synchronize()
    assert cuda.equal(full, ref)


def test_push_argument_checks(capi, cuda):
    s = cuda.zeros(8, dtype=cuda.int32, device="cuda")
    k = cuda.zeros(4, dtype=cuda.int32, device="cuda")
    with pytest.raises(capi.BitsortError) as e:
        capi.bitset_push(k.data_ptr(), 4, 1 << 10, [s.data_ptr()], 6)  # not a multiple of 4
    assert e.value.status == capi.Status.ERROR_RANGE
    with pytest.raises(capi.BitsortError) as e:
        capi.bitset_push(k.data_ptr(), 4, 1 << 10, [s.data_ptr()], 4)  # 4 words cover 128 keys only
    assert e.value.status == capi.Status.ERROR_RANGE
    with pytest.raises(capi.BitsortError) as e:
        capi.bitset_push(k.data_ptr(), 4, 1 << 7, [s.data_ptr() + 4], 4)  # misaligned slice
    assert e.value.status == capi.Status.ERROR_DATA


def test_ipc_handle_offsets(capi, cuda):
    t = cuda.empty(1 << 20, dtype=cuda.int32, device="cuda")
    h0, off0 = capi.ipc_get_handle(t.data_ptr())
    h1, off1 = capi.ipc_get_handle(t[1000:].data_ptr())
    assert len(h0) == capi.IPC_HANDLE_BYTES and h0 == h1 and off1 == off0 + 4000


@pytest.mark.parametrize("variant", ["reduce_scatter", "all_to_all", "p2p", "push"])
def test_distributed_sort_nccl_single_rank(capi, cuda, variant):
    """dist.distributed_sort (bitset build, NCCL reduce-scatter, all-gather,
    K3 on the slice) and dist.distributed_sort_a2a (range split, NCCL
    all-to-all, range sort) over a real NCCL process group (world size 1 on
    the one GPU available). Multi-rank host logic is covered on gloo in
    tests/test_dist_gloo.py."""
    import torch.distributed as dist

    from paper_1312_0138_b200.dist import distributed_sort as rs
    from paper_1312_0138_b200.dist import distributed_sort_a2a as a2a
    from paper_1312_0138_b200.dist import distributed_sort_p2p as p2p
    from paper_1312_0138_b200.dist import distributed_sort_push as push

    distributed_sort = {"all_to_all": a2a, "p2p": p2p, "push": push}.get(variant, rs)

    store = dist.HashStore()
    dist.init_process_group("nccl", store=store, rank=0, world_size=1,
                            device_id=cuda.device("cuda", 0))
    try:
        keys = np.random.default_rng(77).choice(1 << 24, size=1 << 22, replace=False).astype(np.uint32)
        t = cuda.from_numpy(keys.view(np.int32)).cuda()
        res = distributed_sort(t, 1 << 24)
        assert res.total == keys.size and res.offset == 0 and res.count == keys.size
        assert np.array_equal(res.keys.cpu().numpy().view(np.uint32), np.sort(keys))
        bad = keys.copy()
        bad[5] = bad[6]
        from paper_1312_0138_b200.capi import BitsortError

        with pytest.raises(BitsortError):
            distributed_sort(cuda.from_numpy(bad.view(np.int32)).cuda(), 1 << 24)
    finally:
        dist.destroy_process_group()


def test_concurrent_host_threads(capi):
    """The reference is reentrant: concurrent bws_sort calls from
    several host threads on distinct arrays must all succeed."""
    import threading

    rng = np.random.default_rng(123)
    arrays = [rng.choice(1 << 26, size=200_000 + 1000 * i, replace=False).astype(np.uint32) for i in range(6)]
    expected = [np.sort(a) for a in arrays]
    errors = []

    def work(i):
        try:
            for _ in range(3):
                a = arrays[i].copy()
                capi.sort(a)
                assert np.array_equal(a, expected[i])
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(arrays))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


def test_pageable_and_pinned_host_paths(capi, cuda):
    keys = np.random.default_rng(9).choice(1 << 28, size=1 << 21, replace=False).astype(np.uint32)
    pageable = keys.copy()
    capi.sort(pageable)
    pinned_t = cuda.empty(keys.size, dtype=cuda.int32, pin_memory=True)
    pinned = pinned_t.numpy().view(np.uint32)
    np.copyto(pinned, keys)
    capi.sort(pinned)
    assert np.array_equal(pageable, np.sort(keys)) and np.array_equal(pinned, pageable)


def test_async_check_survives_other_calls(capi, cuda):
    """bws_gpu_sort_check validates the most recent ASYNC sort even when other
    library calls (a bws_sort, a bitset build) ran on the device in between:
    their control-block resets no longer overwrite its result."""
    rng = np.random.default_rng(21)
    stream = cuda.cuda.current_stream().cuda_stream
    for n in (1 << 12, 1 << 22):  # direct and bucketed pipelines
        keys = rng.choice(1 << 24, size=n, replace=False).astype(np.uint32)
        bad = keys.copy()
        bad[7] = bad[9]  # one duplicate
        for arr, ok in ((keys, True), (bad, False)):
            t = cuda.from_numpy(arr.view(np.int32)).cuda()
            out = cuda.empty_like(t)
            capi.sort_device_async(t.data_ptr(), n, out.data_ptr(), 1 << 24, stream)
            other = rng.choice(1 << 20, size=5000, replace=False).astype(np.uint32)
            capi.sort(other)  # a synchronous sort reuses the control block
            bits = cuda.empty((1 << 24) // 32, dtype=cuda.int32, device="cuda")
            capi.bitset_build(t.data_ptr(), 100, bits.data_ptr(), 1 << 24, stream)  # so does a build
            if ok:
                assert capi.sort_check(stream) == n
                assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))
            else:
                with pytest.raises(capi.BitsortError) as e:
                    capi.sort_check(stream)
                assert e.value.status == capi.Status.ERROR_DATA


def test_async_without_hint_is_graph_capturable(capi, cuda):
    """bws_gpu_sort_device_async with key_range == 0 derives the range on the
    device (no host round trip), so it can be captured in a CUDA graph."""
    n = 1 << 21
    keys = np.random.default_rng(22).choice(1 << 26, size=n, replace=False).astype(np.uint32)
    t = cuda.from_numpy(keys.view(np.int32)).cuda()
    out = cuda.empty_like(t)
    s = cuda.cuda.Stream()
    with cuda.cuda.stream(s):
        capi.sort_device_async(t.data_ptr(), n, out.data_ptr(), 0, s.cuda_stream)  # warm-up
    s.synchronize()
    g = cuda.cuda.CUDAGraph()
    with cuda.cuda.graph(g, stream=s):
        capi.sort_device_async(t.data_ptr(), n, out.data_ptr(), 0, s.cuda_stream)
    out.zero_()
    g.replay()
    s.synchronize()
    assert capi.sort_check(s.cuda_stream) == n
    assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))


@pytest.mark.parametrize("layout", ["uniform", "clustered", "sorted"])
def test_chunked_layout(capi, cuda, layout):
    """Distinct keys over 2^32 that do not fit the slab take the chunked
    layout (no KB1 histogram): runs claimed into pool chunks allocated on
    first touch, including runs longer than a chunk (sorted / clustered)."""
    capi.set_path(capi.Path.BUCKETED)
    rng = np.random.default_rng(23)
    n = (1 << 22) + 5
    if layout == "uniform":
        keys = np.unique(rng.integers(0, 1 << 32, size=n + n // 64, dtype=np.uint64).astype(np.uint32))[:n]
        rng.shuffle(keys)
    elif layout == "clustered":  # 64 dense clusters, cluster-ordered
        centres = rng.choice((1 << 32) - (1 << 20), size=64, replace=False)
        keys = np.unique(np.concatenate([c + rng.choice(1 << 19, size=n // 64 + 1, replace=False)
                                         for c in centres]).astype(np.uint32))
        keys = np.concatenate([np.sort(keys[i::64]) for i in range(64)])
    else:
        keys = np.sort(np.unique(rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)))
    s = cuda.cuda.current_stream().cuda_stream
    d = cuda.from_numpy(keys.view(np.int32)).cuda()
    out = cuda.full((keys.size + 4,), -1, dtype=cuda.int32, device="cuda")
    capi.set_kernel_timing(True)
    capi.kernel_timings()
    try:
        capi.sort_device_async(d.data_ptr(), keys.size, out.data_ptr(), 1 << 32, s)
        assert capi.sort_check(s) == keys.size
        kernels = capi.kernel_timings()
    finally:
        capi.set_kernel_timing(False)
    assert "bucket_hist" not in kernels and "bucket_partition" in kernels, kernels
    got = out.cpu().numpy().view(np.uint32)
    assert got[keys.size:].tolist() == [0xFFFFFFFF] * 4
    assert np.array_equal(got[: keys.size], np.sort(keys))
