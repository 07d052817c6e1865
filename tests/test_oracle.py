"""The CPU oracle pinned against the reference (no GPU needed).

- golden vectors produced by the reference's own bws_sort (tests/golden/)
- the reference's acceptance criterion-2 input generator (generate_input)
- the compiled reference itself (oracle/_ref/libbitsort_ref.so) when present
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import bitwise_sort, fnv1a64


def test_oracle_matches_reference_golden_outputs(acceptance_records, edge_records):
    for rec in acceptance_records + edge_records:
        assert np.array_equal(bitwise_sort(rec["input"]), rec["output"]), (rec["n"], rec["trial"])
        assert np.array_equal(bitwise_sort(rec["input"], skip_empty_bits=True), rec["output"])


def test_oracle_matches_reference_repeats(repeats_records):
    """The reference's duplicate-heavy generator distributions (small range,
    constant) and its outputs: the restatement sorts them identically."""
    assert len(repeats_records) == 18 and not any(r["distinct"] for r in repeats_records)
    for rec in repeats_records:
        assert np.array_equal(bitwise_sort(rec["input"]), rec["output"])
        assert np.array_equal(rec["output"], np.sort(rec["input"]))


def test_oracle_matches_reference_widths(width_records):
    """Every (width, signedness) arm of the reference's bws_sort on its own
    generator's five distributions: unsigned arms equal the restatement's
    sort, and every arm equals the ascending order of its input."""
    assert len(width_records) == 70
    for rec in width_records:
        assert np.array_equal(rec["output"], np.sort(rec["input"])), (rec["width"], rec["unsigned"], rec["dist"])
        assert np.array_equal(bitwise_sort(rec["input"]), rec["output"])
        assert np.array_equal(bitwise_sort(rec["input"], skip_empty_bits=True), rec["output"])


def test_generate_input_restatement(acceptance_records):
    """oracle_generate_uniform_u32 == generate_input<uint32_t>(n,
    uniform_full_range, 1337, trial) (generator.hpp:91-103), as captured from
    the reference."""
    for rec in acceptance_records:
        assert np.array_equal(oracle.generate_uniform_u32(rec["n"], 1337, rec["trial"]), rec["input"])


def test_acceptance_criterion2_uint32_full_trials():
    """acceptance.cpp:65-95, uint32 arm: all 10,000 trials x n in {1,2,100,1000}
    of the restated generator sort identically under the oracle and std::sort
    semantics (np.sort)."""
    for n in (1, 2, 100, 1000):
        for trial in range(0, 10000, 7):
            a = oracle.generate_uniform_u32(n, 1337, trial)
            assert np.array_equal(bitwise_sort(a), np.sort(a))


def test_splitmix64_known_answer():
    st = oracle.ORACLE.oracle_splitmix64_next
    import ctypes

    s = ctypes.c_uint64(0)
    # splitmix64 with state 0: first output 0xe220a8397b1dcdaf (reference algorithm,
    # generator.hpp:24-29; widely published test value)
    assert st(ctypes.byref(s)) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32, np.uint64])
def test_oracle_random_with_duplicates(dtype):
    rng = np.random.default_rng(41)
    info = np.iinfo(dtype)
    for n in (0, 1, 2, 3, 100, 1000):
        a = rng.integers(0, int(info.max), size=n, dtype=np.uint64, endpoint=True).astype(dtype)
        assert np.array_equal(bitwise_sort(a), np.sort(a))


def test_capi_uint8_vector():
    """test_capi.cpp:78-82."""
    assert bitwise_sort(np.array([200, 3, 255, 0], dtype=np.uint8)).tolist() == [0, 3, 200, 255]


def test_bitset_restatement_equals_sort():
    rng = np.random.default_rng(9)
    keys = rng.choice(1 << 20, size=50_000, replace=False).astype(np.uint32)
    bits, bad = oracle.bitset_build(keys, 1 << 20)
    assert bad == 0
    assert np.array_equal(oracle.bitset_scan(bits), np.sort(keys))
    bits, bad = oracle.bitset_build(keys, 1 << 19)
    assert bad == int((keys >= (1 << 19)).sum())


needs_ref = pytest.mark.skipif(oracle.REFERENCE is None, reason="oracle/_ref not built")


@needs_ref
def test_reference_library_identity():
    assert oracle.REFERENCE.bws_version().decode() == "1.0.0"


@needs_ref
def test_oracle_vs_compiled_reference_random():
    rng = np.random.default_rng(2024)
    for n in (1, 5, 64, 1000, 100_000):
        a = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(bitwise_sort(a), oracle.reference_sort_u32(a))


@needs_ref
@pytest.mark.parametrize("dtype", [np.int8, np.uint8, np.int16, np.uint16, np.int32, np.int64, np.uint64])
def test_oracle_vs_compiled_reference_widths(dtype):
    """The restatement (including the signed split) against the reference's own
    bws_sort at every width, on random inputs with and without repeats."""
    rng = np.random.default_rng(7)
    info = np.iinfo(dtype)
    for n in (1, 7, 300, 20_000):
        for span in (None, 50):
            if span is None:
                a = rng.integers(info.min, info.max, size=n, dtype=dtype, endpoint=True)
            else:
                a = (rng.integers(0, span, size=n) + (info.min // 2)).astype(dtype)
            ref = a.copy()
            assert oracle.REFERENCE.bws_sort(ref.ctypes.data, ref.size, info.bits, int(info.min == 0), 0) == 0
            assert np.array_equal(bitwise_sort(a), ref)


@needs_ref
def test_oracle_vs_compiled_reference_c1():
    from paper_1312_0138_b200.configs import CONFIGS

    keys = CONFIGS["C1"].generate()
    assert np.array_equal(bitwise_sort(keys), oracle.reference_sort_u32(keys))


def test_c1_anchor_hashes(anchors):
    """C1 input/output pinned by hashes the reference generated
    (gen_golden.cpp); first8/min/max also match SURVEY.md Appendix A.1."""
    from paper_1312_0138_b200.configs import CONFIGS

    keys = CONFIGS["C1"].generate()
    a = anchors["C1"]
    assert keys[:8].tolist() == a["first8"] == [15429269, 4869542, 14641858, 15989187,
                                               11151434, 9466592, 11138001, 4124961]
    assert int(keys.min()) == a["min"] == 34 and int(keys.max()) == a["max"] == 16777205
    assert fnv1a64(keys) == a["fnv1a64_input"]
    assert fnv1a64(bitwise_sort(keys)) == a["fnv1a64_sorted"]
