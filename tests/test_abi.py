"""The drop-in C ABI surface, host-side logic only (no GPU needed).

Mirrors the reference's test_capi.cpp conventions (:10-13, :22-30, :64-70,
:94-97): status codes, thread-local bws_last_error cleared on success,
algorithm names, null-data and width errors. Compute calls are not made here,
except to show that without a GPU the sort fails loudly (no CPU fallback).
"""
from __future__ import annotations

import ctypes
import re
import subprocess
import threading
from pathlib import Path

import numpy as np
import pytest

from paper_1312_0138_b200 import capi

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").rglob("*.h"):
        text = h.read_text()
        names |= set(re.findall(r"BITSORT_API\s+[\w\s\*]+?\b(bws_\w+)\s*\(", text))
    return names


def test_every_declared_symbol_is_exported():
    declared = declared_symbols()
    assert {"bws_sort", "bws_last_error", "bws_version", "bws_algorithm_name",
            "bws_algorithm_from_name"} <= declared
    for name in declared:
        assert hasattr(capi.lib, name), name
    assert declared == set(capi.EXPORTED)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(capi.LIB_PATH)],
                        capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(bws_\w+)\b", nm))
    assert exported == declared
    # hidden visibility: nothing but bws_* leaks (static cudart stays internal)
    others = [l for l in nm.splitlines() if l.strip() and " T " in l and "bws_" not in l]
    assert others == []


def test_soname_matches_reference():
    out = subprocess.run(["readelf", "-d", str(capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "libbitsort.so.1" in out


def test_enums_match_reference_values():
    # bitsort.h:29-45
    assert [s.value for s in capi.Status] == [0, 1, 2, 3, 4, 5]
    assert [a.value for a in capi.Algorithm] == [0, 1, 2, 3, 4, 5]


def test_version_and_error_strings_exist():
    assert capi.version() == "1.0.0"
    assert isinstance(capi.last_error(), str)


def test_algorithm_names():
    # test_capi.cpp:64-70
    assert capi.algorithm_name(capi.Algorithm.BITWISE) == "bitwise"
    names = ["bitwise", "bitwise_skip_empty", "insertion", "merge", "counting", "platform"]
    for i, name in enumerate(names):
        assert capi.algorithm_name(i) == name
        assert capi.algorithm_from_name(name) == i
    assert capi.algorithm_name(99) == "unknown"
    assert capi.algorithm_from_name("merge") == capi.Algorithm.MERGE
    with pytest.raises(capi.BitsortError) as e:
        capi.algorithm_from_name("quick")
    assert e.value.status == capi.Status.ERROR_CONFIG
    assert "quick" in capi.last_error()
    out = ctypes.c_int(0)
    assert capi.lib.bws_algorithm_from_name(None, ctypes.byref(out)) == capi.Status.ERROR_CONFIG


def test_empty_and_null_data():
    # test_capi.cpp:94-97 (signed width 32, count 0 -> OK as in the reference)
    assert capi.sort_raw(None, 0, 32, 0, capi.Algorithm.BITWISE) == capi.Status.OK
    assert capi.last_error() == ""
    assert capi.sort_raw(None, 3, 32, 0, capi.Algorithm.BITWISE) == capi.Status.ERROR_DATA
    assert "null data" in capi.last_error()
    assert capi.sort_raw(None, 0, 32, 1, capi.Algorithm.BITWISE) == capi.Status.OK


def test_config_errors():
    a = np.array([3, 1, 2], dtype=np.uint32)
    p = a.ctypes.data
    assert capi.sort_raw(p, 3, 24, 1, 0) == capi.Status.ERROR_CONFIG  # dispatch.hpp:36-38
    assert "unsupported width 24" in capi.last_error()
    assert capi.sort_raw(p, 3, 32, 1, 99) == capi.Status.ERROR_CONFIG  # capi.cpp:69
    assert "unknown algorithm id" in capi.last_error()
    assert a.tolist() == [3, 1, 2]


def test_every_algorithm_needs_the_gpu():
    """Every algorithm id goes to the GPU pipelines (no CPU fallback): without a
    device the call fails loudly with BWS_ERROR_INTERNAL and leaves the data."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present (tests/test_gpu_parity.py covers the sorts)")
    a = np.array([3, 1, 2], dtype=np.uint32)
    for alg in capi.Algorithm:
        assert capi.sort_raw(a.ctypes.data, 3, 32, 1, alg) == capi.Status.ERROR_INTERNAL
        assert "no CUDA device" in capi.last_error()
    assert a.tolist() == [3, 1, 2]


def test_last_error_is_thread_local_and_cleared():
    assert capi.sort_raw(None, 3, 32, 1, 0) == capi.Status.ERROR_DATA
    seen = {}

    def other():
        seen["before"] = capi.last_error()
        capi.sort_raw(None, 0, 32, 1, 0)
        seen["after"] = capi.last_error()

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen["before"] == ""
    assert "null data" in capi.last_error()
    capi.algorithm_from_name("bitwise")  # success clears
    assert capi.last_error() == ""


def test_extension_argument_checks():
    assert capi.lib.bws_sort_u32_range(None, 3, 16) == capi.Status.ERROR_DATA
    assert capi.lib.bws_gpu_set_scatter_mode(7) == capi.Status.ERROR_CONFIG
    assert capi.lib.bws_gpu_bitset_scan(None, 0, 0, None, 0, None, None) == capi.Status.ERROR_DATA
    assert capi.launch_count() >= 0
    import ctypes

    w = ctypes.c_uint64(0)
    # range split: parts and range are checked before any device is touched
    assert capi.lib.bws_gpu_range_split(None, 0, 1 << 20, 0, None, None, ctypes.byref(w), None) == \
        capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_range_split(None, 0, 0, 2, None, None, ctypes.byref(w), None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_range_split(None, 5, 1 << 20, 2, None, None, ctypes.byref(w), None) == \
        capi.Status.ERROR_DATA
    # range sort: [key_lo, key_lo + key_range) must be non-empty and within 2^32
    assert capi.lib.bws_gpu_sort_range_device_async(None, 0, None, 5, 0, None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_sort_range_device_async(None, 0, None, 1 << 31, 1 << 31 | 1, None) == \
        capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_sort_range_device_async(None, 3, None, 0, 16, None) == capi.Status.ERROR_DATA
    # OR-gather: 1..8 sources
    assert capi.lib.bws_gpu_bitset_or_gather(None, 0, 0, None, None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_bitset_or_gather(None, 9, 0, None, None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_bitset_scan_sources(None, 0, 0, 0, None, 0, None, None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_bitset_scan_sources(None, 9, 0, 0, None, 0, None, None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_bitset_push(None, 0, 1 << 10, None, 0, 32, None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_bitset_push(None, 0, 1 << 10, None, 1, 30, None) == capi.Status.ERROR_RANGE
    assert capi.lib.bws_gpu_ipc_get_handle(None, None, None) == capi.Status.ERROR_DATA


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    a = np.array([3, 1, 2], dtype=np.uint32)
    assert capi.sort_raw(a.ctypes.data, 3, 32, 1, 0) == capi.Status.ERROR_INTERNAL
    assert "no CPU fallback" in capi.last_error()
    assert a.tolist() == [3, 1, 2]
    s = np.array([3, -1, 2], dtype=np.int32)  # signed int32 goes to the GPU too
    assert capi.sort_raw(s.ctypes.data, 3, 32, 0, 0) == capi.Status.ERROR_INTERNAL
    assert "no CPU fallback" in capi.last_error()
    assert s.tolist() == [3, -1, 2]


def test_device_count_configuration_errors():
    """bws_gpu_set_device_count / bws_gpu_set_devices reject bad arguments with
    BWS_ERROR_CONFIG before touching a device."""
    assert capi.lib.bws_gpu_set_device_count(0) == capi.Status.ERROR_CONFIG
    assert "device count" in capi.last_error()
    assert capi.lib.bws_gpu_set_devices(None, 2) == capi.Status.ERROR_CONFIG
    assert capi.device_count() == 1
