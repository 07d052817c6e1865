"""ctypes mirror of the bitsort C ABI (B200 build).

Names, argument meaning and status codes follow the reference interface
(/root/reference/proj/include/bitsort/bitsort.h:29-90, proj/src/capi.cpp:19-41,
:164-197) so the parity tests read like the reference's test_capi.cpp. Every
call goes through ``lib/libbitsort.so.1``; if that library is missing the import
fails loudly -- there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes
import enum
from typing import Optional

import numpy as np

from . import LIB_DIR

import os as _os
from pathlib import Path as _Path

# BITSORT_LIB overrides the library path (A/B experiments on kernel builds)
LIB_PATH = _Path(_os.environ["BITSORT_LIB"]) if _os.environ.get("BITSORT_LIB") else LIB_DIR / "libbitsort.so.1"


class Status(enum.IntEnum):
    """bws_status (bitsort.h:29-36)."""

    OK = 0
    ERROR_CONFIG = 1
    ERROR_DATA = 2
    ERROR_INTEGRITY = 3
    ERROR_RANGE = 4
    ERROR_INTERNAL = 5


class Algorithm(enum.IntEnum):
    """bws_algorithm (bitsort.h:38-45)."""

    BITWISE = 0
    BITWISE_SKIP_EMPTY = 1
    INSERTION = 2
    MERGE = 3
    COUNTING = 4
    PLATFORM = 5


class ScatterMode(enum.IntEnum):
    """bws_scatter_mode (bitsort_gpu.h)."""

    AUTO = 0
    PLAIN = 1
    WARP_AGG = 2
    SMEM = 3


class Path(enum.IntEnum):
    """bws_path (bitsort_gpu.h)."""

    AUTO = 0
    DIRECT = 1
    BUCKETED = 2
    FUSED = 3
    FUSED_DIRECT = 4
    SMALL = 5


class BitsortError(RuntimeError):
    """A non-OK bws_status, with the thread's bws_last_error() text."""

    def __init__(self, status: int, message: str):
        self.status = Status(status)
        self.message = message
        super().__init__(f"{self.status.name}: {message}")


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 bitset sort has no fallback implementation)")
    lib = ctypes.CDLL(str(LIB_PATH))
    u32, u64, sz, vp, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int
    sigs = {
        "bws_version": (ctypes.c_char_p, []),
        "bws_last_error": (ctypes.c_char_p, []),
        "bws_algorithm_name": (ctypes.c_char_p, [i32]),
        "bws_algorithm_from_name": (i32, [ctypes.c_char_p, ctypes.POINTER(i32)]),
        "bws_sort": (i32, [vp, sz, u32, i32, i32]),
        "bws_sort_u32_range": (i32, [vp, sz, u64]),
        "bws_gpu_sort_device_async": (i32, [vp, sz, vp, u64, vp]),
        "bws_gpu_sort_check": (i32, [vp, ctypes.POINTER(u64)]),
        "bws_gpu_sort_range_device_async": (i32, [vp, sz, vp, u32, u64, vp]),
        "bws_gpu_range_split": (i32, [vp, sz, u64, i32, vp, vp, ctypes.POINTER(u64), vp]),
        "bws_gpu_bitset_or_gather": (i32, [ctypes.POINTER(vp), i32, u64, vp, vp]),
        "bws_gpu_bitset_scan_sources": (i32, [ctypes.POINTER(vp), i32, u64, u32, vp, u64, vp, vp]),
        "bws_gpu_bitset_push": (i32, [vp, sz, u64, ctypes.POINTER(vp), i32, u64, vp]),
        "bws_gpu_ipc_get_handle": (i32, [vp, vp, ctypes.POINTER(u64)]),
        "bws_gpu_ipc_open": (i32, [vp, ctypes.POINTER(vp)]),
        "bws_gpu_ipc_close": (i32, [vp]),
        "bws_gpu_bitset_build": (i32, [vp, sz, vp, u64, vp]),
        "bws_gpu_bitset_scan": (i32, [vp, u64, u32, vp, u64, vp, vp]),
        "bws_gpu_set_scatter_mode": (i32, [i32]),
        "bws_gpu_set_path": (i32, [i32]),
        "bws_gpu_launch_count": (u64, []),
        "bws_gpu_set_kernel_timing": (i32, [i32]),
        "bws_gpu_kernel_timings": (i32, [ctypes.c_char_p, sz]),
        "bws_gpu_set_device_count": (i32, [i32]),
        "bws_gpu_set_devices": (i32, [ctypes.POINTER(i32), i32]),
        "bws_gpu_device_count": (i32, []),
        "bws_gpu_shutdown": (None, []),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

#: every symbol include/bitsort/*.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "bws_version", "bws_last_error", "bws_algorithm_name", "bws_algorithm_from_name",
    "bws_sort", "bws_sort_u32_range", "bws_gpu_sort_device_async", "bws_gpu_sort_check",
    "bws_gpu_sort_range_device_async", "bws_gpu_range_split",
    "bws_gpu_bitset_or_gather", "bws_gpu_bitset_scan_sources", "bws_gpu_bitset_push", "bws_gpu_ipc_get_handle", "bws_gpu_ipc_open", "bws_gpu_ipc_close",
    "bws_gpu_bitset_build", "bws_gpu_bitset_scan", "bws_gpu_set_scatter_mode", "bws_gpu_set_path",
    "bws_gpu_launch_count",
    "bws_gpu_set_kernel_timing", "bws_gpu_kernel_timings",
    "bws_gpu_set_device_count", "bws_gpu_set_devices", "bws_gpu_device_count",
    "bws_gpu_shutdown",
)


def _check(status: int) -> None:
    if status != Status.OK:
        raise BitsortError(status, last_error())


def version() -> str:
    return lib.bws_version().decode()


def last_error() -> str:
    return lib.bws_last_error().decode()


def algorithm_name(algorithm: int) -> str:
    return lib.bws_algorithm_name(int(algorithm)).decode()


def algorithm_from_name(name: str) -> Algorithm:
    out = ctypes.c_int(-1)
    _check(lib.bws_algorithm_from_name(name.encode(), ctypes.byref(out)))
    return Algorithm(out.value)


def sort_raw(ptr: Optional[int], count: int, width: int = 32, is_unsigned: int = 1,
             algorithm: int = Algorithm.BITWISE) -> int:
    """The bare ABI call: returns the bws_status integer."""
    return lib.bws_sort(ptr, count, width, is_unsigned, int(algorithm))


def _ptr_count(data) -> tuple[int, int]:
    if isinstance(data, np.ndarray):
        if data.dtype != np.uint32 or not data.flags.c_contiguous:
            raise TypeError("expected a C-contiguous uint32 numpy array")
        return data.ctypes.data, data.size
    # torch tensor (host or CUDA)
    if str(data.dtype) not in ("torch.uint32", "torch.int32"):
        raise TypeError("expected a uint32/int32 torch tensor")
    if not data.is_contiguous():
        raise TypeError("expected a contiguous tensor")
    return data.data_ptr(), data.numel()


def sort(data, algorithm: int = Algorithm.BITWISE) -> None:
    """In-place bws_sort(data, n, 32, 1, algorithm) of a uint32 array/tensor
    (host numpy, pinned or pageable host tensor, or CUDA tensor)."""
    ptr, n = _ptr_count(data)
    _check(sort_raw(ptr, n, 32, 1, algorithm))


def sort_u32_range(data, key_range: int) -> None:
    ptr, n = _ptr_count(data)
    _check(lib.bws_sort_u32_range(ptr, n, key_range))


def sort_device_async(keys_ptr: int, count: int, out_ptr: int, key_range: int, stream: int = 0) -> None:
    _check(lib.bws_gpu_sort_device_async(keys_ptr, count, out_ptr, key_range, stream or None))


def sort_range_device_async(keys_ptr: int, count: int, out_ptr: int, key_lo: int, key_range: int,
                            stream: int = 0) -> None:
    """Device sort of keys in [key_lo, key_lo + key_range); check with sort_check."""
    _check(lib.bws_gpu_sort_range_device_async(keys_ptr, count, out_ptr, key_lo, key_range, stream or None))


def range_split(keys_ptr: int, count: int, key_range: int, parts: int, out_ptr: int, counts_ptr: int,
                stream: int = 0) -> int:
    """Groups device keys by part (part p = keys in [p*W, (p+1)*W)); writes uint32
    counts per part to the device array at counts_ptr; returns W."""
    w = ctypes.c_uint64(0)
    _check(lib.bws_gpu_range_split(keys_ptr, count, key_range, parts, out_ptr, counts_ptr,
                                   ctypes.byref(w), stream or None))
    return int(w.value)


def sort_check(stream: int = 0) -> int:
    out = ctypes.c_uint64(0)
    _check(lib.bws_gpu_sort_check(stream or None, ctypes.byref(out)))
    return out.value


def bitset_build(keys_ptr: int, count: int, bits_ptr: int, key_range: int, stream: int = 0) -> None:
    _check(lib.bws_gpu_bitset_build(keys_ptr, count, bits_ptr, key_range, stream or None))


def bitset_scan(bits_ptr: int, n_words: int, key_base: int, out_ptr: int, out_capacity: int,
                d_total_ptr: int, stream: int = 0) -> None:
    _check(lib.bws_gpu_bitset_scan(bits_ptr, n_words, key_base, out_ptr, out_capacity,
                                   d_total_ptr, stream or None))


IPC_HANDLE_BYTES = 64


def bitset_or_gather(src_ptrs, n_words: int, dst_ptr: int, stream: int = 0) -> None:
    """dst[i] = OR of src[i] over the (local or peer) device pointers src_ptrs."""
    arr = (ctypes.c_void_p * len(src_ptrs))(*src_ptrs)
    _check(lib.bws_gpu_bitset_or_gather(arr, len(src_ptrs), n_words, dst_ptr, stream or None))


def bitset_scan_sources(src_ptrs, n_words: int, key_base: int, out_ptr: int, out_capacity: int,
                        d_total_ptr: int, stream: int = 0) -> None:
    """bitset_scan of the OR of the (local or peer) slices src_ptrs, fused in
    one kernel (bws_gpu_bitset_scan_sources)."""
    arr = (ctypes.c_void_p * len(src_ptrs))(*src_ptrs)
    _check(lib.bws_gpu_bitset_scan_sources(arr, len(src_ptrs), n_words, key_base, out_ptr,
                                           out_capacity, d_total_ptr, stream or None))


def bitset_push(keys_ptr: int, count: int, key_range: int, slice_ptrs, slice_words: int, stream: int = 0) -> None:
    """OR the bitset of the keys into the owners' slices (bws_gpu_bitset_push)."""
    arr = (ctypes.c_void_p * len(slice_ptrs))(*slice_ptrs)
    _check(lib.bws_gpu_bitset_push(keys_ptr, count, key_range, arr, len(slice_ptrs), slice_words, stream or None))


def ipc_get_handle(dev_ptr: int) -> tuple[bytes, int]:
    """(handle of dev_ptr's allocation, dev_ptr's offset in it)."""
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    off = ctypes.c_uint64(0)
    _check(lib.bws_gpu_ipc_get_handle(dev_ptr, buf, ctypes.byref(off)))
    return buf.raw, int(off.value)


def ipc_open(handle: bytes) -> int:
    out = ctypes.c_void_p(0)
    _check(lib.bws_gpu_ipc_open(ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES), ctypes.byref(out)))
    return int(out.value)


def ipc_close(dev_ptr: int) -> None:
    _check(lib.bws_gpu_ipc_close(dev_ptr))


def set_scatter_mode(mode: int) -> None:
    _check(lib.bws_gpu_set_scatter_mode(int(mode)))


def set_path(path: int) -> None:
    _check(lib.bws_gpu_set_path(int(path)))


def launch_count() -> int:
    return lib.bws_gpu_launch_count()


def set_kernel_timing(enable: bool) -> None:
    _check(lib.bws_gpu_set_kernel_timing(int(enable)))


def kernel_timings() -> dict[str, tuple[int, float]]:
    """{kernel: (launches, total_ms)} since the previous call (synchronises)."""
    buf = ctypes.create_string_buffer(1 << 14)
    _check(lib.bws_gpu_kernel_timings(buf, len(buf)))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


def set_device_count(count: int) -> None:
    """Multi-GPU bws_sort on devices 0 .. count-1 (1 = single GPU)."""
    _check(lib.bws_gpu_set_device_count(int(count)))


def set_devices(devices) -> None:
    """Multi-GPU bws_sort on an explicit device list (a device may repeat:
    logical ranks sharing a GPU)."""
    arr = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
    _check(lib.bws_gpu_set_devices(arr, len(devices)))


def device_count() -> int:
    return int(lib.bws_gpu_device_count())


def shutdown() -> None:
    lib.bws_gpu_shutdown()
