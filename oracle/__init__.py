"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package; the product path never does.
``ORACLE`` is the plain-C restatement (bitsort_oracle.c); ``REFERENCE`` is the
reference's own C ABI compiled from /root/reference by oracle/Makefile into
oracle/_ref/ (None when that build is absent).
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_PATH = HERE / "build" / "liboracle.so"
REFERENCE_PATH = HERE / "_ref" / "libbitsort_ref.so"


def _load_oracle():
    if not ORACLE_PATH.exists():
        raise ImportError(f"{ORACLE_PATH} missing; run `make -C oracle`")
    lib = ctypes.CDLL(str(ORACLE_PATH))
    vp, sz, u64, u32, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
    for w in ("u8", "u16", "u32", "u64", "s8", "s16", "s32", "s64"):
        f = getattr(lib, f"oracle_bitwise_sort_{w}")
        f.restype, f.argtypes = i32, [vp, sz, i32]
    lib.oracle_splitmix64_next.restype, lib.oracle_splitmix64_next.argtypes = u64, [ctypes.POINTER(u64)]
    lib.oracle_mix64.restype, lib.oracle_mix64.argtypes = u64, [u64, u64]
    lib.oracle_generate_uniform_u32.restype, lib.oracle_generate_uniform_u32.argtypes = None, [vp, sz, u64, u32]
    lib.oracle_fnv1a64.restype, lib.oracle_fnv1a64.argtypes = u64, [vp, sz]
    lib.oracle_bitset_build.restype, lib.oracle_bitset_build.argtypes = u64, [vp, sz, vp, u64]
    lib.oracle_bitset_scan.restype, lib.oracle_bitset_scan.argtypes = u64, [vp, u64, u32, vp, u64]
    return lib


def _load_reference():
    if not REFERENCE_PATH.exists():
        return None
    lib = ctypes.CDLL(str(REFERENCE_PATH))
    lib.bws_sort.restype = ctypes.c_int
    lib.bws_sort.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_int, ctypes.c_int]
    lib.bws_last_error.restype = ctypes.c_char_p
    lib.bws_version.restype = ctypes.c_char_p
    return lib


ORACLE = _load_oracle()
REFERENCE = _load_reference()

_DT = {np.dtype(np.uint8): "u8", np.dtype(np.uint16): "u16", np.dtype(np.uint32): "u32", np.dtype(np.uint64): "u64",
       np.dtype(np.int8): "s8", np.dtype(np.int16): "s16", np.dtype(np.int32): "s32", np.dtype(np.int64): "s64"}


def bitwise_sort(a: np.ndarray, skip_empty_bits: bool = False) -> np.ndarray:
    """Sorted copy via the C restatement of bitsort.hpp:84-151 (unsigned, or
    signed with the reference's sign split)."""
    out = np.ascontiguousarray(a).copy()
    rc = getattr(ORACLE, f"oracle_bitwise_sort_{_DT[out.dtype]}")(out.ctypes.data, out.size, int(skip_empty_bits))
    if rc != 0:
        raise MemoryError("oracle scratch allocation failed")
    return out


def reference_sort_u32(a: np.ndarray) -> np.ndarray:
    """Sorted copy via the reference's own bws_sort(…, 32, 1, BWS_ALG_BITWISE)."""
    if REFERENCE is None:
        raise RuntimeError("oracle/_ref/libbitsort_ref.so not built")
    out = np.ascontiguousarray(a, dtype=np.uint32).copy()
    rc = REFERENCE.bws_sort(out.ctypes.data, out.size, 32, 1, 0)
    if rc != 0:
        raise RuntimeError(f"reference bws_sort failed: {REFERENCE.bws_last_error().decode()}")
    return out


def generate_uniform_u32(n: int, seed: int, trial: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    ORACLE.oracle_generate_uniform_u32(out.ctypes.data, n, seed, trial)
    return out


def fnv1a64(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return f"{ORACLE.oracle_fnv1a64(a.ctypes.data, a.nbytes):016x}"


def bitset_build(keys: np.ndarray, key_range: int) -> tuple[np.ndarray, int]:
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    bits = np.empty((key_range + 31) // 32, dtype=np.uint32)
    bad = ORACLE.oracle_bitset_build(keys.ctypes.data, keys.size, bits.ctypes.data, key_range)
    return bits, bad


def bitset_scan(bits: np.ndarray, key_base: int = 0, capacity: int | None = None) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint32)
    cap = capacity if capacity is not None else int(np.unpackbits(bits.view(np.uint8)).sum())
    out = np.empty(cap, dtype=np.uint32)
    cnt = ORACLE.oracle_bitset_scan(bits.ctypes.data, bits.size, key_base, out.ctypes.data, cap)
    return out[: min(cnt, cap)]
