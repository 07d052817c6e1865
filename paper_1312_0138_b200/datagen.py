"""Seeded synthetic inputs (ctypes over lib/libbws_datagen.so, csrc/datagen.c).

Recipes follow SURVEY.md Appendix A with the reference's splitmix64
(/root/reference/proj/src/generator.hpp:21-30); see csrc/datagen.c.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import LIB_DIR

_LIB_PATH = LIB_DIR / "libbws_datagen.so"
if not _LIB_PATH.exists():
    raise ImportError(f"{_LIB_PATH} is not built; run __graft_entry__.build()")
_lib = ctypes.CDLL(str(_LIB_PATH))
_u64, _vp = ctypes.c_uint64, ctypes.c_void_p
_lib.bws_gen_fnv1a64.restype = _u64
_lib.bws_gen_fnv1a64.argtypes = [_vp, ctypes.c_size_t]
for _name, _args in {
    "bws_gen_shuffle_prefix": [_vp, _u64, _u64, _u64],
    "bws_gen_permutation": [_vp, _u64, _u64],
    "bws_gen_dedup_draws": [_vp, _u64, _u64],
    "bws_gen_clustered": [_vp, _u64, ctypes.c_uint32, ctypes.c_double, _u64, _u64, _vp],
    "bws_gen_cluster_sizes": [_vp, _vp, ctypes.c_uint32, _u64, ctypes.c_double],
}.items():
    getattr(_lib, _name).restype = ctypes.c_int
    getattr(_lib, _name).argtypes = _args


def _rc(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what} failed with code {rc}")


def _empty(n: int, out: np.ndarray | None) -> np.ndarray:
    if out is None:
        return np.empty(n, dtype=np.uint32)
    if out.dtype != np.uint32 or out.size < n or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous uint32 array of at least n elements")
    return out[:n]


def fnv1a64(arr: np.ndarray) -> str:
    """FNV-1a 64 over the array's little-endian bytes, as 16 hex digits."""
    a = np.ascontiguousarray(arr)
    return f"{_lib.bws_gen_fnv1a64(a.ctypes.data, a.nbytes):016x}"


def shuffle_prefix(n: int, key_range: int, seed: int = 42, out=None) -> np.ndarray:
    """C1/C2: first n of a forward Fisher-Yates shuffle of [0, key_range)."""
    o = _empty(n, out)
    _rc(_lib.bws_gen_shuffle_prefix(o.ctypes.data, n, key_range, seed), "shuffle_prefix")
    return o


def permutation(n: int, seed: int = 42, out=None) -> np.ndarray:
    """C3: seeded Feistel permutation of [0, n)."""
    o = _empty(n, out)
    _rc(_lib.bws_gen_permutation(o.ctypes.data, n, seed), "permutation")
    return o


def dedup_draws(n: int, seed: int = 42, out=None) -> np.ndarray:
    """C4: n distinct uint32 splitmix64 draws, draw order."""
    o = _empty(n, out)
    _rc(_lib.bws_gen_dedup_draws(o.ctypes.data, n, seed), "dedup_draws")
    return o


def clustered(n: int, clusters: int = 4096, zipf_s: float = 1.2, half_window: int = 1 << 18,
              seed: int = 42, out=None, return_centres: bool = False):
    """C5: clustered Zipf keys (see csrc/datagen.c for the pinned rule)."""
    o = _empty(n, out)
    centres = np.empty(clusters, dtype=np.uint32)
    _rc(_lib.bws_gen_clustered(o.ctypes.data, n, clusters, zipf_s, half_window, seed,
                               centres.ctypes.data), "clustered")
    return (o, centres) if return_centres else o


def cluster_sizes(caps: np.ndarray, n: int, zipf_s: float = 1.2) -> np.ndarray:
    caps = np.ascontiguousarray(caps, dtype=np.uint64)
    sizes = np.empty_like(caps)
    _rc(_lib.bws_gen_cluster_sizes(sizes.ctypes.data, caps.ctypes.data, caps.size, n, zipf_s),
        "cluster_sizes")
    return sizes
