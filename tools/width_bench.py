"""Throughput of bws_sort's non-headline paths on one GPU (development tool):
repeated 32-bit keys (bitset pass + counting pass), 8/16-bit keys (counting
sort), 64-bit keys narrowed to the 32-bit path (span < 2^32) and the 64-bit
LSD radix sort (full span). Device-resident arrays, the synchronous
bws_sort call timed with CUDA events (median of --iters), fresh copy of the
input before every call (outside the events), one JSON line per case.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_0138_b200 import capi  # noqa: E402

WIDTH = {np.dtype(np.uint8): 8, np.dtype(np.uint16): 16, np.dtype(np.uint32): 32, np.dtype(np.uint64): 64,
         np.dtype(np.int64): 64, np.dtype(np.int16): 16}


SELECT: list[str] = []


def case(name, keys: np.ndarray, iters: int):
    if SELECT and not any(x in name for x in SELECT):
        return
    src = torch.from_numpy(keys.view(np.uint8).copy()).cuda()
    work = torch.empty_like(src)
    w = WIDTH[keys.dtype]
    uns = int(keys.dtype.kind == "u")
    ts = []
    for _ in range(iters + 1):
        work.copy_(src)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st = capi.sort_raw(work.data_ptr(), keys.size, w, uns, 0)
        b.record()
        b.synchronize()
        assert st == capi.Status.OK, capi.last_error()
        ts.append(a.elapsed_time(b) * 1e-3)
    got = work.cpu().numpy().view(keys.dtype)
    assert np.array_equal(got[:: max(1, keys.size // 4096)], np.sort(keys)[:: max(1, keys.size // 4096)])
    t = float(np.median(ts[1:]))
    print(json.dumps({"case": name, "n": int(keys.size), "width": w, "ms": round(t * 1e3, 3),
                      "Gkeys_s": round(keys.size / t / 1e9, 2),
                      "GBps_key_bytes": round(2 * keys.nbytes / t / 1e9, 1)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=26)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--cases", default="", help="comma-separated case-name substrings (default: all)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    SELECT.extend(x for x in a.cases.split(",") if x)
    n = 1 << a.log2n
    rng = np.random.default_rng(42)
    case("u32_repeats_range_2^24", rng.integers(0, 1 << 24, size=n, dtype=np.uint32), a.iters)
    case("u32_distinct_reference_point", rng.choice(1 << 28, size=n, replace=False).astype(np.uint32), a.iters)
    case("u8_uniform", rng.integers(0, 256, size=n, dtype=np.uint8), a.iters)
    case("u16_uniform", rng.integers(0, 1 << 16, size=n, dtype=np.uint16), a.iters)
    case("i16_constant", np.full(n, -5, dtype=np.int16), a.iters)
    case("u64_span_2^30", (np.uint64(1 << 50) + rng.integers(0, 1 << 30, size=n).astype(np.uint64)), a.iters)
    case("u64_full_range", rng.integers(0, np.iinfo(np.uint64).max, size=n, dtype=np.uint64, endpoint=True),
         a.iters)
    case("i64_full_range", rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, size=n, dtype=np.int64,
                                        endpoint=True), a.iters)


if __name__ == "__main__":
    main()
