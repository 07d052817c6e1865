"""Small sorts that launch every kernel of the library once or more, each
checked against numpy. Plain runs work everywhere; where compute-sanitizer is
allowed (it is closed on this build's GPU pool) the same driver serves:

  compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py --quick
  compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Each case checks its result against numpy, so a run that exits 0 with
"ERROR SUMMARY: 0 errors" is both race/bounds clean and correct.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_0138_b200 import capi  # noqa: E402
from paper_1312_0138_b200.dist import CudaRankOps, push_slice_words, shard_bounds, slice_words  # noqa: E402


def check_sort(keys: np.ndarray, width: int = 32, is_unsigned: int = 1, device: bool = True, tag: str = ""):
    expected = np.sort(keys)
    if device:
        t = torch.from_numpy(keys.view(np.uint8).copy()).cuda()
        st = capi.sort_raw(t.data_ptr(), keys.size, width, is_unsigned, 0)
        got = t.cpu().numpy().view(keys.dtype)
    else:
        got = keys.copy()
        st = capi.sort_raw(got.ctypes.data, got.size, width, is_unsigned, 0)
    assert st == capi.Status.OK, (tag, capi.last_error())
    assert np.array_equal(got, expected), tag
    print("ok", tag, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="smaller inputs (racecheck is ~100x slower)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(5)
    big = 1 << (19 if a.quick else 21)

    # direct path: K2 scatter (every mode) + K3 scan
    capi.set_path(capi.Path.DIRECT)
    for mode in (capi.ScatterMode.AUTO, capi.ScatterMode.PLAIN, capi.ScatterMode.WARP_AGG, capi.ScatterMode.SMEM):
        capi.set_scatter_mode(mode)
        check_sort(rng.choice(1 << 20, size=30_001, replace=False).astype(np.uint32), tag=f"direct mode {int(mode)}")
    capi.set_scatter_mode(capi.ScatterMode.AUTO)
    capi.set_path(capi.Path.BUCKETED)
    # slab layout, bulk-store KB3 (<= 512 buckets) and in-place KB3 (1024 buckets), KB4
    check_sort(rng.choice(1 << 22, size=big, replace=False).astype(np.uint32), tag="slab bulk-store")
    check_sort(rng.choice(1 << 28, size=big, replace=False).astype(np.uint32), device=False, tag="slab 2^28")
    check_sort(rng.permutation(1 << 20).astype(np.uint32) + np.uint32(1 << 29), tag="slab 1024 buckets dense")
    # packed layout (KB1/KB2, KB4 order + L2 hints), sparse KB4
    check_sort(rng.choice(1 << 32, size=big // 4, replace=False).astype(np.uint32), tag="packed sparse")
    # signed, repeats (KB4m), misaligned device pointer
    check_sort(rng.integers(-(1 << 31), 1 << 31, size=big // 2, dtype=np.int64).astype(np.int32), 32, 0,
               tag="signed")
    check_sort(rng.integers(0, 1 << 18, size=big // 2, dtype=np.uint32), tag="repeats")
    # other widths: counting sort, 64-bit narrowing and radix
    check_sort(rng.integers(0, 256, size=100_003, dtype=np.uint8), 8, 1, tag="u8")
    check_sort(rng.integers(-(1 << 15), 1 << 15, size=100_003, dtype=np.int64).astype(np.int16), 16, 0, tag="i16")
    check_sort((rng.integers(0, 1 << 30, size=50_001).astype(np.uint64) + np.uint64(1 << 40)), 64, 1, tag="u64 narrow")
    check_sort(rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, size=50_001, dtype=np.int64), 64, 0,
               tag="i64 radix")
    # multi-GPU building blocks with emulated ranks: bitset build (KB4b), scan,
    # fused scan over sources, push build (KB4p), OR-gather, range split + range sort
    ops = CudaRankOps()
    world, M, n = 3, 1 << 22, big // 2
    keys = rng.choice(M, size=n, replace=False).astype(np.uint32)
    words, per = slice_words(M, world)
    bitsets = []
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        sh = torch.from_numpy(keys[lo:hi].view(np.int32)).cuda()
        bitsets.append(ops.bitset_build(sh, M, words).clone())
    parts = []
    for r in range(world):
        out, cnt = ops.or_scan([bitsets[r]] + [b for q, b in enumerate(bitsets) if q != r], r * per, per,
                               r * per * 32, n)
        parts.append(out[: int(cnt.item())].cpu().numpy().view(np.uint32).copy())
    assert np.array_equal(np.concatenate(parts), np.sort(keys))
    sl = ops.or_gather(bitsets, 0, per)
    assert int(sl.ne(0).sum()) > 0
    print("ok multi-GPU p2p blocks", flush=True)
    pw = push_slice_words(M, world)
    slices = [ops.alloc_slice(pw) for _ in range(world)]
    for r in range(world):
        lo, hi = shard_bounds(n, r, world)
        ops.bitset_push(torch.from_numpy(keys[lo:hi].view(np.int32)).cuda(), M, slices, pw)
    parts = []
    for r in range(world):
        out, cnt = ops.bitset_scan(slices[r], r * pw * 32, n)
        parts.append(out[: int(cnt.item())].cpu().numpy().view(np.uint32).copy())
    assert np.array_equal(np.concatenate(parts), np.sort(keys))
    print("ok multi-GPU push blocks", flush=True)
    grouped, counts, width, ok = ops.range_split(torch.from_numpy(keys.view(np.int32)).cuda(), M, world)
    assert ok
    c = counts.tolist()
    off = 0
    for r in range(world):
        part = grouped[off: off + c[r]]
        srt, ok = ops.sort_range(part, min(r * width, M), max(1, min((r + 1) * width, M) - min(r * width, M)))
        assert ok
        off += c[r]
    print("ok multi-GPU a2a blocks", flush=True)
    capi.set_path(capi.Path.AUTO)
    print("all cases ok")


if __name__ == "__main__":
    main()
