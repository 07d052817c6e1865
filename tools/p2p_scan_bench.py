"""Fused exchange + scan vs OR-gather then scan, on one GPU (development tool).

Emulates rank 0 of a G-rank p2p sort (dist.distributed_sort_p2p): G full
bitsets of disjoint random key shards sit in this GPU's memory (on a real node
G-1 of them are peers' bitsets read over NVLink through CUDA IPC). Times, with
CUDA events on the launching stream and L2 flushed before each launch:
  two_kernel: bws_gpu_bitset_or_gather (slice written to HBM) + bws_gpu_bitset_scan
  fused:      bws_gpu_bitset_scan_sources (peers' words ORed in the scan's SMEM tiles)
and checks that both produce the same keys. Local sources make this an HBM
measurement; on NVLink the peer reads are bounded by ~900 GB/s per direction.
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
from paper_1312_0138_b200.dist import CudaRankOps, slice_words  # noqa: E402


def timed(fn, flush, iters):
    ts = []
    s = torch.cuda.current_stream()
    for _ in range(iters):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts)), float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--key-range-log2", type=int, default=30)
    ap.add_argument("--density", type=float, default=1.0)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    G, M = args.world, 1 << args.key_range_log2
    words, per = slice_words(M, G)
    gen = torch.Generator(device="cuda").manual_seed(42)
    # disjoint shards: every key of the range present with probability density,
    # owned by a random rank
    bitsets = [torch.zeros(words, dtype=torch.int32, device="cuda") for _ in range(G)]
    chunk = 1 << 26
    for lo in range(0, M, chunk):
        k = torch.arange(lo, min(M, lo + chunk), device="cuda", dtype=torch.int64)
        keep = torch.rand(k.numel(), device="cuda", generator=gen) < args.density
        k = k[keep]
        owner = torch.randint(0, G, (k.numel(),), device="cuda", generator=gen)
        for r in range(G):
            kr = k[owner == r]
            w = (kr >> 5)
            v = torch.ones_like(kr) << (kr & 31)
            acc = torch.zeros(words, dtype=torch.int64, device="cuda")
            acc.index_add_(0, w, v)  # disjoint bits: sum == or
            bitsets[r] |= torch.where(acc >= 1 << 31, acc - (1 << 32), acc).to(torch.int32)
    ops = CudaRankOps()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    rank = 0
    cap = per * 32
    slice_buf = torch.empty(per, dtype=torch.int32, device="cuda")
    out_a = torch.empty(cap, dtype=torch.int32, device="cuda")
    out_b = torch.empty(cap, dtype=torch.int32, device="cuda")
    tot_a = torch.zeros(1, dtype=torch.int64, device="cuda")
    tot_b = torch.zeros(1, dtype=torch.int64, device="cuda")
    ptrs = [b.data_ptr() + 4 * rank * per for b in bitsets]
    stream = torch.cuda.current_stream().cuda_stream

    def two_kernel():
        capi.bitset_or_gather(ptrs, per, slice_buf.data_ptr(), stream)
        capi.bitset_scan(slice_buf.data_ptr(), per, rank * per * 32, out_a.data_ptr(), cap, tot_a.data_ptr(), stream)

    def fused():
        capi.bitset_scan_sources(ptrs, per, rank * per * 32, out_b.data_ptr(), cap, tot_b.data_ptr(), stream)

    for f in (two_kernel, fused):
        f()
    torch.cuda.synchronize()
    n = int(tot_a.item())
    assert n == int(tot_b.item()) and torch.equal(out_a[:n], out_b[:n]), "fused != two-kernel"
    ta = timed(two_kernel, flush, args.iters)
    tb = timed(fused, flush, args.iters)
    src_bytes = G * per * 4
    print(json.dumps({"world": G, "key_range": M, "density": args.density, "slice_words": per, "keys": n,
                      "two_kernel_us": round(ta[0] * 1e6, 1), "fused_us": round(tb[0] * 1e6, 1),
                      "fused_source_GBps": round(src_bytes / tb[0] / 1e9, 1),
                      "fused_alg_GBps": round((src_bytes + 4 * n) / tb[0] / 1e9, 1)}))


if __name__ == "__main__":
    main()
