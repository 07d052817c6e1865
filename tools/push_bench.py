"""Push build (bws_gpu_bitset_push) vs full-bitset build (bws_gpu_bitset_build)
for one rank's shard, on one GPU (development tool).

Emulates rank 0 of a G-rank sort: its shard (n/G keys of the config) is built
either into a full local bitset (the reduce-scatter variant's step 1; the NCCL
reduce-scatter would follow) or pushed bucket by bucket into G slice buffers
(the push variant: build and exchange in one kernel; here all slices are
local, on a node G-1 of them are peers' memory over NVLink). CUDA events on
the launching stream, median of --iters, L2 flushed before each launch.
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
from paper_1312_0138_b200.configs import CONFIGS  # noqa: E402
from paper_1312_0138_b200.dist import push_slice_words, shard_bounds  # noqa: E402


def timed(fn, flush, iters):
    ts = []
    s = torch.cuda.current_stream()
    for _ in range(iters + 1):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts[1:]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C5")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    flush = torch.empty(1 << 26, dtype=torch.int32, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    for name in a.configs.split(","):
        cfg = CONFIGS[name]
        keys = cfg.generate()
        lo, hi = shard_bounds(cfg.n, 0, a.world)
        shard = torch.from_numpy(keys[lo:hi].view(np.int32)).cuda()
        del keys
        M = cfg.key_range
        words = (M + 31) // 32
        full = torch.empty(words, dtype=torch.int32, device="cuda")
        per = push_slice_words(M, a.world)
        slices = torch.zeros(per * a.world, dtype=torch.int32, device="cuda")
        ptrs = [slices.data_ptr() + 4 * r * per for r in range(a.world)]

        def build():
            capi.bitset_build(shard.data_ptr(), shard.numel(), full.data_ptr(), M, sp)

        def push():
            slices.zero_()
            capi.bitset_push(shard.data_ptr(), shard.numel(), M, ptrs, per, sp)

        def zero_only():
            slices.zero_()

        t_build = timed(build, flush, a.iters)
        t_zero = timed(zero_only, flush, a.iters)
        t_push = timed(push, flush, a.iters)
        torch.cuda.synchronize()
        assert torch.equal(slices[:words], full), "push != build"
        print(json.dumps({"config": name, "world": a.world, "shard_keys": int(shard.numel()), "key_range": M,
                          "build_full_bitset_us": round(t_build * 1e6, 1),
                          "push_us_incl_slice_zeroing": round(t_push * 1e6, 1),
                          "slice_zeroing_us": round(t_zero * 1e6, 1)}), flush=True)
        del full, slices, shard
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
