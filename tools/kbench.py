"""Per-phase timing of the bitset sort on one GPU (development tool).

For each config: K1+K2 (bitset_build on a caller buffer), K3 (bitset_scan, no
clear), and the full device-resident sort (sort_device_async: K2 + K3-with-
clear on the cached bitset). CUDA events on the launching stream, median of
--iters, L2 flushed (256 MiB write) before every timed launch.
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
from paper_1312_0138_b200.configs import CONFIGS, hbm_peak  # noqa: E402


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
    ap.add_argument("--configs", default="C1,C2,C4")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--modes", default="AUTO")
    ap.add_argument("--paths", default="DIRECT,BUCKETED")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    flush = torch.empty(1 << 26, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for name in args.configs.split(","):
        cfg = CONFIGS[name]
        keys_h = cfg.generate()
        keys = torch.from_numpy(keys_h.view(np.int32)).cuda()
        out = torch.empty_like(keys)
        words = (cfg.key_range + 31) // 32
        bits = torch.empty(words, dtype=torch.int32, device="cuda")
        total = torch.zeros(1, dtype=torch.int64, device="cuda")
        for mode, path in [(m, p) for p in args.paths.split(",") for m in args.modes.split(",")]:
            capi.set_scatter_mode(getattr(capi.ScatterMode, mode))
            capi.set_path(getattr(capi.Path, path))
            build = lambda: capi.bitset_build(keys.data_ptr(), cfg.n, bits.data_ptr(), cfg.key_range, stream)
            scan = lambda: capi.bitset_scan(bits.data_ptr(), words, 0, out.data_ptr(), cfg.n, total.data_ptr(), stream)
            full = lambda: capi.sort_device_async(keys.data_ptr(), cfg.n, out.data_ptr(), cfg.key_range, stream)
            for f in (build, scan, full):
                f()
            torch.cuda.synchronize()
            tb = timed(build, flush, args.iters)
            ts = timed(scan, flush, args.iters)
            tf = timed(full, flush, args.iters)
            ok = capi.sort_check(stream) == cfg.n
            gbs = cfg.alg_bytes / tf[0] / 1e9
            print(json.dumps({"config": name, "mode": mode, "path": path, "n": cfg.n, "M": cfg.key_range,
                              "build_us": round(tb[0] * 1e6, 1), "scan_us": round(ts[0] * 1e6, 1),
                              "sort_us": round(tf[0] * 1e6, 1), "sort_min_us": round(tf[1] * 1e6, 1),
                              "gkeys_s": round(cfg.n / tf[0] / 1e9, 2), "alg_GBps": round(gbs, 1),
                              "frac_meas": round(gbs / hbm_peak()[0], 3), "ok": ok}), flush=True)
        del keys, out, bits


if __name__ == "__main__":
    main()
