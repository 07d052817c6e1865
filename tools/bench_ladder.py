"""GPU records in the reference benchmark's CSV schema, plus its slope fit
(SURVEY.md §8(f) f3).

The reference harness (proj/src/bench.cpp:128-160 run_bench) times one
in-place sort per (algorithm, width, n, trial) with steady_clock and writes
`algorithm,width,n,seed,trial,elapsed_ns,ns_per_element` (records_csv,
bench.cpp:219-231); fit_scaling (bench.cpp:162-217) fits log(median elapsed)
against log(n) per algorithm. This tool does the same for the B200 library:

  bitwise         bws_sort(host array, n, 32, 1, BWS_ALG_BITWISE) — the drop-in
                  call, host->device->host included (steady wall clock)
  bitwise_device  the device-resident sort of the same keys
                  (bws_gpu_sort_device_async with the range hint), CUDA events

Inputs: distinct keys, the first n of a seed-42 splitmix64 Fisher-Yates shuffle
of [0, 4n) (the C2 density; the reference's generate_input never yields
distinct keys). The slope is a secondary check of the
O(n + M) behaviour: with M = 4n it should be close to 1 once launch latency
stops dominating.

usage: python tools/bench_ladder.py [--sizes 65536,...] [--trials 5] [--out PREFIX]
"""
from __future__ import annotations

import argparse
import math
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

DEFAULT_SIZES = [1 << k for k in range(16, 27, 2)]


def measured_hbm_gbs() -> float:
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else the profiling recipe's fallback."""
    from paper_1312_0138_b200.configs import hbm_peak

    return hbm_peak()[0]


class ConfigError(ValueError):
    """bench.cpp's config_error (a slope fit over fewer than 4 sizes)."""


def fit_scaling(records):
    """bench.cpp:162-217: per algorithm (first-seen order), median elapsed per n
    (mean of the middle two for an even trial count), least squares of
    log(median) on log(n); [(algorithm, slope, RMS residual in log space,
    [(n, median), ...])]. Fewer than 4 distinct sizes -> ConfigError."""
    out = []
    for alg in dict.fromkeys(r[0] for r in records):
        by_n = {}
        for r in records:
            if r[0] == alg:
                by_n.setdefault(r[2], []).append(r[5])
        if len(by_n) < 4:
            raise ConfigError(f"slope fit needs at least 4 distinct sizes for algorithm '{alg}', "
                              f"got {len(by_n)}")
        pts = [(n, float(statistics.median(v))) for n, v in sorted(by_n.items())]
        xs = [math.log(n) for n, _ in pts]
        ys = [math.log(t) for _, t in pts]
        mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
        sxx = sum((x - mx) ** 2 for x in xs)
        slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
        icpt = my - slope * mx
        resid = math.sqrt(sum((y - (icpt + slope * x)) ** 2 for x, y in zip(xs, ys)) / len(xs))
        out.append((alg, slope, resid, pts))
    return out


def records_csv(records) -> str:
    """bench.cpp:219-231: the reference's seven-column records CSV."""
    return "algorithm,width,n,seed,trial,elapsed_ns,ns_per_element\n" + "".join(
        f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]},{r[5]},{r[6]:.3f}\n" for r in records)


def reports_csv(reports) -> str:
    """bench.cpp reports_csv: algorithm,slope,residual with 6 decimals."""
    return "algorithm,slope,residual\n" + "".join(f"{alg},{s:.6f},{e:.6f}\n" for alg, s, e, _ in reports)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default=",".join(map(str, DEFAULT_SIZES)))
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "ladder"))
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_1312_0138_b200 import capi, datagen

    sizes = [int(s) for s in a.sizes.split(",")]
    if len(sizes) < 4:
        raise SystemExit("slope fit needs at least 4 sizes (bench.cpp:117-124)")
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    records = []
    for n in sizes:
        m = 4 * n
        keys = datagen.shuffle_prefix(n, m, a.seed)
        pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
        host = pinned.numpy().view(np.uint32)
        kd = torch.from_numpy(keys.view(np.int32)).to(dev)
        od = torch.empty_like(kd)
        # warm-up (allocations, first-touch) outside the records
        np.copyto(host, keys)
        capi.sort(host)
        capi.sort_device_async(kd.data_ptr(), n, od.data_ptr(), m, stream.cuda_stream)
        capi.sort_check(stream.cuda_stream)
        expected = np.sort(keys)
        for trial in range(a.trials):
            np.copyto(host, keys)
            t0 = time.perf_counter_ns()
            capi.sort(host)
            ns = max(1, time.perf_counter_ns() - t0)
            assert np.array_equal(host, expected), "unsorted output"  # check_sorted_output
            records.append(("bitwise", 32, n, a.seed, trial, ns, ns / n))
        for trial in range(a.trials):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(stream)
            capi.sort_device_async(kd.data_ptr(), n, od.data_ptr(), m, stream.cuda_stream)
            e1.record(stream)
            assert capi.sort_check(stream.cuda_stream) == n
            ns = max(1, int(e0.elapsed_time(e1) * 1e6))
            records.append(("bitwise_device", 32, n, a.seed, trial, ns, ns / n))
        assert np.array_equal(od.cpu().numpy().view(np.uint32), expected)
    # the reference's seven columns first (bench.cpp:220), then the GPU
    # extension of SURVEY.md §5: gpus, config, algorithmic bytes 8n + M/4,
    # achieved GB/s and its fraction of the measured / nominal HBM peak
    peak = measured_hbm_gbs()
    rows = []
    for r in records:
        n = r[2]
        alg_bytes = 8 * n + (4 * n) // 4
        gbps = alg_bytes / r[5]  # bytes per ns == GB/s
        rows.append(f"{r[0]},{r[1]},{n},{r[3]},{r[4]},{r[5]},{r[6]:.3f},1,n={n};M={4 * n},{alg_bytes},"
                    f"{gbps:.1f},{gbps / peak:.4f},{gbps / 8000.0:.4f}\n")
    rec_csv = ("algorithm,width,n,seed,trial,elapsed_ns,ns_per_element,"  # records_csv's 7 + GPU columns
               "gpus,config,alg_bytes,gbps,roofline_frac_meas,roofline_frac_8tbs\n" + "".join(rows))
    fits = fit_scaling(records)
    slope_csv = reports_csv(fits)
    Path(a.out + "_records.csv").parent.mkdir(parents=True, exist_ok=True)
    Path(a.out + "_records.csv").write_text(rec_csv)
    Path(a.out + "_slopes.csv").write_text(slope_csv)
    print(slope_csv)
    for alg, s, e, pts in fits:
        print(alg, " ".join(f"{n}:{t / n:.3f}ns/key" for n, t in pts))


if __name__ == "__main__":
    main()
