#!/usr/bin/env python
"""Benchmark of the B200 bitset sort (BASELINE.json metric: sorted keys/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one complete sort of the workload's keys (device-resident, timed
with CUDA events on the launching stream, L2 flushed by a 256 MiB write
between steps outside the timed events). N > 1 runs under torchrun, one rank
per GPU: every rank holds an input-position shard, and the step is the full
multi-GPU sort (K1+K2 -> NCCL reduce-scatter -> K3 -> count all-gather),
timed as the max over ranks. The default workload is BASELINE.json configs[1]
(C2). Printed: ONE JSON line (rank 0). See DESIGN.md "Measurement".

--impl reference times the reference's own CPU sort (oracle/_ref, the
unmodified bws_sort compiled from /root/reference; the C restatement in
oracle/ if that library is absent) on bounded samples of the same workload,
on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sorted keys/sec (Gkeys/s) at 1/2/4/8 B200; achieved HBM GB/s fraction of roofline"
UNIT = "Gkeys/s"
NOMINAL_HBM_GBS = 8000.0  # B200 HBM3e nominal (SURVEY.md §8(d) reports both fractions)


# The JSON lines go to the process's original stdout; everything else written
# to fd 1 by native code (e.g. NCCL's "NCCL version ..." banner when NCCL_DEBUG
# is set in the environment) is sent to stderr, so stdout carries exactly the
# result lines the driver parses.
_RESULT_OUT = None


def isolate_stdout() -> None:
    global _RESULT_OUT
    if _RESULT_OUT is None:
        sys.stdout.flush()
        _RESULT_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict) -> None:
    out = _RESULT_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2", help="C1..C5 (BASELINE.json configs[0..4]) or 'all'")
    ap.add_argument("--path", choices=["AUTO", "DIRECT", "BUCKETED", "FUSED"], default="AUTO")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-sample-keys", type=int, default=1 << 25,
                    help="keys in the cpu_baseline sample (about 10 s of reference CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU (NCCL reduce-scatter) path even with one rank")
    ap.add_argument("--a2a", action="store_true",
                    help="multi-GPU key all-to-all variant (range split + NCCL all-to-all + range sort)")
    ap.add_argument("--p2p", action="store_true",
                    help="multi-GPU peer-to-peer variant (the exchange fused into the scan over CUDA IPC)")
    ap.add_argument("--push", action="store_true",
                    help="multi-GPU push variant (the exchange fused into the build: bulk ORs into peers' slices)")
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank plumbing only, on gloo without a GPU (CPU test of the launcher)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def host_info():
    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count()}


def measured_peak():
    from paper_1312_0138_b200.configs import hbm_peak

    return hbm_peak()


# --- per-kernel algorithmic bytes ----------------------
def fused_passes(key_range: int, sms: int = 148) -> int:
    """Passes of the fused KF kernel over the keys (fused.cu plan_fused): one
    when a per-SM slice of ceil(M / SMs) bits (rounded up to 2^17) fits next to
    the producer's ~96 KB of SMEM, else two."""
    per = -(-key_range // sms)
    slice_bits = -(-per // (1 << 17)) * (1 << 17)
    return 1 if slice_bits <= 8 * (1 << 17) else 2


def kernel_alg_bytes(kernel: str, n: int, key_range: int, world: int = 1) -> int:
    words_bytes = (key_range + 31) // 32 * 4
    return {
        "fused_sort": 4 * n * (fused_passes(key_range) + 1),  # read keys once per pass, write sorted keys
        "fused_direct": 8 * n,                # KD: read keys, write sorted keys (the bitset stays in L2)
        "small_sort": 8 * n,                  # KS: read keys, write sorted keys (the bitset stays in L2)
        "bucket_hist": 4 * n,                 # read keys
        "bucket_colscan": 0,
        "bucket_partition": 8 * n,            # read keys, write bucketed keys
        "bucket_sort": 8 * n,                 # read bucketed keys, write sorted keys
        "bucket_bitset": 4 * n + words_bytes,  # read bucketed keys, write the bitset (multi-GPU)
        "bucket_push": 4 * n + words_bytes,    # read bucketed keys, OR the bitset into the slices
        "bitset_scatter": 4 * n + words_bytes,          # read keys, write bitset
        "bitset_scan": words_bytes // world + 4 * n,    # read (slice of) bitset, write keys
        "bitset_scan_sources": words_bytes + 4 * n,     # read the slice of every rank's bitset, write keys
    }.get(kernel, 0)


class ClockSampler(threading.Thread):
    """NVML poll of SM clock and clock-event reasons while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        super().__init__(daemon=True)
        self.samples = []
        self.stop_evt = threading.Event()
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.nv = None

    def run(self):
        while self.ok and not self.stop_evt.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def summary(self, t0: float, t1: float):
        self.stop_evt.set()
        self.join(timeout=1.0)
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "note": "NVML unavailable"}
        win = [s for s in self.samples if t0 <= s[0] <= t1] or self.samples
        mask = 0
        for _, _, r in win:
            mask |= r
        reasons = sorted(name for bit, name in self.REASONS.items() if mask & bit)
        return {"sm_mhz": statistics.median(m for _, m, _ in win), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(win)}


# --- CPU reference --------------------------------------------------------
def reference_sorter():
    """(callable sorting a uint32 array in place, kind, what)."""
    import oracle

    if oracle.REFERENCE is not None:
        lib = oracle.REFERENCE

        def run(a):
            rc = lib.bws_sort(a.ctypes.data, a.size, 32, 1, 0)
            if rc != 0:
                raise RuntimeError(lib.bws_last_error().decode())

        return run, "reference", "oracle/_ref/libbitsort_ref.so bws_sort(…,32,1,BWS_ALG_BITWISE)"

    def run_port(a):
        a[:] = oracle.bitwise_sort(a)

    return run_port, "port", "oracle/bitsort_oracle.c oracle_bitwise_sort_u32 (C restatement)"


def cpu_baseline(keys: np.ndarray, sample: int, workload: str):
    sort, kind, what = reference_sorter()
    s = min(sample, keys.size)
    a = keys[:s].copy()
    t0 = time.perf_counter()
    sort(a)
    dt = time.perf_counter() - t0
    assert np.all(a[1:] > a[:-1]), "reference output not strictly ascending"
    out = {"value": round(s / dt / 1e9, 6), "unit": UNIT, "cores": 1, "kind": kind,
           "sample": f"first {s} keys of {workload} ({what}), 1 call, {dt:.2f} s; "
                     "the reference sort is single-threaded (bitsort.hpp:122-128)",
           **host_info()}
    import oracle

    if oracle.REFERENCE is not None:  # second CPU line: the reference's std::sort arm
        b = keys[:s].copy()
        t0 = time.perf_counter()
        rc = oracle.REFERENCE.bws_sort(b.ctypes.data, b.size, 32, 1, 5)  # BWS_ALG_PLATFORM
        dtp = time.perf_counter() - t0
        if rc == 0 and np.array_equal(a, b):
            out["platform_std_sort"] = {"value": round(s / dtp / 1e9, 6), "unit": UNIT, "cores": 1,
                                        "sample": f"same keys, bws_sort(…,BWS_ALG_PLATFORM), {dtp:.2f} s"}
    return out


def run_reference(args, cfg):
    """The reference's own CPU sort (bws_sort(…,32,1,BWS_ALG_BITWISE) from
    oracle/_ref) on the SAME workload as our arm: every step sorts a fresh copy
    of all cfg.n keys (C2: ~8 s per step on one core). The reference sort is
    single-threaded (bitsort.hpp:122-128), so one host core does the work; the
    copy that restores the unsorted input is outside the timed call, as in
    the reference's own bench (bench.cpp:143-147)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    sort, kind, what = reference_sorter()
    keys = cfg.generate()
    a = np.empty_like(keys)
    for _ in range(args.warmup):
        np.copyto(a, keys)
        sort(a)
    times = []
    for _ in range(args.steps):
        np.copyto(a, keys)
        t0 = time.perf_counter()
        sort(a)
        times.append(time.perf_counter() - t0)
    assert np.all(a[1:] > a[:-1]) and a.size == cfg.n
    ms = 1e3 * sum(times) / len(times)
    value = cfg.n / (ms / 1e3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "key_range": cfg.key_range,
                   "recipe": cfg.recipe, "step_sample_keys": cfg.n},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": 1, "kind": kind,
                         "sample": f"all {cfg.n} keys of {cfg.name} per step ({what}); "
                                   "single-threaded reference (bitsort.hpp:122-128, SPEC.md:216)",
                         **host_info()},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# --- our GPU arm ------------------------------------------------------------
def traffic_from_profiles(workload: str, kernel: str):
    """DRAM bytes (read + write) per launch from the committed ncu summary;
    kernel "step" = the sum over the workload's kernels (one sort)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        per = json.loads(p.read_text()).get(workload, {})
    except ValueError:
        return None
    if kernel == "step":
        return float(sum(per.values())) if per else None
    return per.get(kernel)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1312_0138_b200 import capi

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torchrun")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.dist or args.a2a or args.p2p or args.push
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=dev)
    capi.set_path(getattr(capi.Path, args.path))

    keys_h = cfg.generate()
    n_total, M = cfg.n, cfg.key_range
    if use_dist:
        from paper_1312_0138_b200.dist import CudaRankOps, shard_bounds
        from paper_1312_0138_b200.dist import distributed_sort as dist_rs
        from paper_1312_0138_b200.dist import distributed_sort_a2a as dist_a2a
        from paper_1312_0138_b200.dist import distributed_sort_p2p as dist_p2p
        from paper_1312_0138_b200.dist import distributed_sort_push as dist_push

        distributed_sort = (dist_a2a if args.a2a else dist_p2p if args.p2p else
                            dist_push if args.push else dist_rs)

        lo, hi = shard_bounds(n_total, rank, world)
        shard_h = keys_h[lo:hi]
    else:
        shard_h = keys_h
    keys_d = torch.from_numpy(shard_h.view(np.int32)).to(dev)
    out_d = torch.empty_like(keys_d)
    flush = torch.empty(1 << 26, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    if use_dist:
        ops = CudaRankOps(dev)

        def step():
            return distributed_sort(keys_d, M, n_total=n_total, ops=ops)
    else:
        def step():
            capi.sort_device_async(keys_d.data_ptr(), n_total, out_d.data_ptr(), M, sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if use_dist:
        res = step()
        u = res.keys.to(torch.int64) & 0xFFFFFFFF
        assert res.total == n_total and bool((u[1:] > u[:-1]).all()), "distributed output not ascending"
        if res.count:
            assert int(u[0]) >= res.key_lo and int(u[-1]) < res.key_hi
        del u, res
    else:
        assert capi.sort_check(sp) == n_total
        u = out_d.to(torch.int64) & 0xFFFFFFFF
        assert bool((u[1:] > u[:-1]).all()), "output not strictly ascending"
        del u

    def timed_pass(kernel_timing: bool):
        """K steps bracketed by barrier + synchronize; per-step CUDA events on
        the launching stream. With kernel_timing the library also brackets
        every kernel launch with events (its per-kernel durations feed the
        roofline); that costs ~10 us per step, so `value` comes from a pass
        without it."""
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        capi.set_kernel_timing(kernel_timing)
        capi.kernel_timings()  # drop anything recorded before the timed region
        l0 = capi.launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        ta = time.perf_counter()
        for a, b in evs:
            flush.fill_(1)  # L2 flush, outside the step's events
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize(dev)
        tb = time.perf_counter()
        if use_dist:
            dist.barrier()
        kt = capi.kernel_timings() if kernel_timing else {}
        capi.set_kernel_timing(False)
        if not use_dist:
            assert capi.sort_check(sp) == n_total
        return evs, capi.launch_count() - l0, kt, ta, tb

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.05)
    evs, launches, _, t0, t1 = timed_pass(False)
    clocks = sampler.summary(t0, t1)
    evs_k, _, ktimes, _, _ = timed_pass(True)
    total_ms_k = sum(a.elapsed_time(b) for a, b in evs_k)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if use_dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        ts = torch.tensor(step_ms, dtype=torch.float64, device=dev)
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        step_ms = ts.tolist()
    ms_per_step = total_ms / args.steps
    value = n_total / (ms_per_step / 1e3) / 1e9

    # roofline: algorithmic bytes B_alg = 8n + M/4 per sort
    # (key read + bitset write + bitset read + key write) over the step's
    # kernel time (the sum of the live per-launch CUDA-event durations of the
    # sort's kernels in one step; the slowest rank at N > 1), against the
    # measured HBM peak of all N GPUs. The design's own per-kernel traffic
    # fraction (bytes each kernel really has to move) is reported apart as
    # `impl_frac`.
    peak, peak_src = measured_peak()
    kernels = {}
    n_local = shard_h.size
    kernel_ms_per_step = 0.0
    for name, (cnt, ms) in ktimes.items():
        avg_s = ms / cnt / 1e3
        bytes_ = kernel_alg_bytes(name, n_local, M, world)
        kernels[name] = {"launches": cnt, "avg_us": round(avg_s * 1e6, 2),
                         "impl_bytes": bytes_, "GBps": round(bytes_ / avg_s / 1e9, 1) if bytes_ else None,
                         "share": round(ms / max(total_ms_k, 1e-9), 3)}
        kernel_ms_per_step += ms / args.steps
    if use_dist and ktimes:
        t = torch.tensor([kernel_ms_per_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kernel_ms_per_step = float(t.item())
    step_alg = 8 * n_total + M // 4
    roofline = None
    if ktimes:
        dom_name, (dom_cnt, dom_ms) = max(ktimes.items(), key=lambda kv: kv[1][1])
        dom_s = dom_ms / dom_cnt / 1e3
        achieved = step_alg / (kernel_ms_per_step / 1e3) / 1e9
        roofline = {
            "bound": "hbm", "kernel": "+".join(sorted(ktimes)),
            "achieved": round(achieved, 1), "peak": round(peak * world, 1), "unit": "GB/s",
            "frac": round(achieved / (peak * world), 4),
            "frac_of_nominal_8tbs": round(achieved / (NOMINAL_HBM_GBS * world), 4),
            "traffic": traffic_from_profiles(cfg.name, "step"),
            "alg_bytes_per_step": step_alg,
            "formula": "SURVEY.md 8(d): B_alg = 8n + M/4 (key read + bitset write + bitset read + key write) "
                       "/ the step's summed kernel time / (N x peak)",
            "kernel_us_per_step": round(kernel_ms_per_step * 1e3, 2),
            "peak_source": peak_src,
            "timing": "per-launch CUDA events on the launching stream, from a second K-step pass "
                      "(the events add ~10 us per step, so `value` comes from a pass without them)",
            "impl_frac": {"kernel": dom_name,
                          "impl_bytes_per_launch": kernel_alg_bytes(dom_name, n_local, M, world),
                          "achieved": round(kernel_alg_bytes(dom_name, n_local, M, world) / dom_s / 1e9, 1),
                          "frac": round(kernel_alg_bytes(dom_name, n_local, M, world) / dom_s / 1e9 / peak, 4),
                          "traffic": traffic_from_profiles(cfg.name, dom_name),
                          "note": "the dominant kernel's own bytes (the bytes this design moves, "
                                  "DESIGN.md kernel table) over its average launch time"}}
    step_roofline = {"alg_bytes": step_alg,
                     "achieved": round(step_alg / (ms_per_step / 1e3) / 1e9, 1),
                     "frac": round(step_alg / (ms_per_step / 1e3) / 1e9 / (peak * world), 4),
                     "frac_of_nominal_8tbs": round(step_alg / (ms_per_step / 1e3) / 1e9 / (NOMINAL_HBM_GBS * world), 4),
                     "formula": "8n + M/4 over the whole step (events around the step, incl. memsets)"}

    # end to end through the public API: pinned host keys -> sorted host keys
    e2e_steps = max(1, args.e2e_steps)
    pinned = torch.empty(shard_h.size, dtype=torch.int32, pin_memory=True)
    host = pinned.numpy().view(np.uint32)
    # multi-GPU: this rank's sorted slice comes back into a pinned buffer
    # (at most n keys; a fresh pageable tensor per step would time page faults)
    out_pinned = torch.empty(n_total if use_dist else 1, dtype=torch.int32, pin_memory=True)
    times = []
    for i in range(e2e_steps + 1):
        np.copyto(host, shard_h)  # restore the unsorted input (outside the timed region)
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t_a = time.perf_counter()
        if use_dist:
            kd = pinned.to(dev, non_blocking=True)
            res = distributed_sort(kd, M, n_total=n_total, ops=ops)
            out_pinned[:res.count].copy_(res.keys.view(torch.int32), non_blocking=True)  # D2H of the slice
            torch.cuda.synchronize(dev)
        else:
            capi.sort(host)  # bws_sort(host, n, 32, 1, BWS_ALG_BITWISE): H2D + sort + D2H
        if i > 0:
            times.append(time.perf_counter() - t_a)
    if not use_dist:
        assert np.all(host[1:] > host[:-1])
    e2e_s = sum(times) / len(times)
    if use_dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": round(n_total / e2e_s / 1e9, 4), "unit": UNIT,
           "h2d_bytes_per_step": 4 * int(shard_h.size) * world,
           "d2h_bytes_per_step": 4 * int(shard_h.size) * world,
           "ms_per_step": round(e2e_s * 1e3, 3), "steps": e2e_steps,
           "api": "dist.distributed_sort on pinned host shards" if use_dist
           else "bws_sort (C ABI) on a pinned host array"}

    if not use_dist:
        # the PCIe bound of this e2e: plain pinned copies of the same bytes
        # each way (CUDA events), plus the device-resident step
        xfer = torch.empty(shard_h.size, dtype=torch.int32, device=dev)
        cp_ms = {}
        for name, fn in (("h2d", lambda: xfer.copy_(pinned, non_blocking=True)),
                         ("d2h", lambda: pinned.copy_(xfer, non_blocking=True))):
            fn()
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record()
            for _ in range(3):
                fn()
            b_ev.record()
            b_ev.synchronize()
            cp_ms[name] = a_ev.elapsed_time(b_ev) / 3
        del xfer
        nbytes = 4 * int(shard_h.size)
        bound_ms = cp_ms["h2d"] + cp_ms["d2h"] + ms_per_step
        e2e["pcie"] = {"h2d_GBps": round(nbytes / cp_ms["h2d"] / 1e6, 1),
                       "d2h_GBps": round(nbytes / cp_ms["d2h"] / 1e6, 1),
                       "bound_ms": round(bound_ms, 3),
                       "frac_of_bound": round(bound_ms / (e2e_s * 1e3), 4),
                       "note": "bound = pinned H2D + D2H of the keys + the device-resident step"}

    if not use_dist:  # the same drop-in call on ordinary (pageable) host memory
        pg = shard_h.copy()
        ptimes = []
        for i in range(min(e2e_steps, 3) + 1):
            np.copyto(pg, shard_h)
            t_a = time.perf_counter()
            capi.sort(pg)
            if i > 0:
                ptimes.append(time.perf_counter() - t_a)
        assert np.all(pg[1:] > pg[:-1])
        e2e["pageable"] = {"value": round(n_total / (sum(ptimes) / len(ptimes)) / 1e9, 4),
                           "ms_per_step": round(1e3 * sum(ptimes) / len(ptimes), 3)}
        del pg

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(keys_h, args.cpu_sample_keys, cfg.name)

    if use_dist:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "n": n_total, "key_range": M, "recipe": cfg.recipe,
                   "l2": "flushed between steps (256 MiB write, outside the step events)",
                   "path": args.path,
                   "parallelism": (f"key shards x{world} + " + ("NCCL all-to-all of range-split keys"
                                                                  if args.a2a else
                                                                  "scan fused with CUDA IPC peer reads" if args.p2p else
                                                                  "build fused with bulk-OR pushes to peers' slices"
                                                                  if args.push else "NCCL reduce-scatter"))
                   if use_dist else "single GPU"},
        "step_ms": {"median": round(statistics.median(step_ms), 4), "best": round(min(step_ms), 4),
                    "worst": round(max(step_ms), 4)},
        "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
        "step_roofline": step_roofline, "kernels": kernels, "cpu_baseline": cpu, "clocks": clocks,
    }
    emit(line)
    return 0


def free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args) -> int:
    """`python bench.py --gpus N` outside torchrun: re-executes this script
    under torch.distributed.run with N ranks on 127.0.0.1 (one process per
    GPU, the layout the driver's torchrun launch uses). The ranks inherit
    this process's stdout, so rank 0's JSON line is the only result line."""
    import subprocess

    if not args.dry_run:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py --gpus {args.gpus} needs {args.gpus} CUDA devices; "
                             f"this host has {have}\n")
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_dry(args, cfg):
    """--dry-run: the multi-rank plumbing of a step without a GPU (gloo):
    input-position shards, barrier-bracketed timing, max over ranks, one
    JSON line from rank 0. Exercised by tests/test_bench_cpu.py."""
    import torch
    import torch.distributed as dist

    from paper_1312_0138_b200.dist import shard_bounds, slice_words

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    lo, hi = shard_bounds(cfg.n, rank, world)
    times = []
    for _ in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        cnt = torch.tensor([hi - lo], dtype=torch.int64)
        if world > 1:
            dist.all_reduce(cnt)
        times.append(time.perf_counter() - t0)
    assert int(cnt.item()) == cfg.n
    total = torch.tensor([sum(times[args.warmup:])], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    if rank == 0:
        _, per = slice_words(cfg.key_range, world)
        emit({"dry_run": True, "metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": round(1e3 * float(total.item()) / args.steps, 4),
              "config": {"workload": cfg.name, "n": cfg.n, "key_range": cfg.key_range},
              "shard_keys": hi - lo, "slice_words": per,
              "nvlink_bytes_per_rank": (world - 1) * per * 4})
    return 0


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":
            args.gpus = 1  # rank 0 alone runs the reference arm: no ranks to spawn
        else:
            return launch_ranks(args)
    isolate_stdout()
    from paper_1312_0138_b200.configs import CONFIGS

    names = list(CONFIGS) if args.config == "all" else [args.config]
    rc = 0
    for name in names:
        cfg = CONFIGS[name]
        if args.dry_run:
            rc |= run_dry(args, cfg)
        elif args.impl == "reference":
            rc |= run_reference(args, cfg)
        else:
            rc |= run_ours(args, cfg)
    return rc


if __name__ == "__main__":
    sys.exit(main())
