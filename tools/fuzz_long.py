"""Long randomised parity run (development tool): the sweeps of
tests/test_gpu_fuzz.py with a fresh seed per case, for --minutes. Every sort
is compared with numpy; the first mismatch stops the run with its case.

usage: python tools/fuzz_long.py [--minutes 5] [--seed S]
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_0138_b200 import capi  # noqa: E402

DTYPES = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64]


def one_case(rng):
    dt = np.dtype(DTYPES[int(rng.integers(0, len(DTYPES)))])
    info = np.iinfo(dt)
    n = int(rng.choice([rng.integers(1, 3000), rng.integers(3000, 1 << 20), rng.integers(1 << 20, 1 << 24)]))
    distinct = info.bits >= 32 and rng.random() < 0.5
    span_bits = int(rng.integers(max(1, int(np.ceil(np.log2(max(n, 2)))) + (2 if distinct else 0)), info.bits + 1)) \
        if distinct else int(rng.integers(1, info.bits + 1))
    span_bits = min(span_bits, info.bits)
    base = np.frombuffer(rng.bytes(8), dtype=np.uint64)[0]
    udt = np.dtype(f"uint{info.bits}")
    if distinct and span_bits <= 26:
        off = rng.choice(1 << span_bits, size=min(n, 1 << span_bits), replace=False).astype(np.uint64)
    else:
        off = np.frombuffer(rng.bytes(8 * n), dtype=np.uint64) & np.uint64((1 << span_bits) - 1)
        if distinct:
            off = np.unique(off)
            rng.shuffle(off)
    keys = (base + off).astype(udt).view(dt)
    path = str(rng.choice(["AUTO", "DIRECT", "BUCKETED", "FUSED", "FUSED_DIRECT", "SMALL"]))
    on_device = rng.random() < 0.5
    offset = int(rng.integers(0, 3))
    return dt, keys, path, on_device, offset


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=5.0)
    ap.add_argument("--seed", type=int, default=int(time.time()))
    a = ap.parse_args()
    torch.cuda.set_device(0)
    master = np.random.default_rng(a.seed)
    deadline = time.time() + 60 * a.minutes
    done = keys_total = 0
    while time.time() < deadline:
        seed = int(master.integers(0, 2**63))
        dt, keys, path, on_device, offset = one_case(np.random.default_rng(seed))
        info = np.iinfo(dt)
        capi.set_path(getattr(capi.Path, path))
        ctx = f"seed={seed} dtype={dt} n={keys.size} path={path} device={on_device} offset={offset}"
        hinted = dt == np.uint32 and keys.size > 0 and np.unique(keys).size == keys.size and \
            np.random.default_rng(seed ^ 1).random() < 0.5
        if hinted:
            # the range-hint extension (bws_gpu_sort_device_async): KS / KD / KF / K2+K3 / KB3+KB4
            # by path and size, output to a second buffer with guard words
            key_range = min(1 << 32, int(keys.max()) + 1 + int(np.random.default_rng(seed ^ 2).integers(0, 1000)))
            src = torch.zeros(keys.size + offset, dtype=torch.int32, device="cuda")
            src[offset:].copy_(torch.from_numpy(keys.view(np.int32).copy()))
            out = torch.full((keys.size + 4,), -1, dtype=torch.int32, device="cuda")
            s = torch.cuda.current_stream().cuda_stream
            capi.sort_device_async(src[offset:].data_ptr(), keys.size, out.data_ptr(), key_range, s)
            total = capi.sort_check(s)
            res = out.cpu().numpy().view(np.uint32)
            got = res[: keys.size]
            untouched = res[keys.size:].tolist() == [0xFFFFFFFF] * 4 and total == keys.size
            st = capi.Status.OK
            ctx += f" hinted range={key_range}"
        elif on_device:
            buf = torch.zeros(keys.nbytes + (offset + 2) * keys.itemsize, dtype=torch.uint8, device="cuda")
            view = buf[offset * keys.itemsize: offset * keys.itemsize + keys.nbytes]
            view.copy_(torch.from_numpy(keys.view(np.uint8).copy()))
            st = capi.sort_raw(view.data_ptr(), keys.size, info.bits, int(info.min == 0), 0)
            got = view.cpu().numpy().view(dt)
            untouched = int(buf[: offset * keys.itemsize].sum()) == 0 and \
                int(buf[offset * keys.itemsize + keys.nbytes:].sum()) == 0
        else:
            got = keys.copy()
            st = capi.sort_raw(got.ctypes.data, keys.size, info.bits, int(info.min == 0), 0)
            untouched = True
        if st != capi.Status.OK or not untouched or not np.array_equal(got, np.sort(keys)):
            print("MISMATCH", ctx, st, capi.last_error(), "guard ok" if untouched else "guard written", flush=True)
            return 1
        done += 1
        keys_total += keys.size
    capi.set_path(capi.Path.AUTO)
    print(f"ok: {done} cases, {keys_total} keys, seed {a.seed}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
