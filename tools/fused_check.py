"""Quick GPU check of the fused KF path: C1/C2 and edge cases through
bws_gpu_sort_device_async with BITSORT path FUSED, vs np.sort; repeated
sorts (ring laps); CUDA-event timing. Run on the GPU box."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1312_0138_b200 import capi, configs

torch.cuda.set_device(0)
capi.set_path(capi.Path.FUSED)
s = torch.cuda.current_stream().cuda_stream


def run(keys, key_range, reps=1, time_it=False, path=capi.Path.FUSED):
    capi.set_path(path)
    d = torch.from_numpy(keys.view(np.int32)).cuda()
    out = torch.empty_like(d)
    exp = np.sort(keys)
    ok = True
    for r in range(reps):
        out.fill_(-1)
        capi.sort_device_async(d.data_ptr(), keys.size, out.data_ptr(), key_range, s)
        tot = capi.sort_check(s)
        got = out.cpu().numpy().view(np.uint32)
        if tot != keys.size or not np.array_equal(got, exp):
            bad = np.nonzero(got != exp)[0]
            print(f"  MISMATCH rep {r}: total={tot} n={keys.size} first bad idx {bad[:5]} got {got[bad[:5]]} exp {exp[bad[:5]]}")
            ok = False
            break
    t = None
    if time_it:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        for _ in range(3):
            capi.sort_device_async(d.data_ptr(), keys.size, out.data_ptr(), key_range, s)
        torch.cuda.synchronize()
        ts = []
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for _ in range(10):
            flush.fill_(1)
            e0.record()
            capi.sort_device_async(d.data_ptr(), keys.size, out.data_ptr(), key_range, s)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        capi.set_kernel_timing(True)
        capi.kernel_timings()
        for _ in range(5):
            flush.fill_(1)
            capi.sort_device_async(d.data_ptr(), keys.size, out.data_ptr(), key_range, s)
        torch.cuda.synchronize()
        kt = capi.kernel_timings()
        capi.set_kernel_timing(False)
        print("   kernels:", {k: round(v[1] / v[0] * 1000, 1) for k, v in kt.items()}, "us", flush=True)
    return ok, t


if "--trace" in sys.argv:  # BITSORT_KF_TRACE=1 set by the caller
    for cname in ["C1", "C2"]:
        cfg = configs.CONFIGS[cname]
        keys = cfg.generate()
        run(keys, cfg.key_range, reps=4)
        if cname == "C1":
            run(keys, cfg.key_range, reps=4, path=capi.Path.FUSED_DIRECT)
    sys.exit(0)

rng = np.random.default_rng(1)
cases = []
for n, M in [(1, 1 << 20), (3, 1 << 20), (5, 1 << 20), (100, 1 << 20), (4097, 1 << 20), (65537, 1 << 24),
             (1 << 20, 1 << 22), (1 << 22, 1 << 27), (3_000_001, 1 << 28), (1 << 24, 1 << 24)]:
    k = rng.choice(M, size=n, replace=False).astype(np.uint32) if n < M else rng.permutation(M).astype(np.uint32)
    cases.append((f"rand n={n} M=2^{M.bit_length()-1}", k, M))
k = np.arange(1 << 22, dtype=np.uint32); cases.append(("sorted 2^22", k, 1 << 22))
cases.append(("reverse 2^22", k[::-1].copy(), 1 << 22))
cases.append(("top keys", np.array([(1 << 28) - 1, 0, (1 << 27), (1 << 27) - 1], dtype=np.uint32), 1 << 28))
allok = True
for name, keys, M in cases:
    ok, _ = run(keys, M, reps=3)
    print(f"{name}: {'ok' if ok else 'FAIL'}", flush=True)
    allok &= ok
for n, M in [(1 << 16, 1 << 24), (1 << 20, 1 << 24), (1 << 22, 1 << 26), (1 << 22, 1 << 27)]:
    keys = rng.choice(M, size=n, replace=False).astype(np.uint32)
    for path in (capi.Path.SMALL, capi.Path.FUSED_DIRECT, capi.Path.DIRECT, capi.Path.BUCKETED):
        ok, t = run(keys, M, reps=2, time_it=True, path=path)
        print(f"n=2^{n.bit_length()-1} M=2^{M.bit_length()-1} {path.name}: {'ok' if ok else 'FAIL'} {t*1000:.1f} us", flush=True)
        allok &= ok
for cname in ["C1", "C2"]:
    cfg = configs.CONFIGS[cname]
    keys = cfg.generate()
    if cname == "C1":
        oks, ts = run(keys, cfg.key_range, reps=20, time_it=True, path=capi.Path.SMALL)
        print(f"C1 small (KS): {'ok' if oks else 'FAIL'}  {ts*1000:.1f} us  {cfg.n / ts / 1e6:.1f} Gkeys/s", flush=True)
        allok &= oks
        okd, td = run(keys, cfg.key_range, reps=5, time_it=True, path=capi.Path.FUSED_DIRECT)
        print(f"C1 fused_direct: {'ok' if okd else 'FAIL'}  {td*1000:.1f} us  {cfg.n / td / 1e6:.1f} Gkeys/s", flush=True)
        allok &= okd
    ok, t = run(keys, cfg.key_range, reps=20, time_it=True)
    print(f"{cname} fused: {'ok' if ok else 'FAIL'}  {t*1000:.1f} us  {cfg.n / t / 1e6:.1f} Gkeys/s  frac {cfg.alg_bytes / (t*1e-3) / (configs.hbm_peak()[0] * 1e9):.3f}", flush=True)
    ok2, t2 = run(keys, cfg.key_range, reps=1, time_it=True, path=capi.Path.BUCKETED if cname == "C2" else capi.Path.DIRECT)
    print(f"{cname} previous: {t2*1000:.1f} us", flush=True)
    allok &= ok
print("ALL OK" if allok else "SOME FAILED")
