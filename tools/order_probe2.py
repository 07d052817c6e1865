"""Which earlier sort slows the chunked KB3 of C4? usage: order_probe2.py C1 C2 C4 ... (kernel times of each, in order)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1312_0138_b200 import capi
from paper_1312_0138_b200.configs import CONFIGS

s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(1 << 26, dtype=torch.int32, device="cuda")


def kt(name, reps=6):
    cfg = CONFIGS[name]
    k = torch.from_numpy(cfg.generate().view(np.int32)).cuda()
    o = torch.empty_like(k)
    for _ in range(3):
        capi.sort_device_async(k.data_ptr(), cfg.n, o.data_ptr(), cfg.key_range, s)
    torch.cuda.synchronize()
    capi.set_kernel_timing(True)
    capi.kernel_timings()
    for _ in range(reps):
        flush.fill_(1)
        capi.sort_device_async(k.data_ptr(), cfg.n, o.data_ptr(), cfg.key_range, s)
    torch.cuda.synchronize()
    t = capi.kernel_timings()
    capi.set_kernel_timing(False)
    assert capi.sort_check(s) == cfg.n
    print(name, {a: round(b[1] / b[0] * 1000, 1) for a, b in t.items()}, "keys@%x" % k.data_ptr(), flush=True)
    del k, o


for a in sys.argv[1:]:
    if a == "empty":
        torch.cuda.empty_cache()
        print("empty_cache", flush=True)
    elif a.startswith("cudamalloc"):  # e.g. cudamalloc512: a raw cudaMalloc of that many MiB, kept
        import ctypes
        rt = ctypes.CDLL("libcudart.so")
        ptr = ctypes.c_void_p()
        mb = int(a[len("cudamalloc"):])
        rc = rt.cudaMalloc(ctypes.byref(ptr), ctypes.c_size_t(mb << 20))
        print("cudaMalloc", mb, "MiB ->", rc, hex(ptr.value or 0), flush=True)
    elif a == "shutdown":
        capi.shutdown()
        print("shutdown", flush=True)
    else:
        kt(a)
