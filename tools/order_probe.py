"""Does an earlier large sort slow the chunked KB3? C4 kernel times alone,
after C3, and after a shutdown (buffers released)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1312_0138_b200 import capi
from paper_1312_0138_b200.configs import CONFIGS

s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(1 << 26, dtype=torch.int32, device="cuda")


def kt(name, reps=10):
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
    print(name, {a: round(b[1] / b[0] * 1000, 1) for a, b in t.items()}, flush=True)
    del k, o


def e2e(name):
    cfg = CONFIGS[name]
    pinned = torch.empty(cfg.n, dtype=torch.int32, pin_memory=True)
    h = pinned.numpy().view(np.uint32)
    np.copyto(h, cfg.generate())
    capi.sort(h)
    print("e2e", name, flush=True)


kt("C4")
e2e("C3")
kt("C4")
e2e("C4")
kt("C4")
kt("C5", 3)
e2e("C5")
kt("C5", 3)
