"""KS (small.cu) phase trace over a ladder of sizes: run with BITSORT_KS_TRACE=1
(stderr gets one line per sort). usage: python tools/ks_trace.py [--no-flush]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_0138_b200 import capi  # noqa: E402

capi.set_path(capi.Path.SMALL)
s = torch.cuda.current_stream().cuda_stream
flush = None if "--no-flush" in sys.argv else torch.empty(64 << 20, dtype=torch.int32, device="cuda")
rng = np.random.default_rng(3)
for logn, logm in [(10, 24), (14, 24), (16, 24), (18, 24), (20, 24), (20, 27), (16, 20)]:
    n, m = 1 << logn, 1 << logm
    k = rng.choice(m, size=n, replace=False).astype(np.uint32)
    keys = torch.from_numpy(k.view(np.int32)).cuda()
    out = torch.empty_like(keys)
    print(f"# n=2^{logn} M=2^{logm}", file=sys.stderr, flush=True)
    for _ in range(4):
        if flush is not None:
            flush.fill_(1)
        capi.sort_device_async(keys.data_ptr(), n, out.data_ptr(), m, s)
        assert capi.sort_check(s) == n
    assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(k))
print("ok")
