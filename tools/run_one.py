"""Runs one config's device-resident sort a few times (for ncu launch lists)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_0138_b200 import capi  # noqa: E402
from paper_1312_0138_b200.configs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--path", default="BUCKETED")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--flush", action="store_true", help="write 256 MiB between sorts (cold L2, as bench.py does)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
keys = torch.from_numpy(cfg.generate().view(np.int32)).cuda()
out = torch.empty_like(keys)
capi.set_path(getattr(capi.Path, a.path))
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda") if a.flush else None
for _ in range(a.iters):
    if flush is not None:
        flush.fill_(1)
    capi.sort_device_async(keys.data_ptr(), cfg.n, out.data_ptr(), cfg.key_range, s)
assert capi.sort_check(s) == cfg.n
print("ok", a.config, a.path)
