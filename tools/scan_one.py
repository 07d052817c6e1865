"""Runs the multi-GPU building blocks once on one GPU (bitset_build + bitset_scan) for ncu."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_0138_b200.configs import CONFIGS  # noqa: E402
from paper_1312_0138_b200.dist import CudaRankOps  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
keys = torch.from_numpy(cfg.generate().view(np.int32)).cuda()
ops = CudaRankOps()
words = (cfg.key_range + 31) // 32
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    bits = ops.bitset_build(keys, cfg.key_range, words)
    out, cnt = ops.bitset_scan(bits, 0, cfg.n)
torch.cuda.synchronize()
assert int(cnt.item()) == cfg.n
print("ok", cfg.name)
