"""Debug the chunked layout: the a2a building blocks (range sorts)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1312_0138_b200 import capi
from paper_1312_0138_b200.dist import part_width

s = torch.cuda.current_stream().cuda_stream
world, key_range, n = 3, 1 << 32, 300000
rng = np.random.default_rng(world * 7 + n)
keys = np.unique(rng.integers(0, key_range, size=2 * n, dtype=np.uint64).astype(np.uint32))[:n]
w = part_width(key_range, world)
for chunk in ("1", "0"):
    for d in range(world):
        lo, hi = min(d * w, key_range), min((d + 1) * w, key_range)
        part = keys[(keys.astype(np.uint64) >= lo) & (keys.astype(np.uint64) < hi)]
        rng.shuffle(part)
        dd = torch.from_numpy(part.view(np.int32)).cuda()
        out = torch.full((part.size + 4,), -1, dtype=torch.int32, device="cuda")
        try:
            capi.sort_range_device_async(dd.data_ptr(), part.size, out.data_ptr(), lo, hi - lo, s)
            tot, err = capi.sort_check(s), ""
        except capi.BitsortError as e:
            tot, err = -1, str(e)
        got = out[:part.size].cpu().numpy().view(np.uint32)
        print("part", d, "n", part.size, "lo", lo, "range", hi - lo, "total", tot, err,
              "equal", np.array_equal(got, np.sort(part)), flush=True)
    break
