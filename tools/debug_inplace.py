"""Debug: in-place device bws_sort with repeats (mode-2 recovery)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1312_0138_b200 import capi

rng = np.random.default_rng(31)
for n, M in [((1 << 22) + 3, 1 << 23), ((1 << 21) + 3, 1 << 22), (1 << 22, 1 << 24)]:
    keys = rng.integers(0, M, size=n, dtype=np.uint64).astype(np.uint32)
    d = torch.from_numpy(keys.view(np.int32)).cuda()
    st = capi.sort_raw(d.data_ptr(), n, 32, 1, 0)
    got = d.cpu().numpy().view(np.uint32)
    exp = np.sort(keys)
    print(n, M, "status", st, capi.last_error(), "equal", np.array_equal(got, exp))
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        print("  first bad", bad[:5], got[bad[:5]], exp[bad[:5]], "n bad", bad.size)
        vals, cnts = np.unique(got, return_counts=True)
        ev, ec = np.unique(keys, return_counts=True)
        print("  distinct got", vals.size, "exp", ev.size, "max key got", got.max(), "exp", exp.max())
