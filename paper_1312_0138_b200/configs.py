"""The five BASELINE.json workloads.

B_alg = 8n + M/4 bytes per sort: key read 4n + bitset write M/8 + bitset read
M/8 + output write 4n.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Callable

import numpy as np

from . import datagen

# /opt/skills/guides/B200_PROFILING.md: the HBM figure to use only when the
# driver-written MEASURED_PEAKS.json is absent
FALLBACK_HBM_GBPS = 6650.0
_PEAKS = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"


def hbm_peak() -> tuple[float, str]:
    """(HBM GB/s, source): MEASURED_PEAKS.json hbm_gbs (the driver's measured
    copy bandwidth on this pool's B200s), else the profiling recipe's fallback.
    The one peak every tool divides by."""
    try:
        return float(json.loads(_PEAKS.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, ValueError, KeyError):
        return FALLBACK_HBM_GBPS, "fallback (B200_PROFILING.md, 6.65 TB/s)"


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    key_range: int
    recipe: str
    make: Callable[..., np.ndarray]

    @property
    def alg_bytes(self) -> int:
        return 8 * self.n + self.key_range // 4

    def generate(self, out=None) -> np.ndarray:
        return self.make(out=out)


CONFIGS = {
    "C1": Config("C1", 1_000_000, 1 << 24,
                 "first 1e6 of a seed-42 splitmix64 Fisher-Yates shuffle of [0,2^24)",
                 lambda out=None: datagen.shuffle_prefix(1_000_000, 1 << 24, 42, out)),
    "C2": Config("C2", 1 << 26, 1 << 28,
                 "first 2^26 of a seed-42 splitmix64 Fisher-Yates shuffle of [0,2^28)",
                 lambda out=None: datagen.shuffle_prefix(1 << 26, 1 << 28, 42, out)),
    "C3": Config("C3", 1 << 30, 1 << 30,
                 "seed-42 keyed Feistel permutation of [0,2^30)",
                 lambda out=None: datagen.permutation(1 << 30, 42, out)),
    "C4": Config("C4", 1 << 24, 1 << 32,
                 "2^24 distinct seed-42 splitmix64 uint32 draws (rejection dedup, draw order)",
                 lambda out=None: datagen.dedup_draws(1 << 24, 42, out)),
    "C5": Config("C5", 1 << 28, 1 << 32,
                 "4096 seed-42 centres, Zipf(1.2) sizes water-filled to +-2^18 windows, "
                 "free-key partial Fisher-Yates per window, Feistel shuffle",
                 lambda out=None: datagen.clustered(1 << 28, 4096, 1.2, 1 << 18, 42, out)),
}
