"""Seeded config generators (csrc/datagen.c), pinned by reference-generated
anchors (tests/golden/anchors.json, gen_golden.cpp) where the recipe is the
reference's splitmix64 verbatim."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1312_0138_b200 import datagen
from paper_1312_0138_b200.configs import CONFIGS


def test_c1_matches_reference_anchor(anchors):
    k = CONFIGS["C1"].generate()
    assert k.size == 1_000_000
    assert k[:8].tolist() == anchors["C1"]["first8"]
    assert datagen.fnv1a64(k) == anchors["C1"]["fnv1a64_input"]


@pytest.mark.slow
def test_c2_c4_match_reference_anchors(anchors):
    for name in ("C2", "C4"):
        k = CONFIGS[name].generate()
        assert k[:8].tolist() == anchors[name]["first8"], name
        assert datagen.fnv1a64(k) == anchors[name]["fnv1a64_input"], name
        assert int(k.min()) == anchors[name]["min"] and int(k.max()) == anchors[name]["max"]


@pytest.mark.slow
def test_c5_matches_reference_anchors(anchors):
    """C5 comes from csrc/datagen.c (not the reference's generator); its input
    hash and the reference bws_sort's output hash were recorded by
    gen_golden.cpp from the same generator, so numpy's sort of the keys must
    reproduce the reference's sorted hash."""
    k = CONFIGS["C5"].generate()
    a = anchors["C5"]
    assert k.size == a["n"] and k[:8].tolist() == a["first8"]
    assert datagen.fnv1a64(k) == a["fnv1a64_input"]
    k.sort()
    assert datagen.fnv1a64(k) == a["fnv1a64_sorted"]
    assert int(k[0]) == a["min"] and int(k[-1]) == a["max"]


def test_shuffle_prefix_is_distinct_and_in_range():
    k = datagen.shuffle_prefix(50_000, 1 << 16, seed=7)
    assert np.unique(k).size == k.size and int(k.max()) < 1 << 16
    full = datagen.shuffle_prefix(1 << 12, 1 << 12, seed=7)
    assert np.array_equal(np.sort(full), np.arange(1 << 12, dtype=np.uint32))


@pytest.mark.parametrize("n", [1, 2, 3, 1000, 1 << 16, 100_003])
def test_permutation_is_bijection(n):
    p = datagen.permutation(n, seed=42)
    assert np.array_equal(np.sort(p), np.arange(n, dtype=np.uint32))
    assert np.array_equal(p, datagen.permutation(n, seed=42))
    if n > 100:
        assert not np.array_equal(p, np.arange(n, dtype=np.uint32))


def test_dedup_draws_distinct_and_deterministic():
    a = datagen.dedup_draws(100_000, seed=42)
    assert np.unique(a).size == a.size
    assert np.array_equal(a, datagen.dedup_draws(100_000, seed=42))


def test_cluster_sizes_water_filling():
    caps = np.array([10, 10, 1000, 1000, 1000], dtype=np.uint64)
    sizes = datagen.cluster_sizes(caps, 1500, 1.2)
    assert int(sizes.sum()) == 1500
    assert (sizes <= caps).all()
    assert sizes[0] == 10 and sizes[1] == 10  # capped
    assert sizes[2] >= sizes[3] >= sizes[4]  # Zipf order among the uncapped


def test_clustered_small():
    k, centres = datagen.clustered(200_000, clusters=64, zipf_s=1.2, half_window=1 << 12,
                                   seed=42, return_centres=True)
    assert np.unique(k).size == k.size
    # every key lies in some +-half_window window
    c = np.sort(centres.astype(np.int64))
    kk = k.astype(np.int64)
    idx = np.clip(np.searchsorted(c, kk), 1, c.size - 1)
    d = np.minimum(np.abs(kk - c[idx - 1]), np.abs(kk - c[idx]))
    assert int(d.max()) <= 1 << 12
    assert np.array_equal(k, datagen.clustered(200_000, 64, 1.2, 1 << 12, 42))
