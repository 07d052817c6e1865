"""Shared fixtures. `-m gpu` tests need a CUDA device and call the sm_100a path
through the C ABI; everything else runs on the CPU (oracle, golden vectors,
host logic, ABI surface, gloo multi-rank logic)."""
from __future__ import annotations

import json
import struct
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: full-size configuration (seconds to minutes)")


def read_records(path: Path):
    """tests/golden/*.bin written by tests/golden/gen_golden.cpp."""
    buf = path.read_bytes()
    magic, ver, count = struct.unpack_from("<III", buf, 0)
    assert magic == 0x47535742 and ver == 1
    off = 12
    recs = []
    for _ in range(count):
        n, trial, distinct, _pad = struct.unpack_from("<IIII", buf, off)
        off += 16
        inp = np.frombuffer(buf, dtype="<u4", count=n, offset=off).copy()
        off += 4 * n
        out = np.frombuffer(buf, dtype="<u4", count=n, offset=off).copy()
        off += 4 * n
        recs.append({"n": n, "trial": trial, "distinct": bool(distinct), "input": inp, "output": out})
    assert off == len(buf)
    return recs


@pytest.fixture(scope="session")
def acceptance_records():
    return read_records(GOLDEN / "acceptance_u32.bin")


@pytest.fixture(scope="session")
def edge_records():
    return read_records(GOLDEN / "edge_u32.bin")


WIDTH_DTYPES = {(8, 0): np.int8, (8, 1): np.uint8, (16, 0): np.int16, (16, 1): np.uint16,
                (32, 0): np.int32, (32, 1): np.uint32, (64, 0): np.int64, (64, 1): np.uint64}


def read_width_records(path: Path):
    """tests/golden/widths.bin (gen_golden.cpp write_width_records)."""
    buf = path.read_bytes()
    magic, ver, count = struct.unpack_from("<III", buf, 0)
    assert magic == 0x57535742 and ver == 1
    off = 12
    recs = []
    for _ in range(count):
        width, uns, n, dist = struct.unpack_from("<IIII", buf, off)
        off += 16
        dt = np.dtype(WIDTH_DTYPES[(width, uns)]).newbyteorder("<")
        inp = np.frombuffer(buf, dtype=dt, count=n, offset=off).astype(dt.newbyteorder("="))
        off += n * dt.itemsize
        out = np.frombuffer(buf, dtype=dt, count=n, offset=off).astype(dt.newbyteorder("="))
        off += n * dt.itemsize
        recs.append({"width": width, "unsigned": uns, "n": n, "dist": dist, "input": inp, "output": out})
    assert off == len(buf)
    return recs


@pytest.fixture(scope="session")
def width_records():
    return read_width_records(GOLDEN / "widths.bin")


@pytest.fixture(scope="session")
def repeats_records():
    return read_records(GOLDEN / "repeats_u32.bin")


@pytest.fixture(scope="session")
def anchors():
    return json.loads((GOLDEN / "anchors.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
