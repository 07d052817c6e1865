"""`bitsort sort` (tools/bitsort_cli.cpp): the reference CLI's sort subcommand
(proj/tools/main.cpp:97-144, :206-223) over the B200 library. Parsing,
option and exit-status behaviour run on CPU; sorting needs the GPU.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_1312_0138_b200" / "lib" / "bitsort"


def run(args, stdin=None):
    return subprocess.run([str(CLI), *args], input=stdin, capture_output=True, text=True)


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not CLI.exists():
        pytest.skip("bitsort CLI not built (run __graft_entry__.build())")


def test_parse_errors_report_file_and_line(tmp_path):
    f = tmp_path / "in.txt"
    f.write_text("5\n# comment\n\n  7 \nseven\n")
    r = run(["sort", str(f)])
    assert r.returncode == 2  # main.cpp:20-31: data errors exit 2
    assert f"{f}:5: cannot parse 'seven' as an integer" in r.stderr
    r = run(["sort", "-"], stdin="1\n-2147483649\n")
    assert r.returncode == 2 and "<stdin>:2: value -2147483649 out of range for signed 32-bit" in r.stderr
    r = run(["sort", "-", "--unsigned"], stdin="4294967296\n")
    assert r.returncode == 2 and "out of range for unsigned 32-bit" in r.stderr


def test_usage_and_config_errors(tmp_path):
    assert run([]).returncode == 1
    assert run(["bits", "5"]).returncode == 1
    assert run(["sort"]).returncode == 1
    f = tmp_path / "in.txt"
    f.write_text("3\n1\n")
    r = run(["sort", str(f), "--width", "24"])
    assert r.returncode == 1 and "unsupported width 24" in r.stderr
    r = run(["sort", "-", "--width", "8"], stdin="1\n128\n")
    assert r.returncode == 2 and "<stdin>:2: value 128 out of range for signed 8-bit" in r.stderr
    r = run(["sort", "-", "--width", "16", "--unsigned"], stdin="65536\n")
    assert r.returncode == 2 and "out of range for unsigned 16-bit" in r.stderr
    r = run(["sort", str(f), "--algorithm", "nonsense"])
    assert r.returncode == 1 and "unknown algorithm" in r.stderr
    assert run(["sort", str(f), "--bogus"]).returncode == 1


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_device_is_an_error(tmp_path):
    f = tmp_path / "in.txt"
    f.write_text("3\n1\n")
    r = run(["sort", str(f)])
    assert r.returncode == 1 and "no CPU fallback" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("signed", [True, False])
def test_sort_file_on_gpu(tmp_path, signed):
    rng = np.random.default_rng(3)
    if signed:
        keys = np.unique(rng.integers(-(1 << 31), 1 << 31, size=300_000, dtype=np.int64))
    else:
        keys = np.unique(rng.integers(0, 1 << 32, size=300_000, dtype=np.uint64))
    keys = rng.permutation(keys)
    f = tmp_path / "in.txt"
    f.write_text("# header\n" + "\n".join(str(int(k)) for k in keys) + "\n\n")
    out = tmp_path / "out.txt"
    args = ["sort", str(f), "--out", str(out), "--threads", "4"] + ([] if signed else ["--unsigned"])
    r = run(args)
    assert r.returncode == 0, r.stderr
    got = [int(x) for x in out.read_text().split()]
    assert got == sorted(int(k) for k in keys)
    # stdin -> stdout; repeated keys sort like the reference's
    r = run(["sort", "-"] + ([] if signed else ["--unsigned"]), stdin="3\n1\n2\n")
    assert r.returncode == 0 and r.stdout == "1\n2\n3\n"
    r = run(["sort", "-"], stdin="3\n1\n3\n")
    assert r.returncode == 0 and r.stdout == "1\n3\n3\n", r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("width", [8, 16, 64])
@pytest.mark.parametrize("signed", [True, False])
def test_sort_other_widths(tmp_path, width, signed):
    """--width 8/16/64 (main.cpp's width option) through bws_sort at that width."""
    rng = np.random.default_rng(width)
    if width == 64:
        lo = -(1 << 63) + 5 if signed else (1 << 64) - (1 << 31)
        keys = [lo + int(x) for x in rng.integers(0, 1 << 30, size=5000)]
    else:
        lo, hi = (-(1 << (width - 1)), 1 << (width - 1)) if signed else (0, 1 << width)
        keys = [int(x) for x in rng.integers(lo, hi, size=5000)]
    keys += [keys[0], keys[1]]  # repeats
    f = tmp_path / "in.txt"
    f.write_text("\n".join(str(k) for k in keys) + "\n")
    r = run(["sort", str(f), "--width", str(width)] + ([] if signed else ["--unsigned"]))
    assert r.returncode == 0, r.stderr
    assert [int(x) for x in r.stdout.split()] == sorted(keys)


@pytest.mark.gpu
@pytest.mark.parametrize("devices", ["0,0", "0,0,0,0"])
def test_sort_on_logical_ranks(tmp_path, devices):
    """The unchanged CLI sorts on G devices when BITSORT_DEVICES lists them
    (here G logical ranks sharing the one GPU): bws_sort's multi-GPU path."""
    import os

    rng = np.random.default_rng(17)
    keys = rng.permutation(np.unique(rng.integers(0, 1 << 32, size=400_000, dtype=np.uint64)))
    f = tmp_path / "in.txt"
    f.write_text("\n".join(str(int(k)) for k in keys) + "\n")
    env = dict(os.environ, BITSORT_DEVICES=devices, BITSORT_MULTI_MIN_KEYS="0")
    r = subprocess.run([str(CLI), "sort", str(f), "--unsigned"], capture_output=True, text=True, env=env)
    assert r.returncode == 0, r.stderr
    assert [int(x) for x in r.stdout.split()] == sorted(int(k) for k in keys)
