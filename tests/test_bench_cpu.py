"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line and the per-kernel algorithmic-byte formulas."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         check=True).stdout.strip().splitlines()
    assert len(out) == 1
    d = json.loads(out[0])
    assert d["impl"] == "reference" and d["unit"] == "Gkeys/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["cores"] == 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "C1"


def test_kernel_alg_bytes():
    sys.path.insert(0, str(ROOT))
    import bench

    n, m = 1 << 26, 1 << 28
    assert bench.kernel_alg_bytes("bucket_partition", n, m) == 8 * n
    assert bench.kernel_alg_bytes("bucket_sort", n, m) == 8 * n
    assert bench.kernel_alg_bytes("bucket_hist", n, m) == 4 * n
    assert bench.kernel_alg_bytes("bitset_scatter", n, m) == 4 * n + m // 8
    assert bench.kernel_alg_bytes("bitset_scan", n, m, world=2) == m // 16 + 4 * n


def test_native_stdout_goes_to_stderr():
    """Anything native code writes to fd 1 (e.g. NCCL's version banner when
    NCCL_DEBUG is set) must not reach stdout, which carries only result lines."""
    code = ("import os, sys; sys.argv = ['bench.py']; sys.path.insert(0, %r); import bench; "
            "bench.isolate_stdout(); os.write(1, b'NCCL version banner\\n'); "
            "bench.emit({'metric': 'm', 'value': 1})" % str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, check=True)
    assert r.stdout.strip().splitlines() == ['{"metric": "m", "value": 1}']
    assert "NCCL version banner" in r.stderr


def test_launcher_dry_run_two_ranks():
    """`python bench.py --gpus 2` outside torchrun re-executes itself under
    torch.distributed.run with two ranks; --dry-run runs the ranks' plumbing on
    gloo (no GPU). Exactly one JSON line comes back, from rank 0."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run", "--config", "C2",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] is True and d["n_gpus"] == 2 and d["steps"] == 3
    assert d["shard_keys"] == (1 << 26) // 2
    assert d["nvlink_bytes_per_rank"] == (1 << 28) // 32 // 2 * 4


def test_launcher_rejects_missing_devices():
    """Without N CUDA devices `--gpus N` fails with a clear message (exit 2)
    instead of a torchrun error."""
    import torch

    if torch.cuda.device_count() >= 4:
        return
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 2
    assert "needs 4 CUDA devices" in r.stderr
    assert r.stdout.strip() == ""
