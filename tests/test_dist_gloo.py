"""Multi-rank host logic of dist.distributed_sort on gloo, world_size 2 and 3.

The per-rank compute is the CPU oracle's bitset restatement (test
infrastructure); the collectives (reduce-scatter SUM, all-gather of counts),
the slice/offset arithmetic and duplicate detection are the product code that
runs unchanged over NCCL on GPUs.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1312_0138_b200.dist import (distributed_sort, distributed_sort_a2a, distributed_sort_p2p,
                                       distributed_sort_push, part_width, push_slice_words, shard_bounds,
                                       slice_words)


class OracleRankOps:
    def bitset_build(self, keys, key_range, words):
        bits, _ = oracle.bitset_build(keys.numpy().view(np.uint32), key_range)
        full = np.zeros(words, dtype=np.uint32)
        full[: bits.size] = bits
        return torch.from_numpy(full.view(np.int32))

    def bitset_scan(self, bits, key_base, capacity):
        b = bits.numpy().view(np.uint32)
        out = np.zeros(max(capacity, 1), dtype=np.uint32)
        cnt = oracle.ORACLE.oracle_bitset_scan(b.ctypes.data, b.size, key_base, out.ctypes.data, capacity)
        return torch.from_numpy(out.view(np.int32)), torch.tensor([cnt], dtype=torch.int64)

    def range_split(self, keys, key_range, parts):
        k = keys.numpy().view(np.uint32).astype(np.uint64)
        if k.size and int(k.max()) >= key_range:
            return keys, torch.zeros(parts, dtype=torch.int64), 0, False
        w = part_width(key_range, parts)
        dest = k // w
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest.astype(np.int64), minlength=parts)[:parts]
        grouped = k[order].astype(np.uint32)
        return torch.from_numpy(grouped.view(np.int32)), torch.from_numpy(counts.astype(np.int64)), w, True

    # p2p variant: a rank "exports" its bitset as a file the other ranks map
    # read-only (the CUDA build exports a CUDA IPC handle)
    def export_bitset(self, bits):
        import tempfile

        fd, path = tempfile.mkstemp(prefix="bws_p2p_", suffix=".u32")
        os.close(fd)
        bits.numpy().view(np.uint32).tofile(path)
        return path

    def import_peer(self, rank, handle):
        return torch.from_numpy(np.fromfile(handle, dtype=np.uint32).view(np.int32))

    def or_gather(self, sources, word_lo, n_words):
        acc = np.zeros(n_words, dtype=np.uint32)
        for src in sources:
            acc |= src.numpy().view(np.uint32)[word_lo:word_lo + n_words]
        return torch.from_numpy(acc.view(np.int32))

    # push variant: slices are shared files every rank maps writable; the OR
    # into a slice holds the file's lock (the GPU's bulk OR is atomic in L2)
    def alloc_slice(self, n_words):
        import tempfile

        fd, path = tempfile.mkstemp(prefix="bws_push_", suffix=".u32")
        os.close(fd)
        np.zeros(max(n_words, 1), dtype=np.uint32).tofile(path)
        self.__dict__.setdefault("_slice_path", {})[n_words] = path
        return torch.from_numpy(np.memmap(path, dtype=np.uint32, mode="r+", shape=(n_words,)).view(np.int32))

    def export_slice(self, slice_):
        return self._slice_path[slice_.numel()]

    def import_slice(self, rank, handle):
        return handle

    def bitset_push(self, keys, key_range, targets, slice_words):
        import fcntl

        bits, _ = oracle.bitset_build(keys.numpy().view(np.uint32), key_range)
        for r, tgt in enumerate(targets):
            path = tgt if isinstance(tgt, str) else self._slice_path[tgt.numel()]
            part = bits[r * slice_words:(r + 1) * slice_words]
            with open(path, "r+b") as fh:
                fcntl.flock(fh, fcntl.LOCK_EX)
                m = np.memmap(path, dtype=np.uint32, mode="r+", shape=(slice_words,))
                m[: part.size] |= part
                m.flush()
                del m
                fcntl.flock(fh, fcntl.LOCK_UN)

    def or_scan(self, sources, word_lo, n_words, key_base, capacity):
        return self.bitset_scan(self.or_gather(sources, word_lo, n_words), key_base, capacity)

    def sort_range(self, keys, key_lo, key_range):
        k = keys.numpy().view(np.uint32)
        ok = bool(((k.astype(np.uint64) >= key_lo) & (k.astype(np.uint64) < key_lo + key_range)).all())
        out = oracle.bitwise_sort(k)
        ok = ok and bool((out[1:] > out[:-1]).all())
        return torch.from_numpy(out.view(np.int32)), ok


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, keys, key_range, q, variant="rs"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_bounds(keys.size, rank, world)
        shard = torch.from_numpy(keys[lo:hi].view(np.int32).copy())
        try:
            sorter = {"a2a": distributed_sort_a2a, "p2p": distributed_sort_p2p,
                      "push": distributed_sort_push}.get(variant, distributed_sort)
            r = sorter(shard, key_range, ops=OracleRankOps())
            q.put((rank, "ok", r.keys.numpy().view(np.uint32).copy(), r.offset, r.total, r.key_lo, r.key_hi))
        except Exception as e:  # noqa: BLE001
            q.put((rank, type(e).__name__, getattr(e, "status", None), str(e), 0, 0, 0))
    finally:
        dist.destroy_process_group()


def run_ranks(keys, key_range, world, variant="rs"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, keys, key_range, q, variant))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,key_range,n", [(2, 1 << 20, 100_000), (3, 1000, 1000), (2, 1 << 32, 50_000)])
def test_distributed_sort_gloo(world, key_range, n):
    rng = np.random.default_rng(world * 31 + n)
    if key_range <= 1 << 24:
        keys = rng.choice(key_range, size=n, replace=False).astype(np.uint32)
    else:
        keys = np.unique(rng.integers(0, key_range, size=2 * n, dtype=np.uint64).astype(np.uint32))[:n]
        rng.shuffle(keys)
    res = run_ranks(keys, key_range, world)
    expected = np.sort(keys)
    words, per = slice_words(key_range, world)
    parts = []
    for rank, status, out, offset, total, lo, hi in res:
        assert status == "ok"
        assert total == n
        assert lo == rank * per * 32
        assert offset == sum(p.size for p in parts)
        assert ((out >= lo) & (out < hi)).all()
        parts.append(out)
    assert np.array_equal(np.concatenate(parts), expected)


def test_distributed_duplicates_across_ranks_rejected():
    keys = np.arange(0, 2000, 2, dtype=np.uint32)
    keys[-1] = keys[0]  # rank 1's last key duplicates rank 0's first key
    res = run_ranks(keys, 1 << 12, 2)
    for rank, status, code, msg, *_ in res:
        assert status == "BitsortError"
        assert int(code) == 2  # BWS_ERROR_DATA
        assert "distinct" in msg


def test_slice_and_shard_arithmetic():
    assert slice_words(1 << 32, 8) == ((1 << 27), (1 << 24))
    assert slice_words(1000, 3) == (33, 11)  # 32 words padded to 33
    bounds = [shard_bounds(10, r, 4) for r in range(4)]
    assert bounds == [(0, 2), (2, 5), (5, 7), (7, 10)]


@pytest.mark.parametrize("world,key_range,n", [(2, 1 << 20, 100_000), (3, 1000, 1000), (3, 1 << 32, 50_000)])
def test_distributed_sort_a2a_gloo(world, key_range, n):
    """Key all-to-all variant: range split, all_to_all_single of the groups,
    per-rank range sort; same global result as the reduce-scatter variant."""
    rng = np.random.default_rng(world * 37 + n)
    if key_range <= 1 << 24:
        keys = rng.choice(key_range, size=n, replace=False).astype(np.uint32)
    else:
        keys = np.unique(rng.integers(0, key_range, size=2 * n, dtype=np.uint64).astype(np.uint32))[:n]
        rng.shuffle(keys)
    res = run_ranks(keys, key_range, world, "a2a")
    w = part_width(key_range, world)
    parts = []
    for rank, status, out, offset, total, lo, hi in res:
        assert status == "ok"
        assert total == n
        assert lo == min(rank * w, key_range) and hi == min((rank + 1) * w, key_range)
        assert offset == sum(p.size for p in parts)
        assert ((out >= lo) & (out < hi)).all()
        parts.append(out)
    assert np.array_equal(np.concatenate(parts), np.sort(keys))


@pytest.mark.parametrize("case", ["cross_rank_duplicate", "out_of_range"])
def test_distributed_a2a_errors(case):
    keys = np.arange(0, 2000, 2, dtype=np.uint32)
    key_range = 1 << 12
    if case == "cross_rank_duplicate":
        keys[-1] = keys[0]  # different input shards, same destination rank
    else:
        keys[-1] = key_range + 5
    res = run_ranks(keys, key_range, 2, "a2a")
    for rank, status, code, msg, *_ in res:
        assert status == "BitsortError"
        assert int(code) == 2  # BWS_ERROR_DATA


def test_part_width():
    assert part_width(1 << 32, 8) == 1 << 29
    assert part_width(1 << 28, 3) == 3 << 25  # 89478486 -> 3 * 2^25 = 100663296
    assert part_width(1000, 3) == 1 << 12     # minimum width 2^12
    for m, g in [(1 << 30, 7), (123456789, 5), (1 << 32, 1), ((1 << 32) - 1, 6)]:
        w = part_width(m, g)
        assert w * g >= m and w <= 2 * -(-m // g)


@pytest.mark.parametrize("world,key_range,n", [(2, 1 << 20, 100_000), (3, 1000, 1000)])
def test_distributed_sort_p2p_gloo(world, key_range, n):
    """Peer-to-peer variant: handle exchange (all_gather_object), the fence,
    each rank's OR-gather of its slice from every rank's bitset, the scan and
    the offsets; same layout as the reduce-scatter variant."""
    keys = np.random.default_rng(world * 41 + n).choice(key_range, size=n, replace=False).astype(np.uint32)
    res = run_ranks(keys, key_range, world, "p2p")
    words, per = slice_words(key_range, world)
    parts = []
    for rank, status, out, offset, total, lo, hi in res:
        assert status == "ok", (status, out)
        assert total == n and lo == rank * per * 32 and offset == sum(p.size for p in parts)
        parts.append(out)
    assert np.array_equal(np.concatenate(parts), np.sort(keys))


def test_distributed_p2p_duplicates_rejected():
    keys = np.arange(0, 2000, 2, dtype=np.uint32)
    keys[-1] = keys[0]
    res = run_ranks(keys, 1 << 12, 2, "p2p")
    for rank, status, code, msg, *_ in res:
        assert status == "BitsortError" and int(code) == 2


@pytest.mark.parametrize("world,key_range,n", [(2, 1 << 20, 100_000), (3, 1000, 1000), (3, (1 << 16) + 5, 3000)])
def test_distributed_sort_push_gloo(world, key_range, n):
    """Push variant: slice handles (all_gather_object), the zeroed-slices
    fence, every rank ORing its bitset into every owner's slice, the
    pushes-landed fence, the owners' scans and the offsets."""
    keys = np.random.default_rng(world * 43 + n).choice(key_range, size=n, replace=False).astype(np.uint32)
    res = run_ranks(keys, key_range, world, "push")
    per = push_slice_words(key_range, world)
    assert per % 4 == 0 and per * world * 32 >= key_range
    parts = []
    for rank, status, out, offset, total, lo, hi in res:
        assert status == "ok", (status, out)
        assert total == n and lo == rank * per * 32 and offset == sum(p.size for p in parts)
        parts.append(out)
    assert np.array_equal(np.concatenate(parts), np.sort(keys))


def test_distributed_push_duplicates_rejected():
    keys = np.arange(0, 2000, 2, dtype=np.uint32)
    keys[-1] = keys[0]
    res = run_ranks(keys, 1 << 12, 2, "push")
    for rank, status, code, msg, *_ in res:
        assert status == "BitsortError" and int(code) == 2
