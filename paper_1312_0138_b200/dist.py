"""Multi-GPU bitset sort, one process per GPU.

Rank r of G holds an input-position shard of the keys. Each rank
  1. builds a FULL bitset of its shard          (K1 clear + K2 scatter, C ABI)
  2. reduce-scatters the bitsets with SUM on 32-bit words -> rank r receives
     words [r*W/G, (r+1)*W/G), i.e. keys [r*M/G, (r+1)*M/G). SUM is exact
     because distinct keys set disjoint bits (NCCL has no bitwise OR).
  3. scans its slice                             (K3, C ABI) -> c_r keys
  4. all-gathers the counts c_r: offset_r = sum(c_<r); sum(c) must equal n,
     otherwise keys were duplicated (cross-rank duplicates carry and lose bits,
     so the total only drops) -> BWS_ERROR_DATA.
The global sorted array is the rank-order concatenation of the local outputs.

The p2p and push variants below are EXPERIMENTAL and opt-in (bench.py --p2p /
--push): their cross-GPU memory ordering has only run with 2-3 processes
sharing one GPU, never across NVLink peers. They fence with a host-side
device synchronisation (every local kernel that wrote peer memory, or whose
memory peers read, has completed) followed by a collective, rather than with
the collective alone. ``distributed_sort`` (NCCL reduce-scatter) is the
default.

Peer-to-peer variant (``distributed_sort_p2p``, NVLink/NVSwitch node): steps 2
and 3 become ONE kernel instead of NCCL + scan — every rank exports its full
bitset through CUDA IPC, and after a cross-rank barrier scans its own slice of
the OR of all G bitsets, the scan's tiles reading the peers' words straight
out of their memory over NVLink (bws_gpu_bitset_scan_sources): no gathered
slice is written to HBM or read back. OR is exact on distinct keys and only
loses bits on duplicates.

Push variant (``distributed_sort_push``, NVLink/NVSwitch node): steps 1 and 2
become ONE kernel — every rank allocates its (zeroed) slice and exports it
through CUDA IPC; each rank then builds its shard's bitset bucket by bucket in
shared memory and ORs every finished bucket straight into the owner ranks'
slices with bulk OR-reductions over NVLink (bws_gpu_bitset_push). No rank
materialises a full bitset and no separate collective runs; after a barrier
each owner scans its slice.

Key all-to-all variant (``distributed_sort_a2a``): rank r
splits its shard by destination key range (range split, C ABI), the ranks
exchange the groups with one all-to-all (4n/G bytes per rank instead of the
reduce-scatter's (G-1)/G * M/8), and each rank sorts the keys of its range
[r*W, (r+1)*W) with the bucketed pipeline offset by r*W. Cheaper than the
bitset reduce-scatter whenever n/M < G/32 (sparse ranges: C4, C5).

The collectives go through torch.distributed (NCCL on GPUs; gloo in the CPU
tests). The per-rank compute is an injectable ``RankOps``: ``CudaRankOps``
(the product, sm_100a kernels through libbitsort.so) or, in tests only, an
oracle-backed CPU implementation that exercises this host logic on gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Protocol

import torch
import torch.distributed as dist
from torch.cuda import nvtx  # ranges around the exchange steps (no-ops unless a profiler attaches)


class RankOps(Protocol):
    def bitset_build(self, keys: torch.Tensor, key_range: int, words: int) -> torch.Tensor:
        """Full bitset (``words`` int32 words, zero beyond key_range) of ``keys``."""

    def bitset_scan(self, bits: torch.Tensor, key_base: int, capacity: int) -> tuple[torch.Tensor, torch.Tensor]:
        """(out[capacity] keys, count as a 1-element int64 tensor) of a slice."""

    def range_split(self, keys: torch.Tensor, key_range: int, parts: int):
        """(keys grouped by part, int64 counts[parts] tensor, part width W, ok):
        part p holds keys in [p*W, (p+1)*W); ok is False if a key >= key_range."""

    def sort_range(self, keys: torch.Tensor, key_lo: int, key_range: int):
        """(sorted keys, ok) for keys in [key_lo, key_lo + key_range); ok is
        False on duplicates or keys outside the range."""

    def export_bitset(self, bits: torch.Tensor):
        """A picklable handle other ranks can open to read ``bits``."""

    def import_peer(self, rank: int, handle):
        """Source for or_gather of the bitset behind another rank's handle."""

    def or_gather(self, sources, word_lo: int, n_words: int) -> torch.Tensor:
        """OR of words [word_lo, word_lo + n_words) over all sources (local
        tensor or imported peers)."""

    def or_scan(self, sources, word_lo: int, n_words: int, key_base: int,
                capacity: int) -> tuple[torch.Tensor, torch.Tensor]:
        """bitset_scan of or_gather(sources, word_lo, n_words) in one step
        (the CUDA build fuses the peer reads into the scan kernel)."""

    def alloc_slice(self, n_words: int) -> torch.Tensor:
        """A zeroed slice this rank owns (push variant)."""

    def export_slice(self, slice_: torch.Tensor):
        """A picklable handle through which other ranks write ``slice_``."""

    def import_slice(self, rank: int, handle):
        """Writable target for bitset_push behind another rank's handle."""

    def bitset_push(self, keys: torch.Tensor, key_range: int, targets, slice_words: int) -> None:
        """OR the bitset of ``keys`` into the slices: targets[r] holds words
        [r * slice_words, (r + 1) * slice_words)."""


@dataclass
class SliceResult:
    keys: torch.Tensor      # this rank's sorted keys (a view of length `count`)
    count: int
    offset: int             # position of keys[0] in the global sorted array
    total: int              # keys over all ranks
    key_lo: int             # this rank's key range [key_lo, key_hi)
    key_hi: int


def push_slice_words(key_range: int, world: int) -> int:
    """Words per rank of the push variant: whole 16-byte units (bulk
    reductions move 16 bytes at a time)."""
    words = (key_range + 31) // 32
    per = (words + world - 1) // world
    return (per + 3) // 4 * 4


def slice_words(key_range: int, world: int) -> tuple[int, int]:
    """(padded total words, words per rank): the bitset is padded so every rank
    owns the same number of whole words."""
    words = (key_range + 31) // 32
    per = (words + world - 1) // world
    return per * world, per


def part_width(key_range: int, parts: int) -> int:
    """Range-split part width: the smallest q * 2^s >= ceil(key_range / parts)
    with q <= 8, s in [12, 31] and s >= 15 when q > 1 (the bucket map of the C
    library's range split, bucket.cu plan_range_split, which this mirrors)."""
    want = -(-key_range // parts)
    best = None
    for s_ in range(12, 32):
        for q in range(1, 9):
            w = q << s_
            if w < want or (q > 1 and s_ < 15):
                continue
            if best is None or w < best:
                best = w
    return best


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Input-position shard [lo, hi) of rank (balanced by construction)."""
    return n * rank // world, n * (rank + 1) // world


class CudaRankOps:
    """Per-rank compute on this process's CUDA device through the C ABI."""

    def __init__(self, device: Optional[torch.device] = None):
        from . import capi  # loads libbitsort.so; raises if it is not built

        self._capi = capi
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self._bits: Optional[torch.Tensor] = None
        self._out: Optional[torch.Tensor] = None
        self._total = torch.zeros(1, dtype=torch.int64, device=self.device)

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def bitset_build(self, keys: torch.Tensor, key_range: int, words: int) -> torch.Tensor:
        if self._bits is None or self._bits.numel() < words:
            self._bits = torch.empty(words, dtype=torch.int32, device=self.device)
        bits = self._bits[:words]
        if words * 32 > key_range:  # padding words beyond the key range stay zero
            bits[(key_range + 31) // 32:].zero_()
        self._capi.bitset_build(keys.data_ptr(), keys.numel(), bits.data_ptr(), key_range,
                                self._stream())
        return bits

    def range_split(self, keys: torch.Tensor, key_range: int, parts: int):
        grouped = torch.empty(max(keys.numel(), 1), dtype=torch.int32, device=self.device)
        counts = torch.zeros(parts, dtype=torch.int32, device=self.device)
        try:
            width = self._capi.range_split(keys.data_ptr(), keys.numel(), key_range, parts,
                                           grouped.data_ptr(), counts.data_ptr(), self._stream())
        except self._capi.BitsortError:
            return grouped, counts.to(torch.int64), 0, False
        return grouped, counts.to(torch.int64), width, True

    def sort_range(self, keys: torch.Tensor, key_lo: int, key_range: int):
        out = torch.empty_like(keys)
        if keys.numel() == 0:
            return out, True
        s = self._stream()
        self._capi.sort_range_device_async(keys.data_ptr(), keys.numel(), out.data_ptr(), key_lo, key_range, s)
        try:
            self._capi.sort_check(s)
        except self._capi.BitsortError:
            return out, False
        return out, True

    def export_bitset(self, bits: torch.Tensor):
        return self._capi.ipc_get_handle(bits.data_ptr())

    def import_peer(self, rank: int, handle):
        raw, offset = handle
        cache = self.__dict__.setdefault("_peers", {})
        old = cache.get(rank)
        if old is None or old[0] != raw:  # a new allocation behind the peer's bitset
            if old is not None:
                self._capi.ipc_close(old[1])
            cache[rank] = (raw, self._capi.ipc_open(raw))
        return cache[rank][1] + offset

    def or_gather(self, sources, word_lo: int, n_words: int) -> torch.Tensor:
        ptrs = [(src.data_ptr() if isinstance(src, torch.Tensor) else int(src)) + 4 * word_lo
                for src in sources]
        buf = self.__dict__.get("_slice")
        if buf is None or buf.numel() < n_words:
            buf = torch.empty(max(n_words, 1), dtype=torch.int32, device=self.device)
            self._slice = buf
        self._capi.bitset_or_gather(ptrs, n_words, buf.data_ptr(), self._stream())
        return buf[:n_words]

    def or_scan(self, sources, word_lo: int, n_words: int, key_base: int, capacity: int):
        ptrs = [(src.data_ptr() if isinstance(src, torch.Tensor) else int(src)) + 4 * word_lo
                for src in sources]
        if self._out is None or self._out.numel() < capacity:
            self._out = torch.empty(max(capacity, 1), dtype=torch.int32, device=self.device)
        self._capi.bitset_scan_sources(ptrs, n_words, key_base, self._out.data_ptr(), capacity,
                                       self._total.data_ptr(), self._stream())
        return self._out, self._total

    def alloc_slice(self, n_words: int) -> torch.Tensor:
        return torch.zeros(max(n_words, 4), dtype=torch.int32, device=self.device)[:n_words]

    def export_slice(self, slice_: torch.Tensor):
        return self.export_bitset(slice_)

    def import_slice(self, rank: int, handle):
        return self.import_peer(rank, handle)

    def bitset_push(self, keys: torch.Tensor, key_range: int, targets, slice_words: int) -> None:
        ptrs = [t.data_ptr() if isinstance(t, torch.Tensor) else int(t) for t in targets]
        self._capi.bitset_push(keys.data_ptr(), keys.numel(), key_range, ptrs, slice_words, self._stream())

    def bitset_scan(self, bits: torch.Tensor, key_base: int, capacity: int):
        if self._out is None or self._out.numel() < capacity:
            self._out = torch.empty(max(capacity, 1), dtype=torch.int32, device=self.device)
        self._capi.bitset_scan(bits.data_ptr(), bits.numel(), key_base, self._out.data_ptr(),
                               capacity, self._total.data_ptr(), self._stream())
        return self._out, self._total


def distributed_sort(keys: torch.Tensor, key_range: int, n_total: Optional[int] = None,
                     ops: Optional[RankOps] = None, group=None) -> SliceResult:
    """Sorts the union of every rank's ``keys`` shard (distinct uint32 keys in
    [0, key_range)); returns this rank's slice of the sorted result."""
    if not 0 < key_range <= 1 << 32:
        raise ValueError("key_range must be in [1, 2^32]")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = ops or CudaRankOps(keys.device)
    words, per = slice_words(key_range, world)
    if n_total is None:
        t = torch.tensor([keys.numel()], dtype=torch.int64, device=keys.device)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())

    bits = ops.bitset_build(keys, key_range, words)
    slice_ = torch.empty(per, dtype=torch.int32, device=bits.device)
    with nvtx.range("bitsort:NCCL reduce-scatter"):
        dist.reduce_scatter_tensor(slice_, bits, op=dist.ReduceOp.SUM, group=group)

    key_lo = rank * per * 32
    key_hi = min((rank + 1) * per * 32, key_range)
    capacity = max(0, min(n_total, key_hi - key_lo))
    out, count_t = ops.bitset_scan(slice_, key_lo, capacity)

    counts_h = _gather_counts(count_t, world, group)
    total = sum(counts_h)
    if total != n_total:
        from .capi import BitsortError, Status

        raise BitsortError(Status.ERROR_DATA,
                           f"keys are not distinct or out of range: {n_total} keys, {total} distinct")
    count = counts_h[rank]
    return SliceResult(keys=out[:count], count=count, offset=sum(counts_h[:rank]), total=total,
                       key_lo=key_lo, key_hi=key_hi)


def _gather_counts(count_t: torch.Tensor, world: int, group) -> list[int]:
    """Every rank's count (one all-gather, then ONE device-to-host read for all
    of them rather than one blocking read per rank)."""
    counts = [torch.empty_like(count_t) for _ in range(world)]
    dist.all_gather(counts, count_t, group=group)
    return [int(c) for c in torch.stack(counts).reshape(-1).tolist()]


def _device_sync(dev: torch.device) -> None:
    """Host-side completion of every kernel queued on this rank's device (a
    no-op for the CPU tensors of the gloo tests)."""
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)


def _data_error(msg: str):
    from .capi import BitsortError, Status

    return BitsortError(Status.ERROR_DATA, msg)


def distributed_sort_a2a(keys: torch.Tensor, key_range: int, n_total: Optional[int] = None,
                         ops: Optional[RankOps] = None, group=None) -> SliceResult:
    """Key all-to-all variant of :func:`distributed_sort`: same inputs, same
    global result; rank r's slice is the sorted keys of [r*W, (r+1)*W) where W
    is the range-split part width."""
    if not 0 < key_range <= 1 << 32:
        raise ValueError("key_range must be in [1, 2^32]")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = ops or CudaRankOps(keys.device)
    dev = keys.device
    if n_total is None:
        t = torch.tensor([keys.numel()], dtype=torch.int64, device=dev)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())

    if world == 1:  # one part: the split is the identity
        grouped, width, ok = keys, part_width(key_range, 1), True
        counts = torch.tensor([keys.numel()], dtype=torch.int64, device=dev)
    else:
        grouped, counts, width, ok = ops.range_split(keys, key_range, world)
    bad = torch.tensor([0 if ok else 1], dtype=torch.int64, device=dev)
    dist.all_reduce(bad, group=group)  # every rank raises together, before the exchange
    if int(bad.item()):
        raise _data_error(f"keys not below the key range {key_range} on {int(bad.item())} rank(s)")
    counts = counts.to(dev)
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    sc = [int(c) for c in counts.tolist()]
    rc = [int(c) for c in recv_counts.tolist()]
    recv = torch.empty(sum(rc), dtype=torch.int32, device=dev)
    with nvtx.range("bitsort:NCCL all-to-all"):
        dist.all_to_all_single(recv, grouped[:sum(sc)], output_split_sizes=rc, input_split_sizes=sc,
                               group=group)

    key_lo = min(rank * width, key_range)
    key_hi = min((rank + 1) * width, key_range)
    out, ok = ops.sort_range(recv, key_lo, max(key_hi - key_lo, 1)) if recv.numel() else (recv, True)
    stat = torch.tensor([recv.numel(), 0 if ok else 1], dtype=torch.int64, device=dev)
    stats = [torch.empty_like(stat) for _ in range(world)]
    dist.all_gather(stats, stat, group=group)
    st = torch.stack(stats).tolist()  # one device-to-host read
    counts_h = [int(x[0]) for x in st]
    errors = sum(int(x[1]) for x in st)
    total = sum(counts_h)
    if errors or total != n_total:
        raise _data_error(f"keys are not distinct: {n_total} keys, duplicates within "
                          f"{errors} rank range(s)")
    count = counts_h[rank]
    return SliceResult(keys=out[:count], count=count, offset=sum(counts_h[:rank]), total=total,
                       key_lo=key_lo, key_hi=key_hi)


def distributed_sort_p2p(keys: torch.Tensor, key_range: int, n_total: Optional[int] = None,
                         ops: Optional[RankOps] = None, group=None) -> SliceResult:
    """:func:`distributed_sort` with the reduce-scatter and the slice scan
    replaced by one fused kernel that scans the OR of every rank's bitset
    slice, reading the peers' words over CUDA IPC (same result layout)."""
    if not 0 < key_range <= 1 << 32:
        raise ValueError("key_range must be in [1, 2^32]")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = ops or CudaRankOps(keys.device)
    dev = keys.device
    words, per = slice_words(key_range, world)
    if n_total is None:
        t = torch.tensor([keys.numel()], dtype=torch.int64, device=dev)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())

    bits = ops.bitset_build(keys, key_range, words)
    key_lo = rank * per * 32
    key_hi = min((rank + 1) * per * 32, key_range)
    capacity = max(0, min(n_total, key_hi - key_lo))
    if world == 1:
        sources = [bits]
    else:
        handles = [None] * world
        dist.all_gather_object(handles, ops.export_bitset(bits), group=group)
        # the local bitset first: the fused scan copies it by TMA, peers by loads
        sources = [bits] + [ops.import_peer(r, h) for r, h in enumerate(handles) if r != rank]
        # barrier: every rank's build has completed (host-side synchronisation,
        # so its bitset writes are visible to the peers) before any rank
        # enqueues the scan that reads the peers' bitsets
        _device_sync(dev)
        fence = torch.zeros(1, dtype=torch.int32, device=dev)
        dist.all_reduce(fence, group=group)
        _device_sync(dev)
    with nvtx.range("bitsort:p2p scan over peer bitsets"):
        out, count_t = ops.or_scan(sources, rank * per, per, key_lo, capacity)
    # the counts' all-gather doubles as the "peers are done reading" barrier
    # (each rank's count is read back only after its scan has completed)
    counts_h = _gather_counts(count_t, world, group)
    total = sum(counts_h)
    if total != n_total:
        raise _data_error(f"keys are not distinct or out of range: {n_total} keys, {total} distinct")
    count = counts_h[rank]
    return SliceResult(keys=out[:count], count=count, offset=sum(counts_h[:rank]), total=total,
                       key_lo=key_lo, key_hi=key_hi)


def distributed_sort_push(keys: torch.Tensor, key_range: int, n_total: Optional[int] = None,
                          ops: Optional[RankOps] = None, group=None) -> SliceResult:
    """:func:`distributed_sort` with the bitset build and the reduce-scatter
    fused: every rank ORs its bucket bitsets straight into the owners' slices
    (bws_gpu_bitset_push over CUDA IPC); each owner then scans its slice.
    Slices hold :func:`push_slice_words` words (a multiple of 4)."""
    if not 0 < key_range <= 1 << 32:
        raise ValueError("key_range must be in [1, 2^32]")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = ops or CudaRankOps(keys.device)
    dev = keys.device
    per = push_slice_words(key_range, world)
    if n_total is None:
        t = torch.tensor([keys.numel()], dtype=torch.int64, device=dev)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())

    own = ops.alloc_slice(per)
    fence = torch.zeros(1, dtype=torch.int32, device=dev)
    if world == 1:
        targets = [own]
    else:
        handles = [None] * world
        dist.all_gather_object(handles, ops.export_slice(own), group=group)
        targets = [own if r == rank else ops.import_slice(r, h) for r, h in enumerate(handles)]
        # every slice is zeroed (completed, host-synchronised) before anyone pushes
        _device_sync(dev)
        dist.all_reduce(fence, group=group)
        _device_sync(dev)
    if keys.numel():
        with nvtx.range("bitsort:push build into owners' slices"):
            ops.bitset_push(keys, key_range, targets, per)
    if world > 1:
        # every rank's pushes have completed (host-synchronised: the bulk ORs
        # into the peers' slices are done) before any owner scans its slice
        _device_sync(dev)
        dist.all_reduce(fence, group=group)
        _device_sync(dev)

    key_lo = rank * per * 32
    key_hi = min((rank + 1) * per * 32, key_range)
    capacity = max(0, min(n_total, key_hi - key_lo))
    out, count_t = ops.bitset_scan(own, key_lo, capacity)
    counts_h = _gather_counts(count_t, world, group)
    total = sum(counts_h)
    if total != n_total:
        raise _data_error(f"keys are not distinct or out of range: {n_total} keys, {total} distinct")
    count = counts_h[rank]
    return SliceResult(keys=out[:count], count=count, offset=sum(counts_h[:rank]), total=total,
                       key_lo=key_lo, key_hi=key_hi)
