"""The CUDA IPC variants of the multi-GPU sort with real processes: two ranks
(processes) share the one GPU of this build, exchange CUDA IPC handles of
their bitsets / slices, and run dist.distributed_sort_p2p (scan kernel reading
the other process's bitset) and dist.distributed_sort_push (build kernel ORing
bucket bitsets into the other process's slice) end to end. The host
collectives run on gloo (NCCL cannot put two ranks on one GPU). No kernel
waits on another rank: cross-process ordering comes from the host fences, as
on a node; the IPC mappings here are same-device instead of NVLink peers.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, keys, key_range, variant, q):
    import torch
    import torch.distributed as dist

    from paper_1312_0138_b200.dist import distributed_sort_p2p, distributed_sort_push, shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_bounds(keys.size, rank, world)
        t = torch.from_numpy(keys[lo:hi].view(np.int32).copy()).cuda()
        fn = distributed_sort_p2p if variant == "p2p" else distributed_sort_push
        res = fn(t, key_range, n_total=keys.size)
        torch.cuda.synchronize()
        q.put((rank, "ok", res.keys.cpu().numpy().view(np.uint32).copy(), res.offset, res.total))
    except Exception as e:  # reported to the parent
        q.put((rank, type(e).__name__, str(e), 0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["p2p", "push"])
@pytest.mark.parametrize("world,key_range,n", [(2, 1 << 24, 1 << 21), (3, (1 << 20) + 3, 300_000)])
def test_ipc_variants_two_processes(cuda, variant, world, key_range, n):
    import torch.multiprocessing as mp

    keys = np.random.default_rng(world * 7 + n).choice(key_range, size=n, replace=False).astype(np.uint32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, keys, key_range, variant, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    parts = []
    for rank, status, out, offset, total in res:
        assert status == "ok", (rank, status, out)
        assert total == n and offset == sum(x.size for x in parts)
        parts.append(out)
    assert np.array_equal(np.concatenate(parts), np.sort(keys))
