"""Multi-rank host logic on CPU: key-range shard split and the candidate
all-gather over torch.distributed (gloo, world size 2)."""
import os
import socket

import numpy as np
import pytest

from paper_2410_15880_b200.parallel import allgather_patterns, shard_ranges


def test_shard_ranges_partition_the_bucket_grid():
    for nb in (4, 7, 1 << 15):
        for g in (1, 2, 3, 8):
            rs = shard_ranges(nb, g)
            assert rs[0][0] == 0 and rs[-1][1] == nb
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def test_allgather_is_identity_without_a_group():
    a = np.array([5, 1, 3], dtype=np.uint64)
    assert allgather_patterns(a).tolist() == [5, 1, 3]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = np.array([rank * 10 + k for k in range(rank + 1)] + [(1 << 63) + rank], dtype=np.uint64)
        got = allgather_patterns(local)
        out_q.put((rank, got.tolist()))
    finally:
        dist.destroy_process_group()


def test_allgather_two_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = sorted([0, 1 << 63, 10, 11, (1 << 63) + 1])
    assert res[0] == want and res[1] == want
