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


def _sv_worker(rank, world, port, scenario, out_q):
    """sharded_search_verify's cross-rank logic with the device call stubbed:
    rank 0's shard stops at a verified factor and searches its pieces, rank
    1's is stopped by it (no PASS row); or rank 1 overflows (flood)."""
    import torch.distributed as dist

    import paper_2410_15880_b200.parallel as par
    import paper_2410_15880_b200.verify as ver
    from paper_2410_15880_b200.errors import RecombineDeviceError

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def fake(prof, p, keys, T, keys3, T3, stats, early, max_rows, shard=0, nshards=1, epoch=0):
        assert nshards == 2 and shard == rank
        if scenario == "flood" and shard == 1:
            raise RecombineDeviceError("70000 raw hits exceed the flood limit 65536")
        pats = np.array([100 + shard, 200 + shard], dtype=np.uint64)
        if shard == 0:  # its own hit (PASS), pieces searched: complete
            verdict = np.array([1, 0], dtype=np.uint8)
            return pats, verdict, np.zeros(2, np.uint8), np.zeros((2, 65), np.int64), True, True
        verdict = np.zeros(2, dtype=np.uint8)  # stopped by the peer: incomplete
        return pats, verdict, np.zeros(2, np.uint8), np.zeros((2, 65), np.int64), False, True

    par.connect_peers = lambda d: False
    ver._search_and_verify = fake
    try:
        fs = ver.FactorStats()
        try:
            out = par.sharded_search_verify(None, None, None, 0, None, 0, 2, fs, True, 1 << 16)
            out_q.put((rank, sorted(int(v) for v in out[0]), bool(out[4]), bool(out[5]), fs.peer_stops))
        except RecombineDeviceError as e:
            out_q.put((rank, "flood" if "raw hits exceed" in str(e) else str(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scenario", ["stop", "flood"])
def test_sharded_search_verify_two_ranks_gloo(scenario):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sv_worker, args=(r, 2, port, scenario, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        item = q.get(timeout=180)
        res[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
    if scenario == "flood":  # one rank's overflow is every rank's
        assert res[0] == ("flood",) and res[1] == ("flood",)
        return
    # both ranks hold the union of the rows; complete (rank 0 searched its
    # pieces), stopped; rank 1 counts one stop by a peer
    assert res[0][:3] == ([100, 101, 200, 201], True, True)
    assert res[1][:3] == res[0][:3]
    assert res[0][3] == 0 and res[1][3] == 1
