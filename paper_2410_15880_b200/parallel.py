"""Multi-GPU form of the search: key-range shards, one rank per GPU.

The reference's multi-worker twin of backend e (``pkg/src/polyfactor/
parallel.py:255-272``, threads over pattern ranges with a shared table) is
replaced by key-range sharding of the bucket grid (DESIGN.md
s5): shard g of G searches buckets [g 2^r / G, (g+1) 2^r / G) of the SAME
folded pattern space; every GPU rebuilds the tiny quarter lists itself, so no
half list crosses NVLink.  The only exchange is the short candidate list:
counts and patterns are all-gathered with torch.distributed (NCCL on GPUs,
gloo in the CPU tests).  Without an initialised process group the shards run
one after another on the local device ("logical shards"), which is how the
single-GPU tests prove the union of shards equals the unsharded result.
"""
from __future__ import annotations

import numpy as np

import ctypes

from . import _lib
from .errors import RecombineDeviceError
from .recombine import CandidateSet, RecombineStats, RhoVector, recombine_e, search_keys


def _dist():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch is in the image
        return None
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist
    return None


def _comm_device(dist):
    """Where this rank's collective buffers live: its engine device for NCCL
    (the device librfr searches on, RFR_DEVICE / LOCAL_RANK -- not whatever
    torch.cuda.current_device() happens to be), the host for gloo."""
    import torch

    if dist.get_backend() == "nccl":
        dev = _lib.device()
        torch.cuda.set_device(dev)
        return torch.device("cuda", dev)
    return torch.device("cpu")


def shard_ranges(nbuckets: int, nshards: int) -> list[tuple[int, int]]:
    """Contiguous bucket ranges per shard (same split as the C ABI)."""
    return [(nbuckets * g // nshards, nbuckets * (g + 1) // nshards) for g in range(nshards)]


def allgather_patterns(local: np.ndarray) -> np.ndarray:
    """All-gather variable-length uint64 pattern lists across ranks (counts
    first, then padded payloads).  Identity without a process group."""
    dist = _dist()
    if dist is None:
        return np.asarray(local, dtype=np.uint64)
    import torch

    dev = _comm_device(dist)
    world = dist.get_world_size()
    cnt = torch.tensor([len(local)], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, cnt)
    counts = [int(c.item()) for c in counts]
    width = max(1, max(counts))
    buf = torch.zeros(width, dtype=torch.int64, device=dev)
    if len(local):
        buf[: len(local)] = torch.from_numpy(np.asarray(local, dtype=np.uint64).view(np.int64)).to(dev)
    parts = [torch.zeros(width, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = [p[:c].cpu().numpy().view(np.uint64) for p, c in zip(parts, counts)]
    return np.sort(np.concatenate(out)) if out else np.zeros(0, dtype=np.uint64)


def sharded_search_keys(keys: np.ndarray, half_width: int, workers: int,
                        stats: RecombineStats | None = None, keys2: np.ndarray | None = None,
                        half_width2: int = 0) -> np.ndarray:
    """Factor-mode search split into `workers` key-range shards: this rank's
    shard(s) on its GPU, then an all-gather of the candidate patterns."""
    kw = dict(keys2=keys2, half_width2=half_width2)
    dist = _dist()
    if dist is not None:
        world, rank = dist.get_world_size(), dist.get_rank()
        mine = [g for g in range(workers) if g % world == rank]
        local = [search_keys(keys, half_width, stats, shard=g, nshards=workers, **kw) for g in mine]
        local = np.concatenate(local) if local else np.zeros(0, dtype=np.uint64)
        return allgather_patterns(local)
    parts = [search_keys(keys, half_width, stats, shard=g, nshards=workers, **kw)
             for g in range(workers)]
    return np.sort(np.concatenate(parts))


def parallel_recombine_e(rho: RhoVector, eps: float, workers: int,
                         stats: RecombineStats | None = None) -> CandidateSet:
    """Backend e over `workers` key-range shards (R/parallel.py:255-272
    contract: the candidate set equals the serial one for any worker count).
    ValueError for workers < 1."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if not isinstance(rho, RhoVector):
        rho = RhoVector.from_values(rho)
    dist = _dist()
    if dist is not None:
        world, rank = dist.get_world_size(), dist.get_rank()
        local = set()
        for g in range(workers):
            if g % world == rank:
                local |= recombine_e(rho, eps, stats, shard=g, nshards=workers).patterns
        allp = allgather_patterns(np.array(sorted(local), dtype=np.uint64))
        return CandidateSet(frozenset(int(v) for v in allp), len(rho))
    pats = set()
    for g in range(workers):
        pats |= recombine_e(rho, eps, stats, shard=g, nshards=workers).patterns
    return CandidateSet(frozenset(pats), len(rho))


# ------------------------------------------------ sharded fused search
_PEERS: dict = {}
_EPOCH = [0]  # sharded searches so far (the stop flags' epoch)


def connect_peers(dist) -> bool:
    """Map the other ranks' stop flags (CUDA IPC handles of their search
    counters, all-gathered once per process group): afterwards a rank whose
    search verifies a factor stops every rank's join over NVLink.  False
    (and no cross-rank stop, results unchanged) when a handle cannot be
    exported or opened."""
    key = (id(dist.group.WORLD), dist.get_world_size(), dist.get_rank())
    if _PEERS.get("key") == key:
        return _PEERS["ok"]
    lib = _lib.load()
    _lib.device()
    world, rank = dist.get_world_size(), dist.get_rank()
    h = ctypes.create_string_buffer(64)
    mine = bytes(h.raw) if lib.rfr_peer_handle(h) == _lib.RFR_OK else None
    handles = [None] * world
    _comm_device(dist)
    dist.all_gather_object(handles, mine)
    ok = False
    if all(x is not None for x in handles) and world - 1 <= 8:
        buf = ctypes.create_string_buffer(b"".join(handles), 64 * world)
        ok = lib.rfr_peer_connect(buf, world, rank) == _lib.RFR_OK
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    _PEERS.update(key=key, ok=ok, all=all(flags))
    return ok


def sharded_search_verify(prof, p, keys, half_width, keys3, half_width3, workers: int, fstats,
                          early_exit: bool, max_rows=None):
    """The fused search + verification (verify._search_and_verify) split into
    `workers` key-range shards: this rank's shards on its GPU, a verified hit
    stops every rank's join (connect_peers), then the rows (pattern, verdict,
    side, coefficients) are all-gathered so every rank holds the same
    candidates.  Without a process group the shards run one after another on
    the local device and the first one that stops at a verified factor (and
    searches its pieces) ends the loop.  Returns (pats, verdict, side, coeffs,
    complete, stopped) like _search_and_verify: complete when every shard was
    searched whole or a stopped shard searched its pieces (then the rows
    cover every factor pattern)."""
    from .verify import _search_and_verify

    dist = _dist()
    if dist is None:
        world, rank = 1, 0
    else:
        world, rank = dist.get_world_size(), dist.get_rank()
        connect_peers(dist)
        dist.barrier()  # start together: a peer's stop flag lands in a running search
    # the search's epoch: the same on every rank (the calls are collective)
    _EPOCH[0] += 1
    epoch = _EPOCH[0]
    rows, err = [], None
    for g in [g for g in range(workers) if g % world == rank]:
        try:
            res = _search_and_verify(prof, p, keys, half_width, keys3, half_width3, fstats.recombine,
                                     early_exit, max_rows, shard=g, nshards=workers, epoch=epoch)
        except RecombineDeviceError as e:
            if "raw hits exceed" not in str(e):
                raise
            err = str(e)
            break
        rows.append(res)
        if res[5]:  # stopped: this rank's or a peer's verified factor
            if not (res[1] == _lib.V_PASS).any():
                fstats.peer_stops += 1
            break
    if dist is not None:
        parts = [None] * world
        _comm_device(dist)
        dist.all_gather_object(parts, (err, rows))
        errs = [e for e, _ in parts if e]
        rows = [r for _, rs in parts for r in rs]
        err = errs[0] if errs else None
    if err:
        raise RecombineDeviceError(err)
    stopped = any(r[5] for r in rows)
    complete = any(r[5] and r[4] for r in rows) or (
        all(r[4] for r in rows) and len(rows) == workers)
    if not rows:
        z = np.zeros(0, dtype=np.uint64)
        return z, np.zeros(0, np.uint8), np.zeros(0, np.uint8), np.zeros((0, 65), np.int64), True, False
    cat = [np.concatenate([r[k] for r in rows]) for k in range(4)]
    return cat[0], cat[1], cat[2], cat[3], complete, stopped
