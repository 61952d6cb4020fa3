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

from .recombine import CandidateSet, RecombineStats, RhoVector, recombine_e, search_keys


def _dist():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch is in the image
        return None
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist
    return None


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

    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
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
