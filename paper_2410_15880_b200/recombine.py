"""The recombination search: drop-in for backend e of the reference.

Mirrors ``pkg/src/polyfactor/recombine.py`` ("R/recombine.py") for the path
the north_star names: ``RhoVector``, ``CandidateSet``, ``RecombineStats``,
``value``, ``accept``, ``GUARD``, ``recombine_e`` and the ``BACKENDS``
registry keep their names, signatures and error behaviour.  The search itself
runs on the GPU (librfr.so, sm_100a); there is no CPU fallback and no second
backend: ``BACKENDS`` holds only ``"e"``.

Two entry points reach the same device join (DESIGN.md sections 2-3):
  * ``recombine_e(rho, eps, stats)`` -- parity mode.  Keys are round(rho *
    2^64); the window is eps + GUARD wide; every hit is re-tested with the
    reference's own float64 ``value``/``accept`` on the device, so the set
    equals the reference's (R/recombine.py:727-775, :148-162).
  * ``search_keys(keys, n, half_width)`` -- factor mode, used by factor():
    exact 64-bit keys from high-precision roots and a window derived from
    their error bounds.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import WidthExceeded
from .rootfinder import RootProfile

GUARD = 1e-12  # R/recombine.py:28-30 (slack added to the discovery band)
MAX_WIDTH = 64  # pattern width cap (R/recombine.py:694-698 caps n at 64)


@dataclass(frozen=True)
class RhoVector:
    """The subset-sum instance: n fractional parts plus prefix sums
    (R/recombine.py:37-63)."""

    values: np.ndarray
    sigma: np.ndarray
    is_sorted: bool

    @classmethod
    def from_values(cls, values, sort: bool = False) -> "RhoVector":
        vals = np.asarray(values, dtype=np.float64)
        if vals.ndim != 1:
            raise ValueError("rho must be one-dimensional")
        if len(vals) and (vals.min() < 0.0 or vals.max() >= 1.0):
            raise ValueError("rho entries must lie in [0, 1)")
        if sort:
            vals = np.sort(vals)
        sigma = np.concatenate(([0.0], np.cumsum(vals)))
        srt = bool(np.all(np.diff(vals) >= 0)) if len(vals) else True
        return cls(values=vals, sigma=sigma, is_sorted=srt)

    @classmethod
    def from_profile(cls, profile: RootProfile) -> "RhoVector":
        return cls.from_values(profile.rho)

    def __len__(self) -> int:
        return len(self.values)


@dataclass(frozen=True)
class CandidateSet:
    """Canonical patterns (min(s, ~s), i.e. bit n-1 clear) that passed the
    accept test (R/recombine.py:66-79)."""

    patterns: frozenset
    n: int

    def nontrivial(self) -> frozenset:
        full = (1 << self.n) - 1
        return frozenset(s for s in self.patterns if s not in (0, full))

    def __len__(self) -> int:
        return len(self.patterns)


@dataclass
class RecombineStats:
    """Counters (R/recombine.py:82-103).  For the device join: visited =
    records enumerated (both folded halves), inserts = A records indexed,
    queries = B records streamed, query_probes = A records compared, plus
    per-phase device milliseconds."""

    visited: int = 0
    inserts: int = 0
    insert_probes: int = 0
    queries: int = 0
    query_probes: int = 0
    find_steps: int = 0
    raw_hits: int = 0
    device_ms: float = 0.0
    # early exit: microseconds from the verified hit to the join's stop (the
    # last search that stopped; -1 when none did)
    hit_to_stop_us: float = -1.0
    # early stops whose two pieces were searched by kernels chained on the
    # device behind the main search (rfr_stats.pieces == 2)
    device_pieces: int = 0

    @property
    def probes_mean(self) -> float:
        return self.insert_probes / self.inserts if self.inserts else 0.0

    def merge(self, other: "RecombineStats") -> None:
        for name in ("visited", "inserts", "insert_probes", "queries", "query_probes",
                     "find_steps", "raw_hits", "device_ms"):
            setattr(self, name, getattr(self, name) + getattr(other, name))


def value(s: int, rho) -> float:
    """Canonical pattern value: frac of the ascending-index float64 sum
    (R/recombine.py:106-118)."""
    vals = rho.values if isinstance(rho, RhoVector) else rho
    x = 0.0
    i = 0
    while s:
        if s & 1:
            x += vals[i]
        s >>= 1
        i += 1
    return x - math.floor(x)


def accept(y: float, eps: float) -> bool:
    """y within eps of an integer end, strict (R/recombine.py:121-123)."""
    return y < eps or (1.0 - y) < eps


def _guard_width(n: int) -> None:
    if n > MAX_WIDTH:
        raise WidthExceeded(f"pattern width is capped at {MAX_WIDTH} bits, got {n}")


def _fill_stats(stats: RecombineStats | None, st: "_lib.RfrStats") -> None:
    if stats is None:
        return
    stats.visited += int(st.visited)
    stats.inserts += int(st.inserts)
    stats.insert_probes += int(st.insert_probes)
    stats.queries += int(st.queries)
    stats.query_probes += int(st.query_probes)
    stats.raw_hits += int(st.raw_hits)
    stats.device_ms += float(st.ms_total)
    if st.us_hit_to_stop >= 0:
        stats.hit_to_stop_us = float(st.us_hit_to_stop)
    stats.device_pieces += int(st.pieces == 2)


def recombine_e(rho: RhoVector, eps: float, stats: RecombineStats | None = None,
                shard: int = 0, nshards: int = 1) -> CandidateSet:
    """Backend e on the GPU: the reference's candidate set for (rho, eps).

    shard/nshards select one key-range slice of the search (multi-GPU); the
    union over shards is the full set.  Raises WidthExceeded for n > 64 and
    ValueError for eps outside (0, 0.5) or rho outside [0, 1)."""
    if not isinstance(rho, RhoVector):
        rho = RhoVector.from_values(rho)
    n = len(rho)
    _guard_width(n)
    if not 0 < eps < 0.5:
        raise ValueError("eps must be in (0, 0.5)")
    if n == 0:
        return CandidateSet(frozenset(), 0)
    lib = _lib.load()
    _lib.device()
    vals = np.ascontiguousarray(rho.values, dtype=np.float64)
    cap = 1 << 16
    while True:
        out = np.empty(cap, dtype=np.uint64)
        nout = ctypes.c_int64(0)
        st = _lib.RfrStats()
        _lib.check(
            lib.rfr_recombine_e(_lib.ptr(vals, _lib.D_P), n, float(eps), shard, nshards,
                                _lib.ptr(out, _lib.U64_P), cap, ctypes.byref(nout),
                                ctypes.byref(st)),
            "rfr_recombine_e",
        )
        if nout.value <= cap:
            break
        cap = int(nout.value)  # grow-and-retry, R/recombine.py:750-757
    _fill_stats(stats, st)
    return CandidateSet(frozenset(int(v) for v in out[: nout.value]), n)


def _window(half_width: int) -> tuple[int, int]:
    T = int(half_width)
    if 2 * T >= (1 << 64) - 1:
        return 0, (1 << 64) - 1
    return (-T) % (1 << 64), 2 * T


def search_keys(keys: np.ndarray, half_width: int, stats: RecombineStats | None = None,
                shard: int = 0, nshards: int = 1, keys2: np.ndarray | None = None,
                half_width2: int = 0) -> np.ndarray:
    """Factor-mode search: sorted uint64 patterns t < 2^(n-1) whose key sum
    lies within +-half_width of 0 (mod 2^64) -- and, when ``keys2`` is given,
    whose ``keys2`` sum lies within +-half_width2 of 0 as well (the secondary
    window is applied on the device, ``rfr_search_keys2``)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    n = len(keys)
    _guard_width(n)
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    lib = _lib.load()
    _lib.device()
    lo, width = _window(half_width)
    if keys2 is not None:
        keys2 = np.ascontiguousarray(keys2, dtype=np.uint64)
        if len(keys2) != n:
            raise ValueError("keys2 must have one key per rho entry")
        lo2, width2 = _window(half_width2)
    cap = 1 << 12
    while True:
        out = np.empty(cap, dtype=np.uint64)
        nout = ctypes.c_int64(0)
        st = _lib.RfrStats()
        if keys2 is None:
            rc = lib.rfr_search_keys(_lib.ptr(keys, _lib.U64_P), n, lo, width, shard, nshards,
                                     _lib.ptr(out, _lib.U64_P), cap, ctypes.byref(nout),
                                     ctypes.byref(st))
        else:
            rc = lib.rfr_search_keys2(_lib.ptr(keys, _lib.U64_P), n, lo, width,
                                      _lib.ptr(keys2, _lib.U64_P), lo2, width2, shard, nshards,
                                      _lib.ptr(out, _lib.U64_P), cap, ctypes.byref(nout),
                                      ctypes.byref(st))
        _lib.check(rc, "rfr_search_keys")
        if nout.value <= cap:
            break
        cap = int(nout.value)
    _fill_stats(stats, st)
    return np.sort(out[: nout.value])


# The registry of the reference (R/recombine.py:778-784) restricted to the
# one backend this engine implements; factor(backend=...) rejects others.
BACKENDS = {"e": recombine_e}
