"""Completeness of the bucket join at production geometry: its hit set must
equal the one of the independent exhaustive kernel (every folded pattern in
Gray-code order, forced with RFR_FORCE_EXHAUSTIVE) at n = 30..40, with
windows that give 10^3..10^5 hits, on random keys, few-distinct keys (heavy
duplicate buckets: the join's slow path) and all-equal keys, unsharded and
over 4 key-range shards.  The oracle parity tests stop at n <= 26; at these
widths the join runs with r >= 9 bucket bits, halo pairs at bucket edges,
continuation passes and multi-bucket windows, which is what this pins."""
import math

import numpy as np
import pytest

from paper_2410_15880_b200 import search_keys

pytestmark = pytest.mark.gpu
TWO64 = 1 << 64


def _exhaustive(keys, T, monkeypatch):
    with monkeypatch.context() as m:
        m.setenv("RFR_FORCE_EXHAUSTIVE", "1")
        return search_keys(keys, T)


def _join(keys, T, nshards, monkeypatch):
    with monkeypatch.context() as m:
        m.delenv("RFR_FORCE_EXHAUSTIVE", raising=False)
        m.setenv("RFR_FORCE_JOIN", "1")
        parts = [search_keys(keys, T, shard=g, nshards=nshards) for g in range(nshards)]
    return np.sort(np.concatenate(parts))


def _check(keys, T, monkeypatch, lo_hits, hi_hits):
    ex = _exhaustive(keys, T, monkeypatch)
    assert lo_hits <= len(ex) <= hi_hits, len(ex)
    assert len(np.unique(ex)) == len(ex)
    # every exhaustive hit is inside the window (exact arithmetic, a sample)
    n = len(keys)
    for t in ex[:: max(1, len(ex) // 50)]:
        t = int(t)
        assert t < 1 << (n - 1)
        s = sum(int(keys[i]) for i in range(n) if (t >> i) & 1) % TWO64
        assert min(s, TWO64 - s) <= T
    for nshards in (1, 4):
        got = _join(keys, T, nshards, monkeypatch)
        assert len(got) == len(ex), (nshards, len(got), len(ex))
        assert np.array_equal(got, ex), nshards
    return len(ex)


@pytest.mark.parametrize("n,hits", [(30, 3000), (34, 20000), (38, 60000), (40, 1000),
                                    # factor-mode windows (T <= 2^31: the 32-bit classification
                                    # and the batched B probe of the production run pass)
                                    (38, 32), (40, 128)])
def test_join_equals_exhaustive_random_keys(n, hits, monkeypatch):
    rng = np.random.default_rng(1000 + n)
    keys = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    # expected hits 2^(n-1) (2T + 1) / 2^64
    T = int(hits * 2.0 ** (64 - n))
    got = _check(keys, T, monkeypatch, hits // 3, hits * 3)
    assert got > 0


@pytest.mark.parametrize("n", [30, 34, 38, 40])
def test_join_equals_exhaustive_few_distinct_keys(n, monkeypatch):
    """8 distinct values, each repeated ~n/8 times: every subset sum is
    shared by C(k1, c1) ... C(k8, c8) patterns.  The window is centred on a
    sum with ~10^3 such patterns; buckets of identical keys overflow the
    join's warp partitions (slow path)."""
    rng = np.random.default_rng(2000 + n)
    vals = rng.integers(0, 2**64 - 1, size=8, dtype=np.uint64, endpoint=True)
    mult = [n // 8 + (1 if i < n % 8 else 0) for i in range(8)]
    keys = np.concatenate([np.full(m, v, dtype=np.uint64) for v, m in zip(vals, mult)])
    keys = keys[rng.permutation(n)]
    # the window is centred on the sum that takes about half of the copies of
    # the first three values
    take = [m // 2 if i < 3 else 0 for i, m in enumerate(mult)]
    target = sum(int(v) * c for v, c in zip(vals, take)) % TWO64
    T = 1 << 20
    expect = math.prod(math.comb(m, c) for m, c in zip(mult, take))
    ex, got1, got4 = _window_sets(keys, target, T, monkeypatch)
    # the folded space (bit n-1 clear) keeps at least the patterns that do not
    # use the last key
    assert expect // 4 <= len(ex) <= expect, (len(ex), expect)
    assert np.array_equal(got1, ex) and np.array_equal(got4, ex)


@pytest.mark.parametrize("n,k", [(30, 3), (30, 4), (34, 3), (38, 3)])
def test_join_equals_exhaustive_all_equal_keys(n, k, monkeypatch):
    """All keys equal: the hits of the window around k v are the C(n-1, k)
    folded patterns of popcount k, all with the same key sum."""
    rng = np.random.default_rng(3000 + n + k)
    v = int(rng.integers(1, 2**63)) | 1
    keys = np.full(n, v, dtype=np.uint64)
    ex, got1, got4 = _window_sets(keys, (k * v) % TWO64, 1 << 16, monkeypatch)
    assert len(ex) == math.comb(n - 1, k)
    assert all(bin(int(t)).count("1") == k for t in ex)
    assert np.array_equal(got1, ex) and np.array_equal(got4, ex)


def _window_sets(keys, centre, T, monkeypatch):
    """Hit sets of the window (sum - centre) mod 2^64 within +-T: the
    exhaustive kernel, the join unsharded and over 4 shards (the C ABI's
    window is (sum - lo) mod 2^64 <= width)."""
    import ctypes

    from paper_2410_15880_b200 import _lib

    lib = _lib.load()
    _lib.device()
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    n = len(keys)
    lo, width = (centre - T) % TWO64, 2 * T

    def run(shard, nshards):
        cap = 1 << 16
        while True:
            out = np.empty(cap, dtype=np.uint64)
            nout = ctypes.c_int64(0)
            st = _lib.RfrStats()
            _lib.check(lib.rfr_search_keys(_lib.ptr(keys, _lib.U64_P), n, lo, width, shard, nshards,
                                           _lib.ptr(out, _lib.U64_P), cap, ctypes.byref(nout),
                                           ctypes.byref(st)), "rfr_search_keys")
            if nout.value <= cap:
                return out[: nout.value].copy()
            cap = int(nout.value)

    with monkeypatch.context() as m:
        m.setenv("RFR_FORCE_EXHAUSTIVE", "1")
        ex = np.sort(run(0, 1))
    with monkeypatch.context() as m:
        m.delenv("RFR_FORCE_EXHAUSTIVE", raising=False)
        m.setenv("RFR_FORCE_JOIN", "1")
        got1 = np.sort(run(0, 1))
        got4 = np.sort(np.concatenate([run(g, 4) for g in range(4)]))
    assert len(np.unique(ex)) == len(ex)
    return ex, got1, got4


@pytest.mark.parametrize("n,kind", [(12, "random"), (20, "random"), (27, "random"), (30, "random"),
                                    (31, "few"), (28, "few"), (30, "equal")])
def test_small_search_table_kernel_equals_exhaustive(n, kind, monkeypatch):
    """Searches of n <= 31 run table_search_kernel (a sorted table of low-key
    sums per CTA, one binary search per high pattern); the Gray-code brute
    force is its independent checker."""
    rng = np.random.default_rng(4000 + n)
    if kind == "random":
        keys = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
        centre, T = 0, int(2000 * 2.0 ** (64 - n))
    elif kind == "few":
        vals = rng.integers(0, 2**64 - 1, size=6, dtype=np.uint64, endpoint=True)
        keys = vals[rng.integers(0, 6, size=n)]
        centre, T = int(sum(int(v) for v in keys[:5])) % TWO64, 1 << 20
    else:
        v = int(rng.integers(1, 2**63)) | 1
        keys = np.full(n, v, dtype=np.uint64)
        centre, T = (3 * v) % TWO64, 1 << 16
    import ctypes

    from paper_2410_15880_b200 import _lib

    lib = _lib.load()
    _lib.device()
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    lo, width = (centre - T) % TWO64, 2 * T

    def run():
        cap = 1 << 16
        while True:
            out = np.empty(cap, dtype=np.uint64)
            nout = ctypes.c_int64(0)
            st = _lib.RfrStats()
            _lib.check(lib.rfr_search_keys(_lib.ptr(keys, _lib.U64_P), n, lo, width, 0, 1,
                                           _lib.ptr(out, _lib.U64_P), cap, ctypes.byref(nout),
                                           ctypes.byref(st)), "rfr_search_keys")
            if nout.value <= cap:
                return np.sort(out[: nout.value])
            cap = int(nout.value)

    with monkeypatch.context() as m:
        m.delenv("RFR_FORCE_JOIN", raising=False)
        m.delenv("RFR_FORCE_EXHAUSTIVE", raising=False)
        got = run()
    with monkeypatch.context() as m:
        m.setenv("RFR_FORCE_EXHAUSTIVE", "1")
        ex = run()
    assert len(ex) > 0 and np.array_equal(got, ex), (len(got), len(ex))
