"""GPU parity of the recombination search (librfr.so, sm_100a).

Parity mode: recombine_e must return exactly the reference's candidate set
(frozen in tests/golden/recombine_cases.json from pkg/src/polyfactor/
recombine.py:727-775).  Factor mode: search_keys must return exactly the
patterns of the exhaustive uint64 window oracle (oracle/rfr_oracle.c) at
sizes the oracle finishes in seconds, and satisfy size-independent properties
(planted solutions found, every hit inside the window, shard unions) at the
BASELINE.json widths (n = 55 .. 64).
"""
import random

import numpy as np
import pytest

from conftest import rho_of
from oracle import recombine_oracle as O
from paper_2410_15880_b200 import RhoVector, parallel_recombine_e, recombine_e, search_keys
from paper_2410_15880_b200.errors import WidthExceeded
from paper_2410_15880_b200.recombine import RecombineStats

pytestmark = pytest.mark.gpu
TWO64 = 1 << 64


@pytest.fixture(params=["exhaustive", "join"])
def search_path(request, monkeypatch):
    """Searches of n <= 31 run the table kernel; the parity tests run
    each case on the quarter-list join as well (RFR_FORCE_JOIN)."""
    if request.param == "join":
        monkeypatch.setenv("RFR_FORCE_JOIN", "1")
    return request.param


def test_recombine_e_matches_reference_candidate_sets(recombine_cases, search_path):
    for case in recombine_cases:
        got = recombine_e(RhoVector.from_values(rho_of(case)), case["eps"]).patterns
        assert got == frozenset(case["patterns"]), case["tag"]


def test_recombine_e_kats():
    # R/recombine.py KATs (pkg/tests/test_recombine.py:87-89, :436-438)
    assert recombine_e(RhoVector.from_values([0.3, 0.7, 0.5]), 1e-6).patterns == frozenset({0, 0b011})
    assert recombine_e(RhoVector.from_values([0.25, 0.75]), 1e-6).patterns == frozenset({0})
    assert recombine_e(RhoVector.from_values([0.5, 0.5]), 1e-6).patterns == frozenset({0})
    assert recombine_e(RhoVector.from_values([]), 1e-6).patterns == frozenset()


def test_recombine_e_guards():
    with pytest.raises(WidthExceeded):
        recombine_e(RhoVector.from_values([0.5] * 65), 1e-6)
    with pytest.raises(ValueError):
        recombine_e(RhoVector.from_values([0.5, 0.25]), 0.5)
    with pytest.raises(ValueError):
        RhoVector.from_values([1.0])


def test_recombine_e_stats_and_shards(recombine_cases):
    case = next(c for c in recombine_cases if c["tag"] == "ac1_n24_0")
    rho = RhoVector.from_values(rho_of(case))
    st = RecombineStats()
    whole = recombine_e(rho, case["eps"], st).patterns
    # n = 24: the exhaustive kernel (one query per pattern) rather than the join
    assert st.visited == (1 << 12) + (1 << 11) and st.queries == 1 << 23 and st.device_ms > 0
    for g in (2, 3, 7):
        union = set()
        for s in range(g):
            union |= recombine_e(rho, case["eps"], shard=s, nshards=g).patterns
        assert union == whole
        assert parallel_recombine_e(rho, case["eps"], g).patterns == whole


def test_recombine_e_against_c_oracle_random(search_path):
    rng = random.Random(77)
    for _ in range(40):
        n = rng.randint(1, 24)
        vals = sorted(rng.random() for _ in range(n))
        eps = rng.choice([1e-9, 1e-6, 1e-4, 1e-2, 0.2, 0.45])
        assert recombine_e(RhoVector.from_values(vals), eps).patterns == O.c_recombine(vals, eps), (n, eps)


def _oracle_keys(keys, T):
    lo, width = (-T) % TWO64, 2 * T
    return O.c_key_window(keys, lo, width)


@pytest.mark.parametrize("seed", range(6))
def test_search_keys_matches_window_oracle(seed, search_path):
    rng = random.Random(seed)
    for _ in range(12):
        n = rng.randint(1, 26)
        keys = np.array([rng.getrandbits(64) for _ in range(n)], dtype=np.uint64)
        T = rng.choice([0, 1, 1000, 1 << 40, 1 << 55, 1 << 58, 1 << 61])
        got = search_keys(keys, T)
        want = _oracle_keys(keys, T)
        assert np.array_equal(got, want), (n, T)


@pytest.mark.parametrize("seed", range(4))
def test_search_keys2_matches_two_window_oracle(seed, search_path):
    """rfr_search_keys2: the first-window set of the oracle, filtered by the
    second key window (computed here exactly on Python ints)."""
    rng = random.Random(100 + seed)
    for _ in range(8):
        n = rng.randint(1, 24)
        keys = np.array([rng.getrandbits(64) for _ in range(n)], dtype=np.uint64)
        keys2 = np.array([rng.getrandbits(64) for _ in range(n)], dtype=np.uint64)
        T = rng.choice([0, 1000, 1 << 50, 1 << 58, 1 << 61])
        T2 = rng.choice([0, 1 << 40, 1 << 60, 1 << 62, (1 << 63)])
        got = search_keys(keys, T, keys2=keys2, half_width2=T2)
        first = _oracle_keys(keys, T)
        k2 = [int(v) for v in keys2]

        def ok(t):
            s = sum(k2[i] for i in range(n) if (int(t) >> i) & 1) % TWO64
            return (s + T2) % TWO64 <= 2 * T2

        want = np.array([t for t in first if ok(t)], dtype=np.uint64)
        assert np.array_equal(got, want), (n, T, T2)


def test_search_keys_skewed_duplicates_match_oracle(search_path):
    # heavy duplicates: few distinct keys drive buckets past their capacity
    rng = random.Random(9)
    for n in (12, 18, 22, 25):
        base = [rng.getrandbits(64) for _ in range(3)]
        keys = np.array([base[i % 3] if i % 2 else (base[0] >> 3) for i in range(n)], dtype=np.uint64)
        for T in (0, 1 << 20):
            assert np.array_equal(search_keys(keys, T), _oracle_keys(keys, T)), (n, T)
    zeros = np.zeros(20, dtype=np.uint64)  # every subset sums to 0
    assert len(search_keys(zeros, 0)) == 1 << 19


def _planted(n, rng):
    """Random keys with one planted subset summing to 0 mod 2^64."""
    keys = [rng.getrandbits(64) for _ in range(n)]
    subset = rng.sample(range(n - 1), rng.randint(2, n - 2))
    s = sum(keys[i] for i in subset[:-1]) % TWO64
    keys[subset[-1]] = (-s) % TWO64
    pat = sum(1 << i for i in subset)
    return np.array(keys, dtype=np.uint64), pat


@pytest.mark.parametrize("n", [40, 48, 55, 61, 64])
def test_full_width_planted_solution_and_window_property(n):
    rng = random.Random(n)
    keys, pat = _planted(n, rng)
    T = 1 << 9
    got = search_keys(keys, T)
    assert pat in set(int(v) for v in got)
    kl = [int(k) for k in keys]
    for t in got.tolist():
        assert t < (1 << (n - 1))
        s = sum(kl[i] for i in range(n) if (t >> i) & 1) % TWO64
        assert min(s, TWO64 - s) <= T
    # expected false hits ~ 2^(n-1) * (2T+1) / 2^64
    assert len(got) < 64 + 8 * (2 ** (n - 1)) * (2 * T + 1) / TWO64


def test_shards_union_at_full_width():
    rng = random.Random(5)
    keys, pat = _planted(55, rng)
    whole = set(search_keys(keys, 1 << 12).tolist())
    union = set()
    for s in range(4):
        union |= set(search_keys(keys, 1 << 12, shard=s, nshards=4).tolist())
    assert union == whole and pat in whole
