"""factor(): the drop-in entry point, with candidate verification on the GPU.

Mirrors ``pkg/src/polyfactor/verify.py`` ("R/verify.py"): ``factor``,
``is_irreducible``, ``FactorizationResult``, ``FactorStats``,
``selected_degree`` keep their names, signatures, result layout and errors;
the output factorization (irreducible factors with multiplicities, sorted by
(degree, coeffs, mult), R/verify.py:222) is the unique one, so it equals the
reference's wherever the reference finishes.

Pipeline for one monic square-free part p:
  1. host (not timed, ``root_seconds``): hp_profile -- roots to ~2^-100,
     exact 64-bit keys of the first two power sums, window half-width T;
  2. GPU (``recombine_seconds``): search every pattern t < 2^(n-1) whose key
     sum is within +-T of 0, then keep those whose third-power-sum key sum
     is within +-T3 of 0 (device filter) -- the true factors and a handful
     of false hits (also for Swinnerton-Dyer inputs, where Tr1 and Tr2 are
     integral for millions of non-factors);
  3. GPU (``verify_seconds``): one warp per candidate expands the smaller
     side in double-double, checks integrality against a derived error bound
     and trial-divides p modulo three primes below 2^63 (R/verify.py:60-155);
  4. host: the minimal passing patterns (atoms) are the irreducible factors;
     the certificate (exact re-multiplication, R/verify.py:224-231) proves
     the product.  The reference instead re-roots and re-searches every
     piece recursively (R/verify.py:280-284); one search here yields all
     factors.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from fractions import Fraction
from functools import lru_cache

from array import array as _array

import numpy as np

from . import _lib
from .polynomial import (
    IntPolynomial,
    _poly,
    divide_exact,
    poly_gcd,
    monic_transform,
    monic_untransform_factor,
    square_free_decompose,
)
from .recombine import BACKENDS, RecombineStats, search_keys
from .errors import NonConvergence, RecombineDeviceError
from .rootfinder import RootProfile, ToleranceConfig, hp_profile

_STRIDE = 65  # smaller side degree <= 64
# The key windows are rigorous (Lemmas 1-2): every root lies
# in a certified inclusion disc, so the key sum of every true factor is within
# key_err of 0 -- no safety factor on top.


@dataclass
class FactorStats:
    """Per-stage counters of one factor() call (R/verify.py:158-170)."""

    backend: str = "e"
    workers: int = 1
    n: int = 0
    root_seconds: float = 0.0
    recombine_seconds: float = 0.0
    verify_seconds: float = 0.0
    candidates: int = 0
    rejected: int = 0
    recombine: RecombineStats = field(default_factory=RecombineStats)
    host_verified: int = 0
    early_exits: int = 0  # searches stopped at a verified factor
    peer_stops: int = 0  # sharded searches stopped by another rank's verified factor


@dataclass(frozen=True)
class FactorizationResult:
    """R/verify.py:173-184."""

    input: IntPolynomial
    content: int
    factors: tuple
    certificate: bool
    stats: FactorStats

    @property
    def irreducible(self) -> bool:
        return len(self.factors) == 1 and self.factors[0][1] == 1


def selected_degree(s: int, profile: RootProfile) -> int:
    """Degree of the factor a pattern selects: 1 per real root, 2 per pair
    (R/verify.py:48-57)."""
    real, pair = _degree_masks(profile.perm, profile.r)
    s = int(s)
    return (s & real).bit_count() + 2 * (s & pair).bit_count()


@lru_cache(maxsize=1024)
def _degree_masks(perm: tuple, r: int) -> tuple[int, int]:
    """Bit masks of the rho indices holding real roots and pairs."""
    real = sum(1 << i for i, e in enumerate(perm) if e < r)
    return real, sum(1 << i for i in range(len(perm))) & ~real


# inputs whose profile was found without splitting integer roots off first:
# the next call skips that screen (a stale entry only costs the polish's own
# NonConvergence fallback, which splits them then)
_PROFILED: set = set()


@lru_cache(maxsize=256)
def _profile_cached(coeffs: tuple) -> RootProfile:
    return hp_profile(IntPolynomial(coeffs))


# Data derived from a root profile alone (packing and key sums: part of the
# untimed preprocessing, like the roots), kept beside the cached profile.
_DERIVED: "OrderedDict[int, tuple]" = None  # id(prof) -> (prof, {name: value})


def _derived(prof: RootProfile, name: str, make):
    global _DERIVED
    if _DERIVED is None:
        from collections import OrderedDict

        _DERIVED = OrderedDict()
    ent = _DERIVED.get(id(prof))
    if ent is None or ent[0] is not prof:
        ent = (prof, {})
        _DERIVED[id(prof)] = ent
        if len(_DERIVED) > 512:
            _DERIVED.popitem(last=False)
    d = ent[1]
    if name not in d:
        d[name] = make(prof)
    return d[name]


def _search_window(prof: RootProfile) -> tuple[np.ndarray, int]:
    """Combined keys (first + second power sum) and the window half-width."""
    return _derived(prof, "window", _search_window_of)


def _search_window_of(prof: RootProfile) -> tuple[np.ndarray, int]:
    k1 = np.asarray(prof.keys1, dtype=np.uint64)
    k2 = np.asarray(prof.keys2, dtype=np.uint64)
    keys = k1 + k2  # uint64 addition wraps: the sum mod 2^64
    # Lemma 2: |sum of a true factor's combined keys| <= key_err1 + key_err2
    T = prof.key_err1 + prof.key_err2
    return keys, T


def _secondary_window(prof: RootProfile) -> tuple[np.ndarray | None, int]:
    """Third-power-sum keys and half-width (the device's secondary filter),
    or (None, 0) for a profile without them."""
    if prof.keys3 is None:
        return None, 0
    return _derived(prof, "window3", lambda pr: (np.ascontiguousarray(pr.keys3, dtype=np.uint64),
                                                 pr.key_err3))


_PRIMES: tuple[int, ...] | None = None
_PRIMES_I64: np.ndarray | None = None


def _p_mod(p: IntPolynomial) -> np.ndarray:
    """p's coefficients modulo the three verification primes (3 x (d+1))."""
    global _PRIMES, _PRIMES_I64
    if _PRIMES is None:
        primes = np.zeros(3, dtype=np.uint64)
        _lib.load().rfr_verify_primes(primes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        _PRIMES = tuple(int(q) for q in primes)
        _PRIMES_I64 = primes.astype(np.int64)
    co = p.coeffs
    try:  # int64 coefficients: reduced natively (rfr_p_mod_i64; Python's sign rule)
        a = _array("q", co)
    except OverflowError:
        a = None
    if a is not None:
        out = np.empty((3, len(co)), dtype=np.uint64)
        if _lib.load().rfr_p_mod_i64(a.buffer_info()[0], len(co) - 1, out.ctypes.data) == 0:
            return out
    return np.array([[c % q for c in co] for q in _PRIMES], dtype=np.uint64)


def _rfr_profile(prof: RootProfile):
    """The profile as an rfr_profile struct (plus the buffer it points into,
    which the caller keeps alive for the duration of the call): the six
    double arrays packed into one buffer, perm as int32."""
    return _derived(prof, "rfr_profile", _rfr_profile_of)


def _rfr_profile_of(prof: RootProfile):
    r, c = prof.r, prof.c

    def lo(a, k):
        return np.zeros(k) if a is None else a

    buf = np.concatenate([prof.real_roots, lo(prof.real_lo, r), prof.pair_sums, lo(prof.sum_lo, c),
                          prof.pair_products, lo(prof.prod_lo, c)]).astype(np.float64, copy=False)
    perm = np.asarray(prof.perm, dtype=np.int32)
    base, pbase = buf.ctypes.data, perm.ctypes.data
    rp = _lib.RfrProfile(
        n=prof.n, r=r, c=c,
        real_hi=base, real_lo=base + 8 * r, sum_hi=base + 16 * r, sum_lo=base + 16 * r + 8 * c,
        prod_hi=base + 16 * r + 16 * c, prod_lo=base + 16 * r + 24 * c,
        perm=pbase, root_err=float(prof.root_err),
    )
    return rp, (buf, perm)


def verify_candidates(prof: RootProfile, p: IntPolynomial, pats: np.ndarray):
    """Device verification of candidate patterns (one warp each).
    Returns (verdict uint8[m], side uint8[m], coeffs int64[m, 65])."""
    lib = _lib.load()
    _lib.device()
    m = len(pats)
    verdict = np.zeros(m, dtype=np.uint8)
    side = np.zeros(m, dtype=np.uint8)
    coeffs = np.zeros((m, _STRIDE), dtype=np.int64)
    if m == 0:
        return verdict, side, coeffs
    rp, keep = _rfr_profile(prof)
    pats = np.ascontiguousarray(pats, dtype=np.uint64)
    pm = np.ascontiguousarray(_p_mod(p))
    _lib.check(
        lib.rfr_verify(ctypes.byref(rp), _lib.ptr(pats, _lib.U64_P), m,
                       _lib.ptr(pm, _lib.U64_P), p.degree,
                       verdict.ctypes.data_as(_lib.U8_P), side.ctypes.data_as(_lib.U8_P),
                       coeffs.ctypes.data_as(_lib.I64_P), _STRIDE, None),
        "rfr_verify",
    )
    return verdict, side, coeffs


def search_and_verify(prof: RootProfile, p: IntPolynomial, keys: np.ndarray, half_width: int,
                      keys3: np.ndarray, half_width3: int, stats=None):
    """One device call (rfr_search_verify): the key-window search, the third
    power-sum window and the verification of every survivor, without the
    candidates leaving the GPU in between.  Returns (pats, verdict, side,
    coeffs) like search_keys + verify_candidates (patterns unsorted)."""
    return _search_and_verify(prof, p, keys, half_width, keys3, half_width3, stats, False)[:4]


# Early termination (north star: "results are checked for early termination";
# SURVEY s8(e)): searches over n >= _EARLY_N entities verify their hits while
# the join runs and stop once one passes.  _PIECES: the library then searches
# the two pieces' pattern spaces in the same call (a complete candidate set);
# otherwise (or for pieces of >= 48 entities) factor() splits p and factors
# the pieces itself.  Smaller searches take ~0.1 ms and run whole.
_EARLY_N = 48
_PIECES = True


def _search_and_verify(prof: RootProfile, p: IntPolynomial, keys: np.ndarray, half_width: int,
                       keys3: np.ndarray, half_width3: int, stats, early_exit: bool,
                       max_rows: int | None = None, shard: int = 0, nshards: int = 1,
                       epoch: int = 0):
    """search_and_verify, optionally with early termination.  Returns (pats,
    verdict, side, coeffs, complete, stopped): stopped when the join ended at
    a verified hit; complete when the candidates nevertheless cover every
    factor pattern (the library searched the pieces), False when the pattern
    space was not exhausted."""
    from .recombine import _fill_stats, _window

    lib = _lib.load()
    _lib.device()
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    keys3 = np.ascontiguousarray(keys3, dtype=np.uint64)
    n = len(keys)
    lo, width = _window(half_width)
    lo2, width2 = _window(half_width3)
    rp, keep = _rfr_profile(prof)
    pm = np.ascontiguousarray(_p_mod(p))
    cap = 1 << 12  # a regrow reruns the whole search: start where the survivors fit
    while True:
        pats, verdict, side, coeffs, addr = _out_buffers(cap)
        nout = ctypes.c_int64(0)
        st = _lib.RfrStats()
        args = (keys.ctypes.data, n, lo, width, keys3.ctypes.data, lo2, width2,
                ctypes.byref(rp), pm.ctypes.data, p.degree, *addr, _STRIDE, cap,
                (1 if _PIECES else 2) if early_exit else 0)
        if nshards > 1:
            rc = lib.rfr_search_verify_shard(*args, shard, nshards, epoch, ctypes.byref(nout),
                                             ctypes.byref(st))
        else:
            rc = lib.rfr_search_verify(*args, ctypes.byref(nout), ctypes.byref(st))
        _lib.check(rc, "rfr_search_verify")
        if nout.value <= cap:
            break
        if max_rows is not None and nout.value > max_rows:
            raise RecombineDeviceError(f"{nout.value} raw hits exceed the flood limit {max_rows}")
        cap = int(nout.value)
    _fill_stats(stats, st)
    m = int(nout.value)
    complete = st.buckets >= st.buckets_planned
    # copies: the buffers are reused by the next call (the recursion on the
    # pieces makes one while the caller still holds these rows)
    return (pats[:m].copy(), verdict[:m].copy(), side[:m].copy(), coeffs[:m].copy(), complete,
            bool(st.early_stop))


_OUT: dict = {}


def _out_buffers(cap: int):
    """Result buffers of rfr_search_verify for cap rows (pats, verdict, side,
    coefficients) and their addresses, kept for reuse across calls."""
    b = _OUT.get(cap)
    if b is None:
        pats = np.empty(cap, dtype=np.uint64)
        verdict = np.empty(cap, dtype=np.uint8)
        side = np.empty(cap, dtype=np.uint8)
        coeffs = np.empty((cap, _STRIDE), dtype=np.int64)
        b = (pats, verdict, side, coeffs,
             (pats.ctypes.data, verdict.ctypes.data, side.ctypes.data, coeffs.ctypes.data))
        if len(_OUT) > 8:
            _OUT.clear()
        _OUT[cap] = b
    return b


def _sub_profile(prof: RootProfile, t: int) -> RootProfile:
    """The profile of the factor whose entities pattern t selects, without new
    root finding (the reference re-runs find_roots on each
    piece, R/verify.py:257): entities keep their double-double values and
    their keys in rho order; the key and root error bounds of the whole
    profile bound every subset sum."""
    bits = [i for i in range(prof.n) if (t >> i) & 1]
    ents = [prof.perm[i] for i in bits]
    reals = np.asarray(sorted(e for e in ents if e < prof.r), dtype=np.int64)
    pairs = np.asarray(sorted(e - prof.r for e in ents if e >= prof.r), dtype=np.int64)
    new_id = {int(e): j for j, e in enumerate(reals)}
    new_id.update({prof.r + int(e): len(reals) + j for j, e in enumerate(pairs)})
    idx = np.asarray(bits, dtype=np.int64)

    def take(a, sel):
        return None if a is None else np.asarray(a)[sel]

    return RootProfile(
        real_roots=prof.real_roots[reals], pair_sums=prof.pair_sums[pairs],
        pair_products=prof.pair_products[pairs], rho=prof.rho[idx],
        perm=tuple(new_id[e] for e in ents),
        real_lo=take(prof.real_lo, reals), sum_lo=take(prof.sum_lo, pairs),
        prod_lo=take(prof.prod_lo, pairs),
        keys1=take(prof.keys1, idx), keys2=take(prof.keys2, idx), keys3=take(prof.keys3, idx),
        key_err1=prof.key_err1, key_err2=prof.key_err2, key_err3=prof.key_err3,
        root_err=prof.root_err,
        hp_real=None if prof.hp_real is None else tuple(prof.hp_real[int(e)] for e in reals),
        hp_pair=None if prof.hp_pair is None else tuple(prof.hp_pair[int(e)] for e in pairs),
        hp_err=prof.hp_err,
    )


def _host_candidate(prof: RootProfile, p: IntPolynomial, t: int) -> IntPolynomial | None:
    """Exact-rational rebuild of the side t for candidates the device could
    not decide (coefficients beyond 2^62 or a loose error bound): multiply
    out the double-double entities as Fractions, round, bound the error,
    and demand exact division (R/verify.py:141-155 semantics)."""
    if prof.hp_real is not None:
        # multiprecision roots (~bits + 160 bits): their products round the
        # factor's coefficients even where double-double cannot (the monic
        # transform of a non-monic p); exact division is the proof
        coeffs = [Fraction(1)]
        for i in range(prof.n):
            if (t >> i) & 1:
                ent = prof.perm[i]
                if ent < prof.r:
                    coeffs = _pmul(coeffs, [-prof.hp_real[ent], Fraction(1)])
                else:
                    tt, mm = prof.hp_pair[ent - prof.r]
                    coeffs = _pmul(coeffs, [mm, -tt, Fraction(1)])
        q = IntPolynomial([round(c) for c in coeffs])
        if q.degree < 1 or not q.is_monic():
            return None
        return q if divide_exact(p, q) is not None else None
    coeffs = [Fraction(1)]
    mag = [1.0]
    magp = [1.0]
    de = prof.root_err
    for i in range(prof.n):
        if not (t >> i) & 1:
            continue
        ent = prof.perm[i]
        if ent < prof.r:
            u = Fraction(float(prof.real_roots[ent])) + Fraction(float(prof.real_lo[ent]))
            fac, fm, fp = [-u, Fraction(1)], [abs(float(u)), 1.0], [abs(float(u)) + de, 1.0]
        else:
            j = ent - prof.r
            tt = Fraction(float(prof.pair_sums[j])) + Fraction(float(prof.sum_lo[j]))
            mm = Fraction(float(prof.pair_products[j])) + Fraction(float(prof.prod_lo[j]))
            dm = 2 * abs(float(mm)) ** 0.5 * de + de * de
            fac = [mm, -tt, Fraction(1)]
            fm = [abs(float(mm)), abs(float(tt)), 1.0]
            fp = [abs(float(mm)) + dm, abs(float(tt)) + 2 * de, 1.0]
        coeffs = _pmul(coeffs, fac)
        mag = _pmul(mag, fm)
        magp = _pmul(magp, fp)
    out = []
    for c, a, b in zip(coeffs, mag, magp):
        r = round(c)
        bound = (b - a) + a * 1e-28 + 1e-30
        if abs(float(c - r)) > 2 * bound + 1e-12:
            return None
        out.append(int(r))
    q = IntPolynomial(out)
    if q.degree < 1 or not q.is_monic():
        return None
    return q if divide_exact(p, q) is not None else None


def _pmul(a, b):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _factor_cells(found: dict, p: IntPolynomial, full: int) -> list:
    """The irreducible factors as (entity pattern, polynomial) cells: the
    partition of the entities that the found factor patterns generate.
    found maps patterns to their (verified) factors of p.  Every irreducible
    factor's entities lie inside or outside each found pattern, and the
    candidate set (a whole search, or a stopped one plus its pieces'
    searches) separates any two of them.  A pattern inside a cell splits it
    by exact division; a partial overlap (rare) by a gcd.  After a stop the
    pieces' patterns only imply some factors (t minus a pattern inside t),
    which a greedy cover by minimal patterns would leave merged."""
    cells = [(full, p)]
    bad = []  # device PASSes the exact division refutes (the device test is a filter)
    for t in sorted(found, key=lambda x: (bin(x).count("1"), x)):
        q = found[t]
        refined = []
        for c, pc in cells:
            inter = c & t
            if inter == 0 or inter == c:
                refined.append((c, pc))
                continue
            if inter == t:  # the pattern lies inside the cell: pc = q * (pc / q)
                g, r = q, divide_exact(pc, q)
                if r is None:
                    bad.append(t)
            else:  # partial overlap: the common factor
                g = poly_gcd(pc, q)
                r = divide_exact(pc, g) if g.degree >= 1 else None
            if r is None or g.degree < 1 or r.degree < 1:
                refined.append((c, pc))
                continue
            refined += [(inter, g), (c & ~t, r)]
        cells = refined
    _factor_cells.bad = bad
    return cells


def _small_factors(prof: RootProfile, p: IntPolynomial) -> list:
    """((pattern,), factor) for factors made of 1 to 3 entities: every such
    entity subset whose combined keys lie inside both windows (vectorised over
    all pairs and triples of the <= 64 entities), rebuilt exactly and
    confirmed by division (smallest first; the caller keeps disjoint ones)."""
    n = prof.n
    keys, T = _search_window(prof)
    keys3, T3 = _secondary_window(prof)
    k1 = np.asarray(keys, dtype=np.uint64)
    k3 = np.asarray(keys3, dtype=np.uint64) if keys3 is not None else None
    TWO = np.uint64

    def close(s, t):
        d = np.minimum(s, (TWO(0) - s))
        return d <= TWO(min(t, (1 << 64) - 1))

    out = []
    # single entities first: a one-entity factor the exact screen above missed
    # must split off before any 2-3 entity union containing it (which would
    # otherwise be confirmed -- it divides p -- and reported as irreducible)
    ok1 = close(k1, T)
    if k3 is not None:
        ok1 &= close(k3, T3)
    cand = [1 << int(a) for a in np.flatnonzero(ok1)]
    i, j = np.triu_indices(n, 1)
    s1 = k1[i] + k1[j]
    ok = close(s1, T)
    if k3 is not None:
        ok &= close(k3[i] + k3[j], T3)
    cand += [((1 << int(a)) | (1 << int(b))) for a, b in zip(i[ok], j[ok])]
    if n <= 64:
        a, b = np.triu_indices(n, 1)
        for c in range(2, n):
            sel = b < c
            aa, bb = a[sel], b[sel]
            s = k1[aa] + k1[bb] + k1[c]
            ok = close(s, T)
            if k3 is not None:
                ok &= close(k3[aa] + k3[bb] + k3[c], T3)
            cand += [((1 << int(x)) | (1 << int(y)) | (1 << c)) for x, y in zip(aa[ok], bb[ok])]
    full = (1 << n) - 1
    for t in sorted(set(cand), key=lambda x: (bin(x).count("1"), x)):
        q = _host_candidate(prof, p, t)
        if q is not None:
            out.append(((t,), q))
    return out


def _single_entity_factors(prof: RootProfile, p: IntPolynomial) -> list:
    """(pattern bit, factor) for every entity that is a factor of p by itself:
    a real root that rounds to an integer r with p(r) = 0 (x - r), or a
    conjugate pair whose sum and product round to integers T, M with
    x^2 - T x + M dividing p (irreducible over Q: its roots are not real).
    Checked exactly; a cheap closeness test screens the rest.  The rounding
    uses the exact double-double value (hi + lo, or the multiprecision one):
    a value at or above 2^53 is not an integer in its high word alone."""
    # vectorised screen: only entities within 1e-6 of integral values are tested
    near_r, near_p = _derived(prof, "near_integral", _near_integral)
    if not len(near_r) and not len(near_p):
        return []
    ru = np.asarray(prof.real_roots, dtype=np.float64)
    pt = np.asarray(prof.pair_sums, dtype=np.float64)
    pm = np.asarray(prof.pair_products, dtype=np.float64)

    def exact(hi, lo, j):
        v = Fraction(float(hi[j]))
        if lo is not None:
            v += Fraction(float(lo[j]))
        return v

    bit_of = {ent: i for i, ent in enumerate(prof.perm)}
    out = []
    for ent in near_r:
        e = int(ent)
        u = prof.hp_real[e] if prof.hp_real is not None else exact(ru, prof.real_lo, e)
        r = round(u)
        acc = 0
        for c in reversed(p.coeffs):
            acc = acc * r + c
        if acc == 0:
            out.append((bit_of[e], IntPolynomial([-r, 1])))
    for j in near_p:
        j = int(j)
        if prof.hp_pair is not None:
            tt, mm = prof.hp_pair[j]
        else:
            tt, mm = exact(pt, prof.sum_lo, j), exact(pm, prof.prod_lo, j)
        q = IntPolynomial([round(mm), -round(tt), 1])
        if divide_exact(p, q) is not None:
            out.append((bit_of[prof.r + j], q))
    return out


def _near_integral(prof: RootProfile):
    """Indices of the real roots, and of the pairs (sum and product), within
    1e-6 (relative) of integers: the only one-entity factor candidates."""
    ru = np.asarray(prof.real_roots, dtype=np.float64)
    near_r = np.abs(ru - np.round(ru)) <= 1e-6 * np.maximum(1.0, np.abs(ru))
    pt = np.asarray(prof.pair_sums, dtype=np.float64)
    pm = np.asarray(prof.pair_products, dtype=np.float64)
    near_p = ((np.abs(pt - np.round(pt)) <= 1e-6 * np.maximum(1.0, np.abs(pt)))
              & (np.abs(pm - np.round(pm)) <= 1e-6 * np.maximum(1.0, np.abs(pm))))
    return np.flatnonzero(near_r), np.flatnonzero(near_p)


def _coeff_bits(p: IntPolynomial) -> int:
    co = p.coeffs
    return max(max(co), -min(co)).bit_length()


def _integer_roots(p: IntPolynomial, scan: bool) -> list:
    """Integer roots of a monic square-free p (its only rational roots),
    exactly: the rounded real parts of the float root seeds (and their
    neighbours), or with scan every integer within Fujiwara's root bound
    (when it is at most 10^4), prefiltered modulo 2^61 - 1."""
    from .rootfinder import _initial_roots

    cs = list(p.coeffs)
    d = len(cs) - 1
    cand = set()
    try:
        for z in _initial_roots(cs):
            if abs(z.imag) < 1.0 and abs(z.real) < 1e15:
                r = int(round(z.real))
                cand.update((r - 1, r, r + 1))
    except NonConvergence:
        pass
    if scan:
        # Fujiwara: every root has |z| <= 2 max_k |c_{d-k}|^(1/k)
        bound = 2.0 * max((abs(cs[d - k]) ** (1.0 / k) if cs[d - k] else 0.0) for k in range(1, d + 1))
        if bound <= 1e4:
            M = (1 << 61) - 1
            cm = [c % M for c in cs]
            for r in range(-int(bound) - 1, int(bound) + 2):
                acc = 0
                rm = r % M
                for c in reversed(cm):
                    acc = (acc * rm + c) % M
                if acc == 0:
                    cand.add(r)
    out = []
    for r in sorted(cand):
        acc = 0
        for c in reversed(cs):
            acc = acc * r + c
        if acc == 0:
            out.append(r)
    return out


# more survivors than this after the search: look for small multi-entity
# factors before processing them one by one
_FLOOD = 512


def _split_small_factors(p, prof, small, cfg, workers, stats, early_exit):
    """Divide the (disjoint, exactly confirmed) small factors out of p and
    factor the rest over its own entities; None when none applies."""
    t0 = time.perf_counter()
    rest, mask, out = p, 0, []
    for bits, q in small:  # bits: one entity's bit index, or (pattern,) for 2-3 entities
        pat = bits[0] if isinstance(bits, tuple) else (1 << bits)
        if pat & mask:
            continue  # overlaps a factor already split off
        r = divide_exact(rest, q)
        if r is None:
            continue
        rest = r
        mask |= pat
        out.append(q)
    stats.verify_seconds += time.perf_counter() - t0
    if not out:
        return None
    left = ((1 << prof.n) - 1) & ~mask
    if rest.degree >= 1:
        out += _factor_monic_squarefree(rest, cfg, workers, stats, _sub_profile(prof, left),
                                        early_exit)
    return out


def _factor_monic_squarefree(p: IntPolynomial, cfg: ToleranceConfig, workers: int,
                             stats: FactorStats, prof: RootProfile | None = None,
                             early_exit: bool = True) -> list[IntPolynomial]:
    """Irreducible factors of a monic square-free p.  prof: p's root profile
    when already known (a piece split off by an earlier search)."""
    if p.degree <= 1:
        return [p]
    if prof is None:
        t0 = time.perf_counter()
        # integer roots make the polish ill-conditioned (a Wilkinson-like
        # product of 39 of them did not converge): split them off exactly
        # before the multiprecision polish, and as a fallback if it fails
        ints = ([] if p.coeffs in _PROFILED
                else _integer_roots(p, scan=False) if _coeff_bits(p) > 100 else [])
        if not ints:
            try:
                prof = _profile_cached(p.coeffs)
                if len(_PROFILED) > 4096:
                    _PROFILED.clear()
                _PROFILED.add(p.coeffs)  # profiled without an integer-root split
            except NonConvergence:
                ints = _integer_roots(p, scan=True)
                if not ints:
                    raise
        stats.root_seconds += time.perf_counter() - t0
        if ints:
            rest = p
            for r in ints:
                rest = divide_exact(rest, IntPolynomial([-r, 1]))
            return [IntPolynomial([-r, 1]) for r in ints] + (
                _factor_monic_squarefree(rest, cfg, workers, stats, None, early_exit)
                if rest.degree >= 1 else [])
    n = prof.n
    if n > 1:
        # one-entity factors first: an integer root, or a conjugate pair with
        # integral t and m, divides p by itself -- and k of them would make
        # every one of their 2^k unions a hit of the search (35 linear
        # factors flooded it with 3e10 hits)
        split = _split_small_factors(p, prof, _single_entity_factors(prof, p), cfg, workers, stats,
                                     early_exit)
        if split is not None:
            return split
    stats.n = max(stats.n, n)

    t0 = time.perf_counter()
    keys, T = _search_window(prof)
    keys3, T3 = _secondary_window(prof)
    complete, stopped = True, False
    if keys3 is not None:
        # one device call: search, Tr3 window and verification back to back
        # (recombine_seconds then covers the device verification too); with
        # workers > 1 every rank runs its key-range shards this way, a rank's
        # verified factor stops the other ranks' joins, and the verified rows
        # are all-gathered (parallel.sharded_search_verify)
        if workers == 1:
            search = lambda limit: _search_and_verify(  # noqa: E731
                prof, p, keys, T, keys3, T3, stats.recombine, early_exit and n >= _EARLY_N, limit)
        else:
            from .parallel import sharded_search_verify

            search = lambda limit: sharded_search_verify(  # noqa: E731
                prof, p, keys, T, keys3, T3, workers, stats, early_exit and n >= _EARLY_N, limit)
        try:
            pats, verdict, side, coeffs, complete, stopped = search(1 << 16)
            flood = len(pats) > _FLOOD
        except RecombineDeviceError as e:
            if "raw hits exceed" not in str(e):
                raise
            flood, pats = True, None
        if flood and n > 3:
            # a flood of candidates: many small multi-entity factors (all 2^k
            # unions of k quadratics x^2 - a are hits) -- split them off first
            split = _split_small_factors(p, prof, _small_factors(prof, p), cfg, workers, stats,
                                         early_exit)
            if split is not None:
                return split
        if pats is None:  # no small factors behind the flood: take every candidate
            pats, verdict, side, coeffs, complete, stopped = search(None)
        stats.early_exits += int(stopped and complete)  # stopped, pieces searched in the call
        keep = pats != 0
        if not keep.all():  # the empty pattern, when it is a row
            pats, verdict, side, coeffs = pats[keep], verdict[keep], side[keep], coeffs[keep]
        stats.recombine_seconds += time.perf_counter() - t0
        stats.candidates += len(pats)
        t0 = time.perf_counter()
    else:
        if workers > 1:
            from .parallel import sharded_search_keys

            pats = sharded_search_keys(keys, T, workers, stats.recombine, keys2=keys3,
                                       half_width2=T3)
        else:
            pats = search_keys(keys, T, stats.recombine, keys2=keys3, half_width2=T3)
        pats = pats[pats != 0]
        stats.recombine_seconds += time.perf_counter() - t0
        stats.candidates += len(pats)
        t0 = time.perf_counter()
        verdict, side, coeffs = verify_candidates(prof, p, pats)
    full = (1 << n) - 1
    found: dict[int, IntPolynomial] = {}  # side pattern -> monic integer factor
    for k in range(len(pats)):
        s = int(pats[k])
        v = int(verdict[k])
        if v == _lib.V_PASS:
            t = (~s & full) if side[k] else s
            e = selected_degree(t, prof)
            found[t] = _poly(coeffs[k, : e + 1].tolist())
        elif v == _lib.V_HOST:
            stats.host_verified += 1
            for t in (s, ~s & full):
                q = _host_candidate(prof, p, t)
                if q is not None:
                    found[t] = q
                    break
            else:
                stats.rejected += 1
        else:
            stats.rejected += 1
    if not complete:
        # early exit: the searched chunks hold a verified factor q but the
        # pattern space was not exhausted, so q and p / q are factored in
        # turn, each over its own entities (no new root finding)
        for t in sorted(found, key=lambda x: (bin(x).count("1"), x)):
            q = found[t]
            rest = divide_exact(p, q)
            if rest is None:
                continue
            stats.verify_seconds += time.perf_counter() - t0
            stats.early_exits += 1
            return (_factor_monic_squarefree(q, cfg, workers, stats, _sub_profile(prof, t))
                    + _factor_monic_squarefree(rest, cfg, workers, stats,
                                               _sub_profile(prof, ~t & full)))
        # a device PASS the exact check rejects (not seen in practice): search
        # the whole space
        stats.verify_seconds += time.perf_counter() - t0
        return _factor_monic_squarefree(p, cfg, workers, stats, prof, early_exit=False)
    if not found:
        stats.verify_seconds += time.perf_counter() - t0
        return [p]
    cells = _factor_cells(found, p, full)
    if _factor_cells.bad:
        # a device PASS that exact division refutes: after a stop its pieces
        # were searched around a non-factor, so search the whole space; after
        # a whole search, drop it
        stats.verify_seconds += time.perf_counter() - t0
        if stopped:
            return _factor_monic_squarefree(p, cfg, workers, stats, prof, early_exit=False)
        for t in _factor_cells.bad:
            found.pop(t, None)
        cells = _factor_cells(found, p, full)
    if stopped and any(pc.degree != selected_degree(c, prof) for c, pc in cells):
        # inconsistent cells after a stopped search (not seen): search the whole space
        stats.verify_seconds += time.perf_counter() - t0
        return _factor_monic_squarefree(p, cfg, workers, stats, prof, early_exit=False)
    factors = [pc for _, pc in cells]
    stats.verify_seconds += time.perf_counter() - t0
    return factors


def factor(
    p: IntPolynomial,
    cfg: ToleranceConfig | None = None,
    backend: str = "e",
    workers: int = 1,
) -> FactorizationResult:
    """Full irreducible factorization over the integers (R/verify.py:187-233).
    ``workers`` > 1 shards the search over that many key ranges (GPUs when
    torch.distributed runs one rank per device).  ValueError on an unknown
    backend, workers < 1 or a constant polynomial."""
    cfg = cfg or ToleranceConfig()
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if p.is_constant():
        raise ValueError("factor requires a non-constant polynomial")
    stats = FactorStats(backend=backend, workers=workers)
    content = p.content()
    prim = p.primitive_part()
    out: list[tuple[IntPolynomial, int]] = []
    for part, mult in square_free_decompose(prim):
        if part.is_monic():
            irr = _factor_monic_squarefree(part, cfg, workers, stats)
        else:
            tr = monic_transform(part)
            irr = [monic_untransform_factor(g, part.leading)
                   for g in _factor_monic_squarefree(tr, cfg, workers, stats)]
        out.extend((g, mult) for g in irr)
    out.sort(key=lambda fm: (fm[0].degree, fm[0].coeffs, fm[1]))
    rebuilt = IntPolynomial([content])
    for g, m in out:
        rebuilt = rebuilt * g**m
    return FactorizationResult(input=p, content=content, factors=tuple(out),
                               certificate=(rebuilt == p), stats=stats)


def is_irreducible(p: IntPolynomial, cfg: ToleranceConfig | None = None,
                   backend: str = "e") -> bool:
    """True when the primitive part of p does not split (R/verify.py:289-297)."""
    if p.is_constant():
        raise ValueError("irreducibility is asked of non-constant polynomials")
    if p.degree == 1:
        return True
    return factor(p, cfg, backend).irreducible
