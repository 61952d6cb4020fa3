"""The reference's factor() path on host threads -- BASELINE INFRASTRUCTURE.

Only bench.py (the ``--impl reference`` arm and the ``cpu_baseline`` leg) and
tests/ use this module; the product package never imports it.

``factor_port`` replays ``_factor_monic_squarefree`` of the reference
(/root/reference/pkg/src/polyfactor/verify.py:246-286, "R/" below) on the
reference's OWN root profiles (frozen by tests/golden/make_ref_c3.py, since
the reference cannot run on the GPU box), with the search and the
verification loop in C threads (oracle/ref_arm.c):

  cands   = parallel_recombine_e(rho, eps, workers)      R/parallel.py:255-272
  ordered = sorted(nontrivial, key=(degree, s))           R/verify.py:267
  first survivor of build_candidate / trace_test /
    round_and_divide, then recursion on q and p / q       R/verify.py:270-284

Root finding is excluded exactly as the GPU arm excludes it (the reference's
own split: FactorStats.root_seconds, R/verify.py:256-258): the profiles come
precomputed, as the GPU arm's come from its cache.
"""
from __future__ import annotations

import ctypes
import time

import numpy as np

from . import recombine_oracle as O


def _lib():
    L = O.lib()
    if not hasattr(L, "_ref_arm_ready"):
        d_p = ctypes.POINTER(ctypes.c_double)
        u64_p = ctypes.POINTER(ctypes.c_uint64)
        i64_p = ctypes.POINTER(ctypes.c_int64)
        i32_p = ctypes.POINTER(ctypes.c_int)
        L.orc_par_recombine_e.restype = ctypes.c_int64
        L.orc_par_recombine_e.argtypes = [d_p, ctypes.c_int, ctypes.c_double, ctypes.c_int, u64_p,
                                          ctypes.c_int64, i64_p]
        L.orc_order_candidates.restype = ctypes.c_int64
        L.orc_order_candidates.argtypes = [u64_p, ctypes.c_int64, i32_p, ctypes.c_int, ctypes.c_int]
        L.orc_verify_first.restype = ctypes.c_int64
        L.orc_verify_first.argtypes = [u64_p, ctypes.c_int64, ctypes.c_int64, d_p, ctypes.c_int, d_p,
                                       d_p, ctypes.c_int, i32_p, ctypes.c_int, i64_p, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_int, i64_p, i32_p, i32_p]
        L._ref_arm_ready = True
    return L


def _p(a, typ):
    return a.ctypes.data_as(ctypes.POINTER(typ))


def par_recombine_e(rho, eps: float, threads: int = 0):
    """parallel_recombine_e(rho, eps, workers=threads) (R/parallel.py:255-272):
    the sorted canonical candidate set (uint64) and the counters."""
    L = _lib()
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    n = len(rho)
    if n < 2:
        return np.array(sorted(O.canonical_set(rho, eps)), dtype=np.uint64), {}
    st = np.zeros(10, dtype=np.int64)
    cap = 1 << 20
    while True:
        out = np.zeros(cap, dtype=np.uint64)
        m = L.orc_par_recombine_e(_p(rho, ctypes.c_double), n, eps, threads, _p(out, ctypes.c_uint64),
                                  cap, _p(st, ctypes.c_int64))
        if m == -1:
            raise MemoryError("orc_par_recombine_e: allocation failure")
        if m == -2:
            raise RuntimeError("lost insertion detected")  # R/parallel.py:186
        if m <= cap:
            break
        cap = int(m)
    stats = dict(inserts=int(st[0]), insert_probes=int(st[1]), queries=int(st[2]),
                 query_probes=int(st[3]), raw=int(st[4]), sums_s=st[5] * 1e-9, build_s=st[6] * 1e-9,
                 query_s=st[7] * 1e-9, filter_s=st[8] * 1e-9, total_s=st[9] * 1e-9)
    return out[:m].copy(), stats


class Profile:
    """The reference's RootProfile fields the path reads (R/rootfinder.py:58-84)."""

    def __init__(self, d):
        h = lambda xs: np.array([float.fromhex(x) for x in xs], dtype=np.float64)  # noqa: E731
        self.real_roots = h(d["real_roots"])
        self.pair_sums = h(d["pair_sums"])
        self.pair_products = h(d["pair_products"])
        self.rho = h(d["rho"])
        self.perm = np.array(d["perm"], dtype=np.int32)
        self.r, self.c, self.n = len(self.real_roots), len(self.pair_sums), len(self.rho)


def verify_first(prof: Profile, pats: np.ndarray, p_coeffs, eps: float, threads: int = 0,
                 start: int = 0):
    """First survivor of R/verify.py:270-284 over the ordered pats[start:]:
    (index, q coefficients or None, status).  status 2: the exact division
    left int128 -- decided by the caller with bigints."""
    L = _lib()
    p = np.array([int(c) for c in p_coeffs], dtype=np.int64)
    q = np.zeros(260, dtype=np.int64)
    deg = ctypes.c_int(0)
    status = ctypes.c_int(0)
    idx = L.orc_verify_first(_p(pats, ctypes.c_uint64), start, len(pats),
                             _p(prof.real_roots, ctypes.c_double), prof.r,
                             _p(prof.pair_sums, ctypes.c_double), _p(prof.pair_products, ctypes.c_double),
                             prof.c, _p(prof.perm, ctypes.c_int), prof.n, _p(p, ctypes.c_int64),
                             len(p) - 1, eps, threads, _p(q, ctypes.c_int64), ctypes.byref(deg),
                             ctypes.byref(status))
    if idx < 0:
        raise MemoryError("orc_verify_first")
    if status.value == 1:
        return int(idx), [int(v) for v in q[: deg.value + 1]], 1
    return int(idx), None, status.value


def _round_and_divide_exact(prof: Profile, s: int, p_coeffs, eps: float):
    """round_and_divide for one candidate with Python bigints (the rare
    quotient beyond int128): R/verify.py:141-155 via the numpy longdouble
    restatement."""
    ok, q = O.verify_candidate(s, {"real_roots": prof.real_roots, "pair_sums": prof.pair_sums,
                                   "pair_products": prof.pair_products, "perm": prof.perm},
                               p_coeffs, eps)
    return q if ok else None


def factor_port(p_coeffs, profiles: dict, eps: float, threads: int = 0, stats: dict | None = None):
    """_factor_monic_squarefree (R/verify.py:246-286) of a monic square-free
    p (coefficients low -> high), with every piece's reference profile looked
    up in `profiles` (tuple(coeffs) -> profile dict).  Returns the factors
    (coefficient lists) in the reference's recursion order."""
    st = stats if stats is not None else {}
    for k in ("candidates", "rejected", "search_s", "verify_s"):
        st.setdefault(k, 0)
    p_coeffs = [int(c) for c in p_coeffs]
    if len(p_coeffs) - 1 <= 1:
        return [p_coeffs]
    prof = Profile(profiles[tuple(p_coeffs)])
    t0 = time.perf_counter()
    cands, _ = par_recombine_e(prof.rho, eps, threads)
    m = _lib().orc_order_candidates(_p(cands, ctypes.c_uint64), len(cands), _p(prof.perm, ctypes.c_int),
                                    prof.r, prof.n)
    ordered = cands[:m]
    st["candidates"] += int(m)
    t1 = time.perf_counter()
    st["search_s"] += t1 - t0
    start = 0
    while True:
        idx, q, status = verify_first(prof, ordered, p_coeffs, eps, threads, start)
        if status == 2:  # decided with bigints, then resume after it
            q = _round_and_divide_exact(prof, int(ordered[idx]), p_coeffs, eps)
        if q is None:
            st["rejected"] += idx - start + (1 if status == 2 else 0)
            if status == 2:
                start = idx + 1
                continue
            st["verify_s"] += time.perf_counter() - t1
            return [p_coeffs]
        st["rejected"] += idx - start
        rest = O.divide_exact(p_coeffs, q)
        st["verify_s"] += time.perf_counter() - t1
        return (factor_port(q, profiles, eps, threads, st)
                + factor_port(rest, profiles, eps, threads, st))
