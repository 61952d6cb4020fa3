"""CPU oracle for the recombination hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module, and only as the checker (or the
timed CPU baseline).  The product package ``paper_2410_15880_b200`` never
imports it and has no CPU fallback.

Restates the reference (``/root/reference/pkg/src/polyfactor``, "R/") in
plain Python/numpy, plus ctypes bindings to the C restatement in
``oracle/rfr_oracle.c`` (built into ``oracle/liborc.so`` by ``make -C
oracle`` or ``__graft_entry__.build()``).  Pinned against the reference's
own outputs frozen in ``tests/golden/*.json`` (see tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import math
import os
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GUARD = 1e-12  # R/recombine.py:28-30


# ------------------------------------------------------ pure restatements
def value(s: int, vals) -> float:
    """R/recombine.py:106-118: frac of the ascending-index float64 sum."""
    x = 0.0
    i = 0
    while s:
        if s & 1:
            x += float(vals[i])
        s >>= 1
        i += 1
    return x - math.floor(x)


def accept(y: float, eps: float) -> bool:
    """R/recombine.py:121-123 (strict)."""
    return y < eps or (1.0 - y) < eps


def canonical_set(vals, eps: float) -> frozenset:
    """The set every reference backend returns (R/recombine.py:148-195):
    canonical patterns t < 2^(n-1) with accept(value(t), eps).  Exhaustive;
    small n only."""
    n = len(vals)
    if n == 0:
        return frozenset()
    vals = [float(v) for v in vals]
    return frozenset(t for t in range(1 << (n - 1)) if accept(value(t, vals), eps))


def rho_keys(vals) -> np.ndarray:
    """Exact fixed-point keys round(rho * 2^64) mod 2^64 (the reference's own
    fixed-point idea, R/recombine.py:828-862, at M = 2^64, round to nearest)."""
    out = np.zeros(len(vals), dtype=np.uint64)
    for i, v in enumerate(vals):
        q = Fraction(float(v)) * (1 << 64)
        k = math.floor(q + Fraction(1, 2))
        out[i] = k % (1 << 64)
    return out


def key_window_py(keys, lo: int, width: int) -> frozenset:
    """Exhaustive uint64 window search (small n): t < 2^(n-1) with
    (sum_{i in t} keys[i] - lo) mod 2^64 <= width."""
    n = len(keys)
    if n == 0:
        return frozenset()
    ks = [int(k) for k in keys]
    out = set()
    for t in range(1 << (n - 1)):
        s = 0
        i = 0
        u = t
        while u:
            if u & 1:
                s += ks[i]
            u >>= 1
            i += 1
        if (s - lo) % (1 << 64) <= width:
            out.add(t)
    return frozenset(out)


# ------------------------------------------------------------- C oracle
_LIB = None


def lib():
    """ctypes handle to oracle/liborc.so (built on demand)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(HERE, "liborc.so")
    src = os.path.join(HERE, "rfr_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        rc = os.system(f"make -s -C {HERE} liborc.so >/dev/null 2>&1")
        if rc != 0 or not os.path.exists(path):
            raise RuntimeError("could not build oracle/liborc.so")
    L = ctypes.CDLL(path)
    d_p = ctypes.POINTER(ctypes.c_double)
    u64_p = ctypes.POINTER(ctypes.c_uint64)
    i64_p = ctypes.POINTER(ctypes.c_int64)
    L.orc_value.restype = ctypes.c_double
    L.orc_value.argtypes = [d_p, ctypes.c_int, ctypes.c_uint64]
    L.orc_accept.restype = ctypes.c_int
    L.orc_accept.argtypes = [ctypes.c_double, ctypes.c_double]
    L.orc_recombine.restype = ctypes.c_int64
    L.orc_recombine.argtypes = [d_p, ctypes.c_int, ctypes.c_double, u64_p, ctypes.c_int64]
    L.orc_key_window.restype = ctypes.c_int64
    L.orc_key_window.argtypes = [
        u64_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, u64_p, ctypes.c_int64
    ]
    L.orc_recombine_e_port.restype = ctypes.c_int64
    L.orc_recombine_e_port.argtypes = [
        d_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_int64, u64_p,
        ctypes.c_int64, i64_p,
    ]
    L.orc_num_threads.restype = ctypes.c_int
    L.orc_set_threads.argtypes = [ctypes.c_int]
    L.orc_divide_exact_i128.restype = ctypes.c_int
    L.orc_divide_exact_i128.argtypes = [i64_p, ctypes.c_int, i64_p, ctypes.c_int, i64_p]
    _LIB = L
    return L


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def c_recombine(vals, eps: float) -> frozenset:
    """Backend-a candidate set from the C restatement (n <= 40)."""
    rho = np.ascontiguousarray(vals, dtype=np.float64)
    n = len(rho)
    cap = 1 << 12
    while True:
        out = np.zeros(cap, dtype=np.uint64)
        cnt = lib().orc_recombine(_dp(rho), n, eps, _u64p(out), cap)
        if cnt < 0:
            raise RuntimeError(f"orc_recombine failed ({cnt})")
        if cnt <= cap:
            return frozenset(int(v) for v in out[:cnt])
        cap = int(cnt)


def c_key_window(keys, lo: int, width: int) -> np.ndarray:
    """Sorted patterns of the exhaustive uint64 window search (n <= 36)."""
    ks = np.ascontiguousarray(keys, dtype=np.uint64)
    n = len(ks)
    cap = 1 << 12
    while True:
        out = np.zeros(cap, dtype=np.uint64)
        cnt = lib().orc_key_window(_u64p(ks), n, lo % (1 << 64), width, _u64p(out), cap)
        if cnt < 0:
            raise RuntimeError(f"orc_key_window failed ({cnt})")
        if cnt <= cap:
            return out[:cnt].copy()
        cap = int(cnt)


def c_recombine_e_port(vals, eps: float, q_lo: int = 0, q_hi: int | None = None):
    """Raw hits of the backend-e port (splat + stream) and its counters.
    Returns (raw uint64 array, stats dict)."""
    rho = np.ascontiguousarray(vals, dtype=np.float64)
    n = len(rho)
    na = n // 2
    if q_hi is None:
        q_hi = 1 << na
    st = np.zeros(6, dtype=np.int64)
    cap = 1 << 16
    while True:
        out = np.zeros(cap, dtype=np.uint64)
        cnt = lib().orc_recombine_e_port(
            _dp(rho), n, eps, q_lo, q_hi, _u64p(out), cap,
            st.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        )
        if cnt < 0:
            raise RuntimeError("orc_recombine_e_port: allocation failure")
        if cnt <= cap:
            stats = dict(inserts=int(st[0]), insert_probes=int(st[1]),
                         queries=int(st[2]), query_probes=int(st[3]),
                         splat_s=st[4] * 1e-9, query_s=st[5] * 1e-9)
            return out[:cnt].copy(), stats
        cap = max(cap * 4, int(cnt))


def canonical_filter(raw, vals, eps: float) -> frozenset:
    """R/recombine.py:148-162."""
    n = len(vals)
    full = (1 << n) - 1
    vl = [float(v) for v in vals]
    out = set()
    for s in raw:
        s = int(s)
        t = min(s, s ^ full)
        if t in out:
            continue
        if accept(value(t, vl), eps):
            out.add(t)
    return frozenset(out)


def recombine_e_port(vals, eps: float) -> frozenset:
    """Backend e end to end on the CPU port: splat/stream + canonical filter
    (R/recombine.py:727-775)."""
    n = len(vals)
    if n == 0:
        return frozenset()
    if n < 2:
        return canonical_set(vals, eps)
    raw, _ = c_recombine_e_port(vals, eps)
    return canonical_filter(raw, vals, eps)


# --------------------------------------------------- verification oracle
def build_candidate(s: int, real_roots, pair_sums, pair_products, perm):
    """R/verify.py:60-120 in numpy.longdouble: (coeffs, traces, scales)."""
    ld = np.longdouble
    r = len(real_roots)
    reals, pairs = [], []
    i = 0
    t = s
    while t:
        if t & 1:
            ent = perm[i]
            if ent < r:
                reals.append(ld(real_roots[ent]))
            else:
                pairs.append((ld(pair_sums[ent - r]), ld(pair_products[ent - r])))
        t >>= 1
        i += 1
    coeffs = np.array([1.0], dtype=ld)
    for u in reals:
        ext = np.zeros(len(coeffs) + 1, dtype=ld)
        ext[1:] += coeffs
        ext[:-1] -= u * coeffs
        coeffs = ext
    for ps, pp in pairs:
        ext = np.zeros(len(coeffs) + 2, dtype=ld)
        ext[2:] += coeffs
        ext[1:-1] -= ps * coeffs
        ext[:-2] += pp * coeffs
        coeffs = ext
    e = len(coeffs) - 1
    traces = np.zeros(e, dtype=ld)
    scales = np.zeros(e, dtype=ld)
    upow = list(reals)
    uabs = [abs(u) for u in reals]
    pstate = [(ld(2.0), ps) for ps, _ in pairs]
    pmag = [ld(2.0) * np.sqrt(pp) for _, pp in pairs]
    for m in range(1, e + 1):
        tr = ld(0.0)
        sc = ld(0.0)
        for idx in range(len(reals)):
            tr += upow[idx]
            sc += uabs[idx]
        for idx in range(len(pairs)):
            tr += pstate[idx][1]
            sc += pmag[idx]
        traces[m - 1] = tr
        scales[m - 1] = sc
        if m < e:
            for idx in range(len(reals)):
                upow[idx] *= reals[idx]
                uabs[idx] *= abs(reals[idx])
            for idx, (ps, pp) in enumerate(pairs):
                prev, cur = pstate[idx]
                pstate[idx] = (cur, ps * cur - pp * prev)
                pmag[idx] *= np.sqrt(pp)
    return coeffs, traces, scales


def trace_test(traces, scales, eps: float) -> bool:
    """R/verify.py:123-138."""
    for m0 in range(len(traces)):
        m = m0 + 1
        scale = float(scales[m0])
        if m * scale * 1e-11 >= eps or scale >= (1 << 62):
            continue
        tr = traces[m0]
        if abs(float(tr - np.rint(tr))) >= eps:
            return False
    return True


def divide_exact(p, q):
    """R/polynomial.py:155-183 on Python ints (coefficient lists, low->high)."""
    p = list(p)
    q = list(q)
    while len(q) > 1 and q[-1] == 0:
        q.pop()
    if all(c == 0 for c in p):
        return [0]
    dp, dq = len(p) - 1, len(q) - 1
    if dp < dq:
        return None
    lq = q[-1]
    rem = list(p)
    quot = [0] * (dp - dq + 1)
    for k in range(dp - dq, -1, -1):
        num = rem[k + dq]
        if num == 0:
            continue
        if num % lq:
            return None
        t = num // lq
        quot[k] = t
        for i, qc in enumerate(q):
            rem[k + i] -= t * qc
    if any(rem):
        return None
    return quot


def round_and_divide(coeffs, p, eps: float):
    """R/verify.py:141-155: rounded integer coefficients or None."""
    rounded = []
    for c in coeffs:
        r = np.rint(c)
        if abs(float(c - r)) > eps:
            return None
        if abs(float(r)) >= (1 << 62):
            return None
        rounded.append(int(r))
    while len(rounded) > 1 and rounded[-1] == 0:
        rounded.pop()
    if len(rounded) - 1 < 1:
        return None
    return rounded if divide_exact(p, rounded) is not None else None


def verify_candidate(s: int, profile: dict, p, eps: float):
    """build_candidate -> trace_test -> round_and_divide for one pattern.
    Returns (trace_ok, q or None)."""
    coeffs, traces, scales = build_candidate(
        s, profile["real_roots"], profile["pair_sums"], profile["pair_products"], profile["perm"]
    )
    if not trace_test(traces, scales, eps):
        return False, None
    return True, round_and_divide(coeffs, p, eps)
