"""Randomised factor() sweep against sympy.factor_list (needs a GPU):
products of 1-4 random factors (degrees summing to 20-110, coefficients up to
10^3, non-monic and negative leads, squares, content).

    python tools/sweep_random.py <seed> <cases>     # prints mismatches and "bad k of n"

The GPU suite runs a 24-case version (tests/test_gpu_factor.py).
"""
import random, signal, sys, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class _Timeout(Exception):
    pass


def _alarm(*_):
    raise _Timeout()


signal.signal(signal.SIGALRM, _alarm)
import sympy
from paper_2410_15880_b200 import IntPolynomial as P, factor
x = sympy.symbols("x")
seed0 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ncases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bad = 0
t_all = time.time()
for case in range(ncases):
    rng = random.Random(seed0 * 1000 + case)
    k = rng.choice([1, 2, 2, 3, 4])
    total = rng.choice([20, 40, 60, 80, 100, 110])
    degs = []
    rem = total
    for i in range(k - 1):
        d = rng.randint(1, max(1, rem - (k - 1 - i)))
        d = max(1, min(d, rem - (k - 1 - i)))
        degs.append(d); rem -= d
    degs.append(max(1, rem))
    cmax = rng.choice([1, 3, 10, 100, 1000])
    prod = sympy.Poly(rng.choice([1, 1, 1, -1, 2, 6]), x)
    used = []
    for i, d in enumerate(degs):
        lead = rng.choice([1, 1, 1, -1, 2, 3, 5]) if rng.random() < 0.3 else 1
        co = [rng.randint(-cmax, cmax) for _ in range(d)] + [lead]
        if co[0] == 0:
            co[0] = 1
        f = sympy.Poly(list(reversed(co)), x)
        mult = 2 if rng.random() < 0.15 else 1
        prod = prod * f ** mult
    if prod.degree() < 1 or prod.degree() > 128:
        continue
    p = P([int(c) for c in reversed(prod.all_coeffs())])
    want_c, want_f = sympy.factor_list(prod.as_expr(), x)
    want = sorted(([int(c) for c in reversed(sympy.Poly(f, x).all_coeffs())], m) for f, m in want_f)
    # normalise sympy's sign convention: leading coefficient positive
    norm = []
    for co, m in want:
        if co[-1] < 0:
            co = [-c for c in co]
        norm.append((co, m))
    want = sorted(norm)
    t0 = time.time()
    signal.alarm(60)
    res = None
    try:
        res = factor(p)
        got = sorted((list(g.coeffs), m) for g, m in res.factors)
        ok = got == want and res.certificate
    except _Timeout:
        ok, got = False, "TIMEOUT"
    except Exception as e:
        ok = False
        got = repr(e)[:200]
    signal.alarm(0)
    dt = time.time() - t0
    if not ok:
        bad += 1
        print(f"case {seed0}/{case}: degs {degs} cmax {cmax} deg {prod.degree()} MISMATCH ({dt:.2f}s) {got if res is None else ''}", flush=True)
        try:
            if res is None:
                raise ValueError("no result")
            wantset = set(tuple(c) for c, _ in want)
            for g, m in res.factors:
                print("    got deg", g.degree, "mult", m, "ok" if tuple(g.coeffs) in wantset else "NOT IN SYMPY", "cert", res.certificate,
                      "n", res.stats.n, "cands", res.stats.candidates, "exits", res.stats.early_exits, "hostv", res.stats.host_verified)
            print("    want degs", sorted((len(c) - 1, m) for c, m in want))
        except Exception as e:
            print("    ", repr(e)[:200])
    else:
        print(f"case {seed0}/{case}: ok deg {prod.degree()} k {k} n {res.stats.n} exits {res.stats.early_exits} {dt:.2f}s", flush=True)
print("bad", bad, "of", ncases, f"total {time.time()-t_all:.1f}s")
