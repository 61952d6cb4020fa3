"""Structured factor() sweep against sympy.factor_list (needs a GPU): many
small factors, x^n -+ 1 / x^n - 2, small Swinnerton-Dyer products, cubed
factors, many integer roots, 10^6-sized coefficients; 60 s per case at most.

    python tools/sweep_structured.py <seed> <cases>

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
from paper_2410_15880_b200 import IntPolynomial as P, factor, gen_swinnerton_dyer
x = sympy.symbols("x")
seed0 = int(sys.argv[1]); ncases = int(sys.argv[2])
bad = 0
for case in range(ncases):
    rng = random.Random(77000 + seed0 * 1000 + case)
    mode = rng.choice(["many_small", "cyclo", "sd", "mult3", "real", "bigcoef"])
    if mode == "many_small":
        prod = sympy.Poly(1, x)
        for _ in range(rng.randint(4, 12)):
            d = rng.randint(1, 6)
            co = [rng.randint(-9, 9) for _ in range(d)] + [rng.choice([1, 1, 1, 2, -1])]
            if co[0] == 0: co[0] = 1
            prod *= sympy.Poly(list(reversed(co)), x)
    elif mode == "cyclo":
        n = rng.randint(2, 110)
        prod = sympy.Poly(x ** n - rng.choice([1, -1, 2]), x)
    elif mode == "sd":
        k = rng.randint(2, 5)
        sd = gen_swinnerton_dyer(k)
        prod = sympy.Poly(list(reversed([int(c) for c in sd.coeffs])), x)
        if rng.random() < 0.5 and 2 ** k <= 60:
            co = [rng.randint(-9, 9) for _ in range(rng.randint(2, 30))] + [1]
            prod *= sympy.Poly(list(reversed(co)), x)
    elif mode == "mult3":
        co = [rng.randint(-20, 20) for _ in range(rng.randint(2, 20))] + [1]
        f = sympy.Poly(list(reversed(co)), x)
        co2 = [rng.randint(-20, 20) for _ in range(rng.randint(2, 30))] + [1]
        prod = f ** 3 * sympy.Poly(list(reversed(co2)), x)
    elif mode == "real":
        roots = rng.sample(range(-60, 60), rng.randint(5, 40))
        prod = sympy.Poly(1, x)
        for r in roots:
            prod *= sympy.Poly(x - r, x)
        co = [rng.randint(-9, 9) for _ in range(rng.randint(2, 40))] + [1]
        prod *= sympy.Poly(list(reversed(co)), x)
    else:
        prod = sympy.Poly(1, x)
        for _ in range(rng.randint(2, 3)):
            d = rng.randint(5, 40)
            co = [rng.randint(-10**6, 10**6) for _ in range(d)] + [1]
            prod *= sympy.Poly(list(reversed(co)), x)
    if prod.degree() < 1 or prod.degree() > 128:
        continue
    p = P([int(c) for c in reversed(prod.all_coeffs())])
    want = []
    for f, m in sympy.factor_list(prod.as_expr(), x)[1]:
        co = [int(c) for c in reversed(sympy.Poly(f, x).all_coeffs())]
        want.append(([-c for c in co] if co[-1] < 0 else co, m))
    want = sorted(want)
    t0 = time.time()
    signal.alarm(60)
    try:
        res = factor(p)
        got = sorted((list(g.coeffs), m) for g, m in res.factors)
        ok = got == want and res.certificate
        info = f"n {res.stats.n} exits {res.stats.early_exits}"
    except _Timeout:
        ok, got, info = False, None, "TIMEOUT 60s"
    except Exception as e:
        ok, got, info = False, None, repr(e)[:160]
    signal.alarm(0)
    if not ok:
        bad += 1
        print(f"case {seed0}/{case} {mode} deg {prod.degree()} MISMATCH {info} ({time.time()-t0:.2f}s)", flush=True)
        if got is not None:
            print("    got degs", sorted((len(c) - 1, m) for c, m in got), "want degs", sorted((len(c) - 1, m) for c, m in want))
print("bad", bad, "of", ncases)
