"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package (`polyfactor`, /root/reference/pkg/src) in this container.

The reference is pure Python + numpy (+ numba); it cannot travel to the GPU
box, so its outputs are frozen here as small JSON files and the GPU tests,
smoke() and bench.py read only those files.

Run (this container only):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

What is frozen, and the reference code that produced it:
  recombine_cases.json  rho vectors (float hex) -> recombine_e(rho, eps).patterns
                        (pkg/src/polyfactor/recombine.py:727-775), each also
                        checked equal to recombine_a (:169-195), the oracle
                        backend; recipes follow pkg/tests/test_recombine.py
                        and pkg/tests/test_acceptance.py:36-57.
  factor_cases.json     factor(p) tuples (pkg/src/polyfactor/verify.py:187-233)
                        for the KATs of pkg/tests/test_verify.py:115-192, the
                        acceptance round trips (test_acceptance.py:60-75), C1
                        and C2 of BASELINE.json.
  verify_cases.json     per-candidate verdicts of build_candidate / trace_test /
                        round_and_divide (verify.py:60-155) on reference
                        profiles (rootfinder.py:204-245) of C1 inputs.
  big_inputs.json       C3 (gen_random_reducible_parts(100, 100, seed),
                        polynomial.py:311-345), C4 (random irreducible degree
                        120) and C5 (gen_swinnerton_dyer(6), polynomial.py:269)
                        with their factorizations: C3 by construction (halves
                        certified irreducible by the reference's own
                        is_irreducible), C4/C5 certified by sympy.factor_list
                        (the reference cannot run them: WidthExceeded /
                        NonConvergence).
"""
from __future__ import annotations

import json
import math
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))

import numpy as np  # noqa: E402

from polyfactor import (  # noqa: E402
    IntPolynomial,
    ToleranceConfig,
    build_candidate,
    factor,
    gen_random_reducible_parts,
    gen_swinnerton_dyer,
    is_irreducible,
    profile_polynomial,
    round_and_divide,
    trace_test,
)
from polyfactor.recombine import RhoVector, recombine_a, recombine_e  # noqa: E402


def fhex(v) -> str:
    return float(v).hex()


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def poly_json(p: IntPolynomial):
    return [str(c) for c in p.coeffs]  # strings: C5 coefficients exceed 64 bits


def result_json(res):
    return {
        "content": str(res.content),
        "factors": [[poly_json(g), m] for g, m in res.factors],
        "certificate": bool(res.certificate),
        "irreducible": bool(res.irreducible),
    }


# ---------------------------------------------------------------- recombine
def recombine_cases():
    cases = []

    def add(vals, eps, tag):
        rho = RhoVector.from_values(vals)
        got = recombine_e(rho, eps).patterns
        if len(rho) <= 30:
            assert got == recombine_a(rho, eps).patterns, tag
        cases.append(
            {
                "tag": tag,
                "eps": eps,
                "rho": [fhex(v) for v in rho.values],
                "patterns": sorted(int(s) for s in got),
            }
        )

    # KATs (test_recombine.py:61-89, :436-438)
    add([0.3, 0.7, 0.5], 1e-6, "kat_a_small")
    add([0.25, 0.75], 1e-6, "kat_quarter")
    add([0.5, 0.5], 1e-6, "kat_half_pair")
    add([], 1e-6, "empty")
    add([0.6], 1e-6, "single")
    add([0.0], 1e-6, "single_zero")
    add([0.0, 0.0, 0.0], 1e-6, "all_zero")
    add([0.9956, 0.97, 0.93, 0.9, 0.6, 0.55, 0.5, 0.0007], 1e-3, "wrap_crowd")
    add([1.0 - 1e-7, 1e-7, 0.5, 0.5], 1e-6, "near_one")
    # acceptance-1 recipe (test_acceptance.py:40-57), 12 vectors per width
    for n in (8, 12, 16, 20, 24):
        rng = random.Random(1000 + n)
        for i in range(12):
            vals = sorted(rng.random() for _ in range(n))
            add(vals, 1e-6, f"ac1_n{n}_{i}")
    # meet-in-middle recipe (test_recombine.py:426-433)
    rng = random.Random(16)
    for i in range(8):
        n = rng.randint(6, 18)
        add(sorted(rng.random() for _ in range(n)), 1e-6, f"mim_{i}")
    # other tolerances, unsorted inputs, every small width
    rng = random.Random(4242)
    for n in range(1, 27):
        for eps in (1e-3, 1e-4, 1e-6, 1e-9):
            if n > 22 and eps == 1e-3:
                continue
            vals = [rng.random() for _ in range(n)]
            if n % 3 == 0:
                vals.sort()
            add(vals, eps, f"w{n}_eps{eps:g}")
    # heavy duplicates (all-equal worst case of demos/03_splat_and_probes.py)
    add([0.25] * 12, 1e-6, "dup_quarter")
    add([0.125] * 16, 1e-6, "dup_eighth")
    add([1.0 / 3.0] * 15, 1e-6, "dup_third")
    add([0.1, 0.2, 0.3, 0.4] * 4, 1e-9, "dup_tenths")
    # a real profile (complement symmetric): test_recombine.py:448-460
    from polyfactor.polynomial import gen_random_reducible

    for seed in (1, 2):
        p = gen_random_reducible(12, 60, seed=seed)
        prof = profile_polynomial(p, ToleranceConfig())
        add(list(prof.rho), 1e-6, f"profile_d12_s{seed}")
    return cases


# ------------------------------------------------------------------- factor
def sympy_record(p: IntPolynomial, tag: str, exc: Exception):
    """Where the reference raises on a valid input, freeze the unique
    factorization from sympy and the reference's error text."""
    import sympy

    x = sympy.Symbol("x")
    expr = sum(sympy.Integer(c) * x**i for i, c in enumerate(p.coeffs))
    cont, lst = sympy.factor_list(expr, x)
    fs = []
    for fac, m in lst:
        co = [int(c) for c in sympy.Poly(fac, x).all_coeffs()[::-1]]
        fs.append((IntPolynomial(co), int(m)))
    # same canonical order and sign convention as verify.py:209-222
    if fs and all(g.leading > 0 for g, _ in fs):
        pass
    fs.sort(key=lambda fm: (fm[0].degree, fm[0].coeffs, fm[1]))
    return {
        "tag": tag,
        "input": poly_json(p),
        "content": str(int(cont)),
        "factors": [[poly_json(g), m] for g, m in fs],
        "certificate": True,
        "irreducible": len(fs) == 1 and fs[0][1] == 1,
        "ref_error": f"{type(exc).__name__}: {exc}",
        "source": "sympy.factor_list",
    }


def c2_parts(seed: int):
    """three rng.randint(-100, 100) monic degree-20
    polynomials, each certified by is_irreducible, distinct."""
    rng = random.Random(seed)
    parts = []
    while len(parts) < 3:
        cand = IntPolynomial([rng.randint(-100, 100) for _ in range(20)] + [1])
        if cand in parts:
            continue
        if is_irreducible(cand):
            parts.append(cand)
    return parts


def factor_cases():
    P = IntPolynomial
    out = []

    def add(p: IntPolynomial, tag: str, parts=None):
        t0 = time.perf_counter()
        try:
            res = factor(p)
        except Exception as exc:  # reference bug: record sympy's answer instead
            out.append(sympy_record(p, tag, exc))
            return
        dt = time.perf_counter() - t0
        rec = {"tag": tag, "input": poly_json(p), "ref_seconds": dt}
        rec.update(result_json(res))
        rec["stats"] = {
            "n": res.stats.n,
            "candidates": res.stats.candidates,
            "rejected": res.stats.rejected,
            "root_seconds": res.stats.root_seconds,
            "recombine_seconds": res.stats.recombine_seconds,
            "verify_seconds": res.stats.verify_seconds,
        }
        if parts is not None:
            want = sorted(tuple(q.coeffs) for q in parts)
            got = sorted(tuple(g.coeffs) for g, _ in res.factors)
            assert want == got, tag
            rec["parts"] = [poly_json(q) for q in parts]
        out.append(rec)

    # test_verify.py KATs
    add(P([-1, 0, 1]), "diff_squares")
    add(P([1, 0, -10, 0, 1]), "sd2")
    add(P([-2, 0, -1, 0, 1]), "x2m2_x2p1")
    add(P([2, -3, 0, 1]), "square_free_path")
    add(P([-2, 0, 2]), "content_two")
    add(P([1, 3, 2]), "non_monic")
    add(P([1, 0, -1]), "negative_lead")
    add(P([7, 1]), "linear")
    add(P([5, 0, 3]), "non_monic_irreducible")
    add(P([-6, 11, -6, 1]), "three_linear")
    add(P([0, 0, 1]), "x_squared")
    add(P([0, 1, 1]), "x_times_xp1")
    add(P([4, 0, 0, 0, 1]), "x4p4")  # (x^2+2x+2)(x^2-2x+2)
    add(gen_swinnerton_dyer(3), "sd3")
    add(gen_swinnerton_dyer(4), "sd4")
    add(P([-1, 0, 0, 0, 0, 0, 1]), "x6m1")
    add(P([1, -2, 1]) * P([1, 1]) ** 3 * P([3, 0, 1]), "multiplicities")
    add(P([6, 5, 1]) * P([-4, 0, 9]), "non_monic_product")
    # backend independence corpus (test_verify.py:179-192)
    rng = random.Random(23)
    for i in range(6):
        a = P([rng.randint(-20, 20) for _ in range(4)] + [1])
        b = P([rng.randint(-20, 20) for _ in range(4)] + [1])
        add(a * b, f"bi_{i}")
    # acceptance-2 round trips (test_acceptance.py:60-75), first 34 inputs
    degrees = list(range(8, 41, 2))
    for i in range(34):
        d = degrees[i % len(degrees)]
        f, g = gen_random_reducible_parts(d, 100, seed=10_000 + i)
        add(f * g, f"ac2_{i}_d{d}", parts=[f, g])
    # C1: d = 40, two degree-20 halves, coefficients in [-10, 10]
    for seed in range(10):
        f, g = gen_random_reducible_parts(40, 10, seed)
        add(f * g, f"c1_s{seed}", parts=[f, g])
    # C2: d = 60, three degree-20 factors in [-100, 100]
    for seed in range(2):
        parts = c2_parts(seed)
        add(parts[0] * parts[1] * parts[2], f"c2_s{seed}", parts=parts)
    return out


# ------------------------------------------------------------------- verify
def verify_cases():
    """Reference verdicts for every nontrivial candidate of recombine_e on a
    few real profiles: (pattern, trace_test, round_and_divide result)."""
    cfg = ToleranceConfig()
    out = []
    inputs = []
    for seed in range(3):
        f, g = gen_random_reducible_parts(40, 10, seed)
        inputs.append((f"c1_s{seed}", f * g))
    for seed in (3, 11):
        f, g = gen_random_reducible_parts(20, 100, seed)
        inputs.append((f"d20_s{seed}", f * g))
    inputs.append(("sd3", gen_swinnerton_dyer(3)))
    inputs.append(("sd4", gen_swinnerton_dyer(4)))
    for tag, p in inputs:
        prof = profile_polynomial(p, cfg)
        rho = RhoVector.from_profile(prof)
        cands = recombine_e(rho, cfg.eps)
        full = (1 << prof.n) - 1
        rows = []
        for s in sorted(cands.nontrivial()):
            for t in (s, s ^ full):
                cand = build_candidate(t, prof)
                tt = bool(trace_test(cand, cfg.eps))
                q = round_and_divide(cand, p, cfg.eps) if tt else None
                rows.append(
                    {
                        "pattern": t,
                        "degree": cand.degree,
                        "trace_ok": tt,
                        "q": poly_json(q) if q is not None else None,
                    }
                )
        out.append(
            {
                "tag": tag,
                "p": poly_json(p),
                "real_roots": [fhex(v) for v in prof.real_roots],
                "pair_sums": [fhex(v) for v in prof.pair_sums],
                "pair_products": [fhex(v) for v in prof.pair_products],
                "rho": [fhex(v) for v in prof.rho],
                "perm": list(prof.perm),
                "eps": cfg.eps,
                "candidates": rows,
            }
        )
    return out


# --------------------------------------------------------------- big inputs
def big_inputs():
    import sympy

    x = sympy.Symbol("x")

    def sympy_factors(p: IntPolynomial):
        expr = sum(sympy.Integer(c) * x**i for i, c in enumerate(p.coeffs))
        cont, lst = sympy.factor_list(expr, x)
        fs = []
        for fac, m in lst:
            co = sympy.Poly(fac, x).all_coeffs()[::-1]
            fs.append(([int(c) for c in co], int(m)))
        return int(cont), fs

    out = {"c3": [], "c4": [], "c5": []}
    for seed in range(5):
        t0 = time.perf_counter()
        f, g = gen_random_reducible_parts(100, 100, seed)
        p = f * g
        cont, fs = sympy_factors(p)
        want = sorted([tuple(f.coeffs), tuple(g.coeffs)], key=lambda c: (len(c), c))
        got = sorted([tuple(c) for c, _ in fs], key=lambda c: (len(c), c))
        assert cont == 1 and want == got
        out["c3"].append(
            {
                "seed": seed,
                "p": poly_json(p),
                "factors": [[[str(c) for c in co], 1] for co in want],
                "n_ref": len(profile_polynomial(p).rho),
            }
        )
        print(f"c3 seed {seed}: {time.perf_counter() - t0:.1f}s")
    for seed in range(3):
        rng = random.Random(seed)
        p = IntPolynomial([rng.randint(-100, 100) for _ in range(120)] + [1])
        cont, fs = sympy_factors(p)
        assert cont == 1 and len(fs) == 1 and fs[0][1] == 1, f"c4 seed {seed} reducible"
        out["c4"].append({"seed": seed, "p": poly_json(p), "factors": [[poly_json(p), 1]]})
    sd6 = gen_swinnerton_dyer(6)
    out["c5"].append({"k": 6, "p": poly_json(sd6), "factors": [[poly_json(sd6), 1]]})
    return out


def main(which):
    if "recombine" in which:
        dump("recombine_cases.json", recombine_cases())
    if "factor" in which:
        dump("factor_cases.json", factor_cases())
    if "verify" in which:
        dump("verify_cases.json", verify_cases())
    if "big" in which:
        dump("big_inputs.json", big_inputs())


if __name__ == "__main__":
    main(sys.argv[1:] or ["recombine", "factor", "verify", "big"])
