"""Exact polynomial layer: KATs mirroring pkg/tests/test_polynomial.py and the
inputs the golden fixtures were built from."""
import random

import pytest

from conftest import poly_of
from paper_2410_15880_b200 import (
    IntPolynomial as P,
    divide_exact,
    gen_random_reducible_parts,
    gen_swinnerton_dyer,
    monic_transform,
    monic_untransform_factor,
    multiply,
    poly_gcd,
    square_free_decompose,
)


def test_construction_strips_and_formats():
    assert P([1, 2, 0, 0]).coeffs == (1, 2)
    assert P([]).coeffs == (0,) and P([0, 0]).is_zero()
    assert str(P([1, 0, -10, 0, 1])) == "x^4 - 10*x^2 + 1"
    assert str(P([-3])) == "-3" and str(P([0, -1])) == "-x"
    assert P.from_text("1 0 -2").to_text() == "1 0 -2"


def test_multiply_divide_round_trip():
    rng = random.Random(1)
    for _ in range(30):
        a = P([rng.randint(-50, 50) for _ in range(rng.randint(1, 8))] + [rng.choice([1, 2, -3])])
        b = P([rng.randint(-50, 50) for _ in range(rng.randint(1, 8))] + [1])
        assert divide_exact(a * b, b) == a
        assert multiply(a, b) == a * b


def test_divide_exact_rejections():
    assert divide_exact(P([1, 0, 1]), P([1, 1])) is None
    assert divide_exact(P([1, 2]), P([0, 0, 1])) is None
    assert divide_exact(P([0]), P([1, 1])) == P([0])
    with pytest.raises(ZeroDivisionError):
        divide_exact(P([1, 1]), P([0]))


def test_content_sign_convention():
    assert P([-2, 0, 2]).content() == 2
    assert P([1, 0, -1]).content() == -1
    assert P([1, 0, -1]).primitive_part() == P([-1, 0, 1])


def test_gcd_and_square_free():
    a = P([-1, 1]) ** 2 * P([2, 1])
    assert poly_gcd(a, a.derivative()) == P([-1, 1])
    parts = square_free_decompose(P([1, -2, 1]) * P([1, 1]) ** 3 * P([3, 0, 1]))
    rebuilt = P([1])
    for f, m in parts:
        rebuilt = rebuilt * f**m
    assert rebuilt == P([1, -2, 1]) * P([1, 1]) ** 3 * P([3, 0, 1])
    assert [m for _, m in parts] == sorted(m for _, m in parts)
    assert square_free_decompose(P([-1, 0, 1])) == [(P([-1, 0, 1]), 1)]
    with pytest.raises(ValueError):
        square_free_decompose(P([5]))


def test_monic_transform_round_trip():
    p = P([1, 3, 2])  # (2x + 1)(x + 1)
    t = monic_transform(p)
    assert t.is_monic()
    # t = 2 * p(x / 2) * 2^(d-1) / 2^d... its factors pull back to p's factors
    assert monic_untransform_factor(P([1, 1]), 2) == P([1, 2])
    assert monic_untransform_factor(P([2, 1]), 2) == P([1, 1])


def test_swinnerton_dyer_matches_reference_inputs(factor_cases, big_inputs):
    by_tag = {c["tag"]: c for c in factor_cases}
    assert gen_swinnerton_dyer(2) == P([1, 0, -10, 0, 1])
    assert gen_swinnerton_dyer(3) == poly_of(by_tag["sd3"]["input"])
    assert gen_swinnerton_dyer(4) == poly_of(by_tag["sd4"]["input"])
    assert gen_swinnerton_dyer(6) == poly_of(big_inputs["c5"][0]["p"])
    assert gen_swinnerton_dyer(6).degree == 64
    with pytest.raises(ValueError):
        gen_swinnerton_dyer(7)


def test_generator_reproduces_reference_draws(factor_cases):
    # with the reference's own accept/reject decisions replayed (the recorded
    # halves are irreducible), the generator draws the same polynomials
    for c in factor_cases:
        if not c["tag"].startswith("c1_s"):
            continue
        seed = int(c["tag"][4:])
        parts = sorted(tuple(int(x) for x in f) for f in c["parts"])
        want = {tuple(int(x) for x in f) for f in c["parts"]}
        f, g = gen_random_reducible_parts(40, 10, seed, irreducible=lambda q: q.coeffs in want)
        assert sorted([f.coeffs, g.coeffs]) == parts


def test_generator_validation():
    with pytest.raises(ValueError):
        gen_random_reducible_parts(5, 10, 0, irreducible=lambda q: True)
    with pytest.raises(ValueError):
        gen_random_reducible_parts(8, 0, 0, irreducible=lambda q: True)


def _school_mul(a, b):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _school_div(p, q):
    """Long division over Z (R/polynomial.py:155-183 semantics), plain lists."""
    dp, dq = len(p) - 1, len(q) - 1
    if dp < dq:
        return None
    rem, quot, lead = list(p), [0] * (dp - dq + 1), q[-1]
    for k in range(dp - dq, -1, -1):
        t, r = divmod(rem[k + dq], lead)
        if r:
            return None
        quot[k] = t
        for i in range(dq + 1):
            rem[k + i] -= t * q[i]
    return None if any(rem[:dq]) else quot


def test_kronecker_multiply_and_divide_match_schoolbook():
    """multiply / divide_exact switch to Kronecker substitution for large
    degrees; both must agree with the schoolbook definitions exactly,
    including huge coefficients, negative leads and near-miss dividends."""
    from paper_2410_15880_b200.polynomial import divide_exact, multiply

    rng = random.Random(11)
    hits = 0
    for _ in range(400):
        dq, dr = rng.randint(0, 40), rng.randint(0, 40)
        bits = rng.choice([2, 17, 64, 140])
        q = [rng.randint(-(1 << bits), 1 << bits) for _ in range(dq)] + [rng.choice([1, -1, 3, -7])]
        r = [rng.randint(-(1 << bits), 1 << bits) for _ in range(dr)] + [rng.choice([1, -2, 5])]
        prod = multiply(P(q), P(r))
        assert list(prod.coeffs) == list(P(_school_mul(q, r)).coeffs)
        pc = list(prod.coeffs)
        if rng.random() < 0.5:
            pc[rng.randrange(len(pc))] += rng.choice([1, -1, 1 << bits])
        got = divide_exact(P(pc), P(q))
        want = _school_div(pc, q)
        if want is None:
            assert got is None
        else:
            hits += 1
            assert got is not None and list(got.coeffs) == list(P(want).coeffs)
    assert hits > 100


def test_divide_exact_monic_native_range_edges():
    """The native monic long division (rfr_divide_monic_i64) hands back to
    the big-integer path when a running quotient coefficient reaches 2^62 or
    the operands leave int64 / 2^31: the answers still equal the schoolbook
    ones on both sides of those limits."""
    from paper_2410_15880_b200.polynomial import divide_exact, multiply

    cases = [
        ([1] + [0] * 9 + [1], [-(1 << 30), 1]),                   # quotient grows past 2^62: not exact
        (list(multiply(P([-(1 << 30), 1]), P([5, 0, 1])).coeffs), [-(1 << 30), 1]),  # exact, small quotient
        (list(multiply(P([(1 << 31) - 1, 1]), P([3, 1])).coeffs), [(1 << 31) - 1, 1]),  # |q_i| at 2^31 - 1
        (list(multiply(P([1 << 31, 1]), P([3, 1])).coeffs), [1 << 31, 1]),  # |q_i| = 2^31: big-integer path
        (list(multiply(P([7, 1]), P([(1 << 61), 2, 1])).coeffs), [7, 1]),  # p beyond 2^62
        ([(1 << 62) - 1, 0, 1], [1, 1]),                                     # not exact, large constant
    ]
    for pc, q in cases:
        got = divide_exact(P(pc), P(q))
        want = _school_div(pc, q)
        if want is None:
            assert got is None
        else:
            assert got is not None and list(got.coeffs) == list(P(want).coeffs)


def test_divide_exact_base_2_64_carries():
    """divide_exact tries the 64-bit Kronecker base first: a quotient whose
    coefficients overflow 64 bits is still found (Mignotte base), and a
    dividend that equals q * r at x = 2^64 only through a carry (p_k + 2^64,
    p_{k+1} - 1) is rejected."""
    from paper_2410_15880_b200.polynomial import divide_exact, multiply

    rng = random.Random(3)
    for _ in range(60):
        dq, dr = rng.randint(8, 30), rng.randint(8, 30)
        q = [rng.randint(-99, 99) for _ in range(dq)] + [1]
        r = [rng.randint(-99, 99) for _ in range(dr)] + [1]
        r[rng.randrange(dr)] = rng.choice([1, -1]) * ((1 << 70) + rng.randint(0, 1 << 40))
        pc = list(multiply(P(q), P(r)).coeffs)
        got = divide_exact(P(pc), P(q))
        assert got is not None and list(got.coeffs) == r
        r_small = [rng.randint(-99, 99) for _ in range(dr)] + [1]
        pc = list(multiply(P(q), P(r_small)).coeffs)
        k = rng.randrange(len(pc) - 1)
        pc[k] += 1 << 64
        pc[k + 1] -= 1
        assert divide_exact(P(pc), P(q)) is None
        assert _school_div(pc, q) is None


@pytest.mark.parametrize("q", [33554393, 2305843009213693951])
def test_squarefree_screen_never_accepts_a_square(q):
    """The native modular screen (rfr_squarefree_mod, pseudo-division Euclid;
    double-precision path below 2^25, 128-bit products above) answers
    'square-free' only for square-free inputs (checked with sympy)."""
    import ctypes

    import numpy as np
    import sympy

    from paper_2410_15880_b200 import _lib

    lib = _lib.load()
    x = sympy.symbols("x")
    rng = random.Random(5)
    accepted = 0
    for _ in range(120):
        d = rng.randint(2, 30)
        co = [rng.randint(-50, 50) for _ in range(d)] + [1]
        if rng.random() < 0.4:
            f = [rng.randint(-5, 5) for _ in range(rng.randint(1, 3))] + [1]
            pp = sympy.Poly(list(reversed(co)), x) * sympy.Poly(list(reversed(f)), x) ** 2
            co = [int(c) for c in reversed(pp.all_coeffs())]
        cm = np.array([c % q for c in co], dtype=np.uint64)
        got = lib.rfr_squarefree_mod(cm.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(co) - 1, q)
        poly = sympy.Poly(list(reversed(co)), x)
        square_free = sympy.gcd(poly, poly.diff(x)).degree() == 0
        if got == 1:
            accepted += 1
            assert square_free
    assert accepted > 30


def test_squarefree_screen_fp_path_is_exact_mod_q():
    """The double-precision path (q < 2^25, symmetric residues reduced by
    round-to-nearest) decides gcd(p, p') = 1 over F_q exactly as sympy's
    GF(q) gcd does, up to degree 140 (where the residues are largest)."""
    import ctypes

    import numpy as np
    import sympy

    from paper_2410_15880_b200 import _lib

    lib = _lib.load()
    x = sympy.symbols("x")
    q = 33554393
    rng = random.Random(11)
    yes = no = 0
    for _ in range(40):
        d = rng.randint(2, 140)
        co = [rng.randrange(q) for _ in range(d)] + [1]
        if rng.random() < 0.5:  # a square factor mod q
            f = [rng.randrange(q) for _ in range(rng.randint(1, 4))] + [1]
            pp = sympy.Poly(list(reversed(co)), x, modulus=q) * sympy.Poly(list(reversed(f)), x, modulus=q) ** 2
            co = [int(c) % q for c in reversed(pp.all_coeffs())]
        cm = np.array(co, dtype=np.uint64)
        got = lib.rfr_squarefree_mod(cm.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(co) - 1, q)
        poly = sympy.Poly(list(reversed(co)), x, modulus=q)
        want = int(sympy.gcd(poly, poly.diff(x)).degree() == 0)
        assert got == want
        yes += want
        no += 1 - want
    assert yes > 5 and no > 5


def test_squarefree_screen_i64_entry_matches_the_residue_entry():
    """rfr_squarefree_i64 (signed coefficients reduced inside) answers as
    rfr_squarefree_mod on the residues, for both prime paths."""
    import ctypes

    import numpy as np

    from paper_2410_15880_b200 import _lib

    lib = _lib.load()
    rng = random.Random(17)
    for q in (33554393, 2305843009213693951):
        for _ in range(60):
            d = rng.randint(1, 120)
            co = [rng.randint(-(1 << 61), 1 << 61) for _ in range(d)] + [rng.choice([1, -3, 7])]
            if rng.random() < 0.3:  # a square factor over Z
                co = list(multiply(P(co[: d // 2 + 1]), multiply(P([rng.randint(-9, 9), 1]), P([rng.randint(-9, 9), 1]))).coeffs)
                if max(abs(c) for c in co) >= 1 << 62:
                    continue
            a = np.array(co, dtype=np.int64)
            cm = np.array([c % q for c in co], dtype=np.uint64)
            want = lib.rfr_squarefree_mod(cm.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(co) - 1, q)
            assert lib.rfr_squarefree_i64(a.ctypes.data, len(co) - 1, q) == want


def test_factor_cells_split_implied_factors():
    """The factor partition (verify._factor_cells): after an early stop the
    candidates may hold t = f3*f4, f3 inside t, f1 inside ~t and nothing for
    f4 or f2 by themselves; the cells are still the four factors (a greedy
    cover by minimal patterns returned f1, f3 and f2*f4 here)."""
    from paper_2410_15880_b200.polynomial import multiply
    from paper_2410_15880_b200.verify import _factor_cells

    f1, f2 = P([-2, 0, 1]), P([1, 1, 0, 1])           # entity bits 0-1, 2-4
    f3, f4 = P([5, -1, 0, 0, 1]), P([3, 2, 1, 1, 0, 1])  # bits 5-8, 9-13
    pats = {1: 0b11, 2: 0b11100, 3: 0b111100000, 4: 0b11111000000000}
    full = (1 << 14) - 1
    p = multiply(multiply(f1, f2), multiply(f3, f4))
    found = {pats[3] | pats[4]: multiply(f3, f4), pats[3]: f3, pats[1]: f1}
    cells = _factor_cells(found, p, full)
    got = sorted((c, pc.coeffs) for c, pc in cells)
    want = sorted((pats[i], f.coeffs) for i, f in ((1, f1), (2, f2), (3, f3), (4, f4)))
    assert got == want
    # a partial overlap (f2*f3 against f3*f4) is resolved by a gcd
    found = {pats[2] | pats[3]: multiply(f2, f3), pats[3] | pats[4]: multiply(f3, f4)}
    cells = sorted((c, pc.coeffs) for c, pc in _factor_cells(found, p, full))
    assert (pats[3], f3.coeffs) in cells and (pats[2], f2.coeffs) in cells and (pats[4], f4.coeffs) in cells
