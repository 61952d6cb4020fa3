"""Host preprocessing: high-precision roots, profile layout, the exact keys
and the completeness of the key window on the benchmark inputs (CPU)."""
import math
from fractions import Fraction

import numpy as np
import pytest

from conftest import poly_of
from paper_2410_15880_b200 import IntPolynomial as P
from paper_2410_15880_b200 import ToleranceConfig, build_profile, find_roots, hp_profile
from paper_2410_15880_b200.rootfinder import frac, hp_roots
from paper_2410_15880_b200.verify import _search_window

TWO64 = 1 << 64


def test_tolerance_config_validation():
    with pytest.raises(ValueError):
        ToleranceConfig(eps=0.0)
    with pytest.raises(ValueError):
        ToleranceConfig(eps=0.5)
    with pytest.raises(ValueError):
        ToleranceConfig(precision="quad")
    assert ToleranceConfig().eps == 1e-6


def test_frac_convention():
    assert frac(-0.25) == 0.75 and frac(2.5) == 0.5


def test_find_roots_layout():
    z = find_roots(P([-2, 0, -1, 0, 1]))  # (x^2-2)(x^2+1)
    assert np.allclose(z[:2].real, [-math.sqrt(2), math.sqrt(2)])
    assert np.all(z[:2].imag == 0)
    assert np.allclose(z[2:], [1j, -1j])


def test_build_profile_kats():
    prof = build_profile(np.array([0.5 + 0j, -0.25 + 0j, 1 + 1j, 1 - 1j]))
    assert prof.r == 2 and prof.c == 1
    assert prof.rho.tolist() == [0.0, 0.5, 0.75]
    assert prof.pair_sums.tolist() == [2.0] and prof.pair_products.tolist() == pytest.approx([2.0])


def test_hp_roots_precision_against_exact_values():
    re_hi, re_lo, im_hi, im_lo, err = hp_roots(P([-2, 0, -1, 0, 1]))
    for i in range(4):
        if im_hi[i] == 0:
            r = Fraction(re_hi[i]) + Fraction(re_lo[i])
            assert abs(r * r - 2) < Fraction(1, 10**28)
        else:
            assert abs(abs(im_hi[i]) - 1) < 1e-28
    assert err.max() < 1e-28


def test_hp_profile_entities_and_keys():
    prof = hp_profile(P([-2, 0, -1, 0, 1]))
    assert prof.n == 3 and prof.r == 2 and prof.c == 1
    # pair x^2 + 1: t = 0, m = 1 -> keys 0 and frac(t^2 - 2m) = 0
    j = prof.perm.index(2)
    assert int(prof.keys1[j]) in (0,) and int(prof.keys2[j]) == 0
    # the two real roots +-sqrt(2): Tr1 = 0, Tr2 = 4 -> key sums vanish
    ks = [i for i in range(3) if prof.perm[i] < 2]
    s1 = sum(int(prof.keys1[i]) for i in ks) % TWO64
    s2 = sum(int(prof.keys2[i]) for i in ks) % TWO64
    assert min(s1, TWO64 - s1) <= prof.key_err1 and min(s2, TWO64 - s2) <= prof.key_err2


def _factor_pattern(prof, root_values, f):
    """rho-index pattern of the entities whose roots are roots of f."""
    pat = 0
    for i, ent in enumerate(prof.perm):
        if ent < prof.r:
            u = float(prof.real_roots[ent])
            if abs(f.evaluate(u)) < 1e-6 * max(1.0, abs(u)) ** f.degree * 1e3:
                pat |= 1 << i
        else:
            t = float(prof.pair_sums[ent - prof.r])
            m = float(prof.pair_products[ent - prof.r])
            # the pair is a factor of f iff f(z) ~ 0 for z = t/2 + i sqrt(m - t^2/4)
            z = complex(t / 2, math.sqrt(max(m - t * t / 4, 0.0)))
            if abs(f.evaluate(z)) < 1e-6 * max(1.0, abs(z)) ** f.degree * 1e3:
                pat |= 1 << i
    return pat


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_true_factor_keys_fall_inside_the_window_c3(big_inputs, seed):
    case = big_inputs["c3"][seed]
    p = poly_of(case["p"])
    f = poly_of(case["factors"][0][0])
    prof = hp_profile(p)
    keys, T = _search_window(prof)
    pat = _factor_pattern(prof, None, f)
    full = (1 << prof.n) - 1
    from paper_2410_15880_b200.verify import selected_degree

    assert selected_degree(pat, prof) == f.degree
    for t in (pat, pat ^ full):
        s = sum(int(keys[i]) for i in range(prof.n) if (t >> i) & 1) % TWO64
        assert min(s, TWO64 - s) <= T, (seed, s)
    assert T < 1 << 9  # ~2n rounding units: false hits ~ 2^(n-1) * 2T / 2^64


def test_hp_profile_c4_and_sd6_certified(big_inputs):
    prof = hp_profile(poly_of(big_inputs["c4"][0]["p"]))
    assert prof.n == 63 and prof.root_err < 1e-20
    sd6 = hp_profile(poly_of(big_inputs["c5"][0]["p"]))  # multiprecision path
    assert sd6.n == 64 and sd6.r == 64 and sd6.root_err < 1e-20


@pytest.mark.parametrize("seed", [0, 3])
def test_sub_profile_of_a_factor_matches_its_own_profile(big_inputs, seed):
    """Early exit splits p by a verified factor's pattern and searches each
    piece over its own entities without new root finding: the sub-profile
    of the true factor's pattern holds the factor's roots (as its own
    hp_profile finds them), keys in rho order, and a permutation."""
    from paper_2410_15880_b200.verify import _sub_profile, selected_degree

    case = big_inputs["c3"][seed]
    p = poly_of(case["p"])
    f = poly_of(case["factors"][0][0])
    prof = hp_profile(p)
    pat = _factor_pattern(prof, None, f)
    full = (1 << prof.n) - 1
    for t, g in ((pat, f), (pat ^ full, poly_of(case["factors"][1][0]))):
        sub = _sub_profile(prof, t)
        own = hp_profile(g)
        assert (sub.n, sub.r, sub.c) == (own.n, own.r, own.c)
        assert sorted(sub.perm) == list(range(sub.n))
        assert np.all(np.diff(sub.rho) >= 0)
        assert selected_degree((1 << sub.n) - 1, sub) == g.degree
        np.testing.assert_allclose(np.sort(sub.real_roots), np.sort(own.real_roots), rtol=1e-12)
        np.testing.assert_allclose(np.sort(sub.pair_sums), np.sort(own.pair_sums), rtol=1e-12)
        np.testing.assert_allclose(np.sort(sub.pair_products), np.sort(own.pair_products), rtol=1e-12)
        # the whole sub-profile is the factor: its Tr1 key sum is an integer
        s = sum(int(k) for k in sub.keys1) % TWO64
        assert min(s, TWO64 - s) <= sub.key_err1 + sub.n
        # each bit's key is its entity's first power sum (root, or t of a pair)
        for j in range(sub.n):
            e = sub.perm[j]
            v = sub.real_roots[e] if e < sub.r else sub.pair_sums[e - sub.r]
            frac = v - np.floor(v)
            assert abs(int(sub.keys1[j]) / TWO64 - frac) < 1e-9 or abs(abs(int(sub.keys1[j]) / TWO64 - frac) - 1) < 1e-9


def _mp_roots(p, dps=80):
    import mpmath

    with mpmath.workdps(dps):
        return [complex(0, 0) if False else r for r in
                mpmath.polyroots([mpmath.mpf(c) for c in reversed(p.coeffs)], maxsteps=800,
                                 extraprec=4 * dps)]


def _check_discs(p):
    """Every certified disc D(z_i, err_i) holds exactly one of the true roots
    (computed independently by mpmath at 80 digits), and the discs are
    pairwise disjoint (Lemma 1)."""
    import mpmath

    re_hi, re_lo, im_hi, im_lo, err = hp_roots(p)
    d = p.degree
    with mpmath.workdps(80):
        true = _mp_roots(p)
        for i in range(d):
            z = mpmath.mpc(mpmath.mpf(re_hi[i]) + mpmath.mpf(re_lo[i]),
                           mpmath.mpf(im_hi[i]) + mpmath.mpf(im_lo[i]))
            inside = [w for w in true if abs(w - z) <= err[i]]
            assert len(inside) == 1, (i, err[i], min(abs(w - z) for w in true))
    return err


@pytest.mark.parametrize("seed", [0, 3])
def test_inclusion_discs_hold_the_true_roots_c3(big_inputs, seed):
    err = _check_discs(poly_of(big_inputs["c3"][seed]["p"]))
    assert err.max() < 1e-22


def test_inclusion_discs_clustered_roots():
    """Mignotte-like x^d - 2 (a x - 1)^2: two real roots ~a^-(d/2+1) apart
    near 1/a -- ill-conditioned; the discs must still hold the true roots
    (or the root finder must escalate precision, never report a wrong disc)."""
    for d, a in ((12, 6), (16, 5), (20, 10)):
        q = P([-2, 4 * a, -2 * a * a] + [0] * (d - 3) + [1])
        err = _check_discs(q)
        assert np.all(err > 0)


def test_inclusion_discs_multiprecision_path():
    """142-bit coefficients (the multiprecision polish) get certified discs
    too: a product of 8 quadratics x^2 - q with large q."""
    p = P([1])
    for q in (2**61 - 1, 2**31 - 1, 1000003, 999983, 104729, 7919, 541, 97):
        p = p * P([-q, 0, 1])
    _check_discs(p)


def test_dyadic_entity_arithmetic_matches_fractions(big_inputs):
    """hp_profile's entity values are exact dyadic rationals (_Dy); computed
    with Fraction instead, every field of the profile (double-double
    entities, rho, keys, key error bounds) is the same."""
    import random
    from fractions import Fraction

    from conftest import poly_of
    from paper_2410_15880_b200 import IntPolynomial
    from paper_2410_15880_b200.rootfinder import hp_profile

    polys = [poly_of(c["p"]) for c in big_inputs["c3"][:2]] + [poly_of(big_inputs["c4"][0]["p"])]
    rng = random.Random(9)
    for _ in range(12):
        d = rng.randint(5, 50)
        polys.append(IntPolynomial([rng.randint(-40, 40) for _ in range(d)] + [1]))
    checked = 0
    for p in polys:
        try:
            a = hp_profile(p)
        except Exception:
            continue
        b = hp_profile(p, num=Fraction)
        for f in ("real_roots", "pair_sums", "pair_products", "rho", "real_lo", "sum_lo", "prod_lo",
                  "keys1", "keys2", "keys3"):
            assert np.array_equal(np.asarray(getattr(a, f)), np.asarray(getattr(b, f))), f
        for f in ("perm", "key_err1", "key_err2", "key_err3", "root_err"):
            assert getattr(a, f) == getattr(b, f), f
        checked += 1
    assert checked >= 10


def test_dyadic_float_is_correctly_rounded_for_wide_mantissas():
    """_Dy -> float is Fraction's correctly rounded value also when the
    mantissa is far wider than a double (a double-double whose low part is
    ~2^-900 below the high part: a 1000-bit mantissa), and for its powers."""
    import random
    from fractions import Fraction

    from paper_2410_15880_b200.rootfinder import _Dy

    rng = random.Random(1)
    for _ in range(3000):
        hi = rng.uniform(-1e6, 1e6) * 2.0 ** rng.randint(-60, 60)
        lo = hi * 2.0 ** -53 * rng.uniform(-1, 1) * 2.0 ** -rng.randint(0, 900)
        d = _Dy.of(hi) + _Dy.of(lo)
        f = Fraction(hi) + Fraction(lo)
        assert float(d) == float(f)
        assert float(d * d * d) == float(f * f * f)
        assert float(d - 3 * d * d) == float(f - 3 * f * f)

