"""The small-factor screens in front of the search (CPU: they use only the
host profile and exact arithmetic).  Regression for a one-entity factor whose
constant term lies above 2^53: the high word of its double-double value is
not the integer, so rounding it alone missed the factor, and the flood path
then confirmed the product of two such quadratics as one "irreducible"
factor (it divides p, so the certificate still passed)."""
from paper_2410_15880_b200 import IntPolynomial as P
from paper_2410_15880_b200.rootfinder import hp_profile
from paper_2410_15880_b200.verify import _single_entity_factors, _small_factors


def _big_pair_product():
    q1, q2 = P([2**53 + 1, 1, 1]), P([2**53 + 3, 1, 1])
    q3, q4 = P([-2, 0, 1]), P([-3, 0, 1])
    return [q1, q2, q3, q4], q1 * q2 * q3 * q4


def test_single_entity_factors_round_the_exact_value_above_2_53():
    (q1, q2, _, _), p = _big_pair_product()
    prof = hp_profile(p)
    got = sorted(tuple(q.coeffs) for _, q in _single_entity_factors(prof, p))
    assert got == sorted([tuple(q1.coeffs), tuple(q2.coeffs)])


def test_small_factors_lists_single_entities_before_their_unions():
    (q1, q2, _, _), p = _big_pair_product()
    prof = hp_profile(p)
    small = _small_factors(prof, p)
    pats = [t[0] for t, _ in small]
    singles = [t for t in pats if bin(t).count("1") == 1]
    assert len(singles) >= 2
    # every single comes before every multi-entity pattern
    first_multi = min(i for i, t in enumerate(pats) if bin(t).count("1") > 1)
    assert all(pats.index(t) < first_multi for t in singles)
    facs = {tuple(q.coeffs) for _, q in small}
    assert tuple(q1.coeffs) in facs and tuple(q2.coeffs) in facs


def test_integer_root_above_2_53_is_split_exactly():
    r = 2**60 + 7
    p = P([-r, 1]) * P([-2, 0, 1]) * P([-5, 0, 1])
    prof = hp_profile(p)
    got = [tuple(q.coeffs) for _, q in _single_entity_factors(prof, p)]
    assert (-r, 1) in got
