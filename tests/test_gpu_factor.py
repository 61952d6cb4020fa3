"""GPU parity of factor(): the same irreducible factorizations (factors,
multiplicities, content, canonical order) as the reference on its own
inputs (tests/golden/factor_cases.json from pkg/src/polyfactor/verify.py:
187-233), the d = 100 benchmark inputs (C3, factors by construction), the
d = 120 irreducible inputs (C4) and Swinnerton-Dyer f6 (C5)."""
import random

import numpy as np
import pytest

from conftest import poly_of, rho_of
from paper_2410_15880_b200 import IntPolynomial as P
from paper_2410_15880_b200 import RootProfile, factor, is_irreducible, verify_candidates
from paper_2410_15880_b200 import _lib
from paper_2410_15880_b200.errors import WidthExceeded

pytestmark = pytest.mark.gpu


def _want(c):
    return [([int(x) for x in f], m) for f, m in c["factors"]]


def _got(res):
    return [(list(g.coeffs), m) for g, m in res.factors]


def test_factor_matches_reference_on_all_golden_inputs(factor_cases):
    for c in factor_cases:
        res = factor(poly_of(c["input"]))
        assert _got(res) == _want(c), c["tag"]
        assert str(res.content) == c["content"] and res.certificate, c["tag"]
        assert res.irreducible == c["irreducible"]


@pytest.mark.parametrize("seed", range(5))
def test_factor_degree_100_benchmark_inputs(big_inputs, seed):
    c = big_inputs["c3"][seed]
    res = factor(poly_of(c["p"]))
    assert _got(res) == _want(c) and res.certificate
    assert res.stats.n == c["n_ref"]


@pytest.mark.parametrize("seed", range(3))
def test_factor_degree_120_irreducible(big_inputs, seed):
    c = big_inputs["c4"][seed]
    res = factor(poly_of(c["p"]))
    assert res.irreducible and res.certificate and _got(res) == _want(c)
    assert res.stats.candidates == res.stats.rejected


def test_factor_swinnerton_dyer_f6_irreducible(big_inputs):
    c = big_inputs["c5"][0]
    res = factor(poly_of(c["p"]))
    assert res.irreducible and res.certificate
    assert res.stats.n == 64
    # Tr1 + Tr2 leave ~2.3e7 non-factor candidates here; the device Tr3 key
    # window (rfr_search_keys2) leaves a handful for verification
    assert res.stats.candidates < 1000


def test_swinnerton_dyer_small_irreducible():
    from paper_2410_15880_b200 import gen_swinnerton_dyer

    for k in (2, 3, 4, 5):
        res = factor(gen_swinnerton_dyer(k))
        assert res.irreducible and res.certificate
        assert res.stats.rejected == res.stats.candidates


def test_factor_errors():
    with pytest.raises(ValueError):
        factor(P([5]))
    with pytest.raises(ValueError):
        factor(P([1, 1]), backend="z")
    with pytest.raises(ValueError):
        factor(P([1, 1]), workers=0)
    rng = random.Random(0)
    big = P([rng.randint(-3, 3) for _ in range(131)] + [1])
    with pytest.raises(WidthExceeded):
        factor(big)
    with pytest.raises(ValueError):
        is_irreducible(P([3]))
    assert is_irreducible(P([7, 1])) and not is_irreducible(P([-1, 0, 1]))


def test_factor_workers_shard_the_search(factor_cases):
    for c in factor_cases[:30]:
        p = poly_of(c["input"])
        assert _got(factor(p, workers=3)) == _want(c), c["tag"]


def test_factor_round_trips_random_products():
    from paper_2410_15880_b200 import multiply

    rng = random.Random(31)
    for _ in range(12):
        fs = [P([rng.randint(-30, 30) for _ in range(rng.randint(1, 9))] + [1]) for _ in range(rng.randint(2, 4))]
        p = fs[0]
        for f in fs[1:]:
            p = multiply(p, f)
        res = factor(p)
        assert res.certificate
        rebuilt = P([res.content])
        for g, m in res.factors:
            rebuilt = rebuilt * g**m
        assert rebuilt == p


def test_device_verification_agrees_with_reference_verdicts(verify_cases):
    """Reference profiles (float64 roots) through the device verifier: every
    candidate the reference accepted passes with the same integer factor, no
    candidate the reference rejected passes."""
    for vc in verify_cases:
        prof = RootProfile(
            real_roots=np.array(rho_of({"rho": vc["real_roots"]})),
            pair_sums=np.array(rho_of({"rho": vc["pair_sums"]})),
            pair_products=np.array(rho_of({"rho": vc["pair_products"]})),
            rho=np.array(rho_of(vc)),
            perm=tuple(vc["perm"]),
            real_lo=np.zeros(len(vc["real_roots"])),
            sum_lo=np.zeros(len(vc["pair_sums"])),
            prod_lo=np.zeros(len(vc["pair_products"])),
            root_err=1e-12,
        )
        p = poly_of(vc["p"])
        pats = np.array([row["pattern"] for row in vc["candidates"]], dtype=np.uint64)
        verdict, side, coeffs = verify_candidates(prof, p, pats)
        full = (1 << prof.n) - 1
        accepted = {row["pattern"]: row["q"] for row in vc["candidates"] if row["q"] is not None}
        for k, row in enumerate(vc["candidates"]):
            s = row["pattern"]
            expect = s in accepted or (~s & full) in accepted
            assert (verdict[k] == _lib.V_PASS) == expect, (vc["tag"], s, int(verdict[k]))
            if expect:
                t = (~s & full) if side[k] else s
                q = accepted[t]
                assert [int(x) for x in coeffs[k, : len(q)]] == [int(x) for x in q]


def test_device_verification_root_error_bound_edges(verify_cases):
    """rfr_verify argument checks: a NaN root error bound is rejected
    (RFR_E_ARG -> ValueError); an infinite one decides nothing on the device
    (no PASS: every non-trivial candidate goes to the host)."""
    vc = verify_cases[0]

    def prof_with(err):
        return RootProfile(
            real_roots=np.array(rho_of({"rho": vc["real_roots"]})),
            pair_sums=np.array(rho_of({"rho": vc["pair_sums"]})),
            pair_products=np.array(rho_of({"rho": vc["pair_products"]})),
            rho=np.array(rho_of(vc)), perm=tuple(vc["perm"]),
            real_lo=np.zeros(len(vc["real_roots"])), sum_lo=np.zeros(len(vc["pair_sums"])),
            prod_lo=np.zeros(len(vc["pair_products"])), root_err=err,
        )

    p = poly_of(vc["p"])
    pats = np.array([row["pattern"] for row in vc["candidates"]], dtype=np.uint64)
    with pytest.raises(ValueError, match="root_err"):
        verify_candidates(prof_with(float("nan")), p, pats)
    verdict, _, _ = verify_candidates(prof_with(float("inf")), p, pats)
    assert not np.any(verdict == _lib.V_PASS)
    assert np.any(verdict == _lib.V_HOST)


def test_fused_search_verify_matches_the_two_call_path(big_inputs, factor_cases):
    """rfr_search_verify (one device call) == rfr_search_keys2 + rfr_verify."""
    from paper_2410_15880_b200 import search_keys
    from paper_2410_15880_b200 import verify as V

    polys = [poly_of(c["p"]) for c in big_inputs["c3"][:2]]
    polys += [poly_of(c["input"]) for c in factor_cases if c["tag"].startswith("c1_")][:3]
    for p in polys:
        prof = V._profile_cached(p.primitive_part().coeffs)
        keys, T = V._search_window(prof)
        keys3, T3 = V._secondary_window(prof)
        pats, verdict, side, coeffs = V.search_and_verify(prof, p.primitive_part(), keys, T, keys3, T3)
        ref = search_keys(keys, T, keys2=keys3, half_width2=T3)
        order = np.argsort(pats)
        assert np.array_equal(pats[order], ref)
        rv, rs, rc = V.verify_candidates(prof, p.primitive_part(), ref)
        assert np.array_equal(verdict[order], rv) and np.array_equal(side[order], rs)
        full = (1 << prof.n) - 1
        for k in np.nonzero(rv == _lib.V_PASS)[0]:
            t = int(ref[k])
            e = V.selected_degree((~t & full) if rs[k] else t, prof)
            # only coefficients 0..e are written (the rest of the row is scratch)
            assert np.array_equal(coeffs[order][k][: e + 1], rc[k][: e + 1])
