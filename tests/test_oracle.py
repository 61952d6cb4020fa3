"""The CPU oracle (oracle/) pinned against the reference's own outputs.

The oracle is test infrastructure: the C restatement (oracle/rfr_oracle.c)
and the numpy restatement (oracle/recombine_oracle.py) must reproduce the
golden vectors that tests/golden/make_golden.py froze from the reference
(recombine.py:106-195 / :297-358, verify.py:60-155, polynomial.py:155-183)
before the GPU path is compared with them.
"""
import random

import numpy as np
import pytest

from conftest import rho_of
from oracle import recombine_oracle as O


def test_c_oracle_matches_reference_candidate_sets(recombine_cases):
    for case in recombine_cases:
        rho = rho_of(case)
        assert O.c_recombine(rho, case["eps"]) == frozenset(case["patterns"]), case["tag"]


def test_python_oracle_matches_reference_small(recombine_cases):
    for case in recombine_cases:
        rho = rho_of(case)
        if len(rho) <= 12:
            assert O.canonical_set(rho, case["eps"]) == frozenset(case["patterns"]), case["tag"]


def test_backend_e_port_matches_reference(recombine_cases):
    # the splat/stream port used as the CPU baseline returns the same sets
    for case in recombine_cases:
        rho = rho_of(case)
        if 2 <= len(rho) <= 22:
            assert O.recombine_e_port(rho, case["eps"]) == frozenset(case["patterns"]), case["tag"]


def test_value_accept_kats():
    # R/recombine.py:106-123, test_recombine.py:61-71
    assert O.value(0, [0.3, 0.9]) == 0.0
    assert O.value(0b11, [0.3, 0.9]) == pytest.approx(0.2, abs=1e-12)
    assert O.value(0b101, [0.25, 0.5, 0.75]) == 0.0
    assert O.accept(0.0, 1e-6) and not O.accept(0.5, 1e-6)
    assert not O.accept(1e-6, 1e-6)  # strict
    lib = O.lib()
    vals = np.array([0.25, 0.5, 0.75])
    assert lib.orc_value(O._dp(vals), 3, 0b101) == 0.0


def test_verification_oracle_matches_reference(verify_cases):
    rows = 0
    for vc in verify_cases:
        prof = {
            "real_roots": rho_of({"rho": vc["real_roots"]}),
            "pair_sums": rho_of({"rho": vc["pair_sums"]}),
            "pair_products": rho_of({"rho": vc["pair_products"]}),
            "perm": vc["perm"],
        }
        p = [int(c) for c in vc["p"]]
        for row in vc["candidates"]:
            trace_ok, q = O.verify_candidate(row["pattern"], prof, p, vc["eps"])
            want_q = [int(c) for c in row["q"]] if row["q"] else None
            assert trace_ok == row["trace_ok"] and q == want_q, (vc["tag"], row["pattern"])
            rows += 1
    assert rows > 600


def test_key_window_oracles_agree():
    rng = random.Random(3)
    for _ in range(20):
        n = rng.randint(1, 14)
        keys = np.array([rng.getrandbits(64) for _ in range(n)], dtype=np.uint64)
        T = rng.choice([0, 5, 1 << 40, 1 << 61])
        lo, width = (-T) % (1 << 64), 2 * T
        assert frozenset(int(v) for v in O.c_key_window(keys, lo, width)) == O.key_window_py(keys, lo, width)


def test_divide_exact_oracle():
    assert O.divide_exact([-2, 0, -1, 0, 1], [1, 0, 1]) == [-2, 0, 1]
    assert O.divide_exact([1, 0, 1], [1, 1]) is None
    q = np.zeros(3, dtype=np.int64)
    p = np.array([-2, 0, -1, 0, 1], dtype=np.int64)
    d = np.array([1, 0, 1], dtype=np.int64)
    I = O.lib().orc_divide_exact_i128
    import ctypes

    P64 = ctypes.POINTER(ctypes.c_int64)
    assert I(p.ctypes.data_as(P64), 4, d.ctypes.data_as(P64), 2, q.ctypes.data_as(P64)) == 1
    assert q.tolist() == [-2, 0, 1]
