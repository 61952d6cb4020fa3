"""The reference arm of bench.py (oracle/ref_arm.c + ref_arm.py): the
reference's multi-worker factor() path on host threads, pinned to the
reference's own outputs (CPU).

  * parallel_recombine_e port == the reference's recombine_e candidate sets
    (tests/golden/recombine_cases.json, R/parallel.py:255-272 promises the
    serial set for any worker count);
  * the verification loop's first survivor == the reference's verdicts
    (tests/golden/verify_cases.json, R/verify.py:267-284);
  * factor() on the reference's own C3 profile (seed 2, n = 52, eps = 1e-11)
    gives the reference's factors AND its FactorStats counters (candidates,
    rejected) exactly (tests/golden/ref_c3.json, frozen by running the
    reference: tests/golden/make_ref_c3.py)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, rho_of
from oracle import ref_arm as R


@pytest.mark.parametrize("threads", [1, 4])
def test_parallel_recombine_port_equals_reference_sets(recombine_cases, threads):
    for case in recombine_cases:
        rho = rho_of(case)
        if len(rho) < 2:
            continue
        got, _ = R.par_recombine_e(np.array(rho), case["eps"], threads)
        assert set(int(v) for v in got) == set(case["patterns"]), case.get("tag")


def test_verification_loop_first_survivor_matches_reference(verify_cases):
    for vc in verify_cases:
        prof = R.Profile(vc)
        n = prof.n
        rows = {r["pattern"]: r for r in vc["candidates"]}
        canon = np.array(sorted(s for s in rows if s < (1 << (n - 1))), dtype=np.uint64)
        L = R._lib()
        m = L.orc_order_candidates(R._p(canon, R.ctypes.c_uint64), len(canon),
                                   R._p(prof.perm, R.ctypes.c_int), prof.r, n)
        ordered = canon[:m]
        want = next((i for i, s in enumerate(ordered) if rows[int(s)]["q"] is not None), len(ordered))
        idx, q, status = R.verify_first(prof, ordered, vc["p"], vc["eps"], threads=3)
        assert status != 2
        assert idx == want, vc["tag"]
        if idx < len(ordered):
            assert q == [int(c) for c in rows[int(ordered[idx])]["q"]]


def test_factor_port_reproduces_reference_counters_c3_seed2():
    path = os.path.join(GOLDEN, "ref_c3.json")
    with open(path) as fh:
        cases = {c["seed"]: c for c in json.load(fh)["cases"]}
    c = cases[2]
    profiles = {tuple(int(x) for x in c["p"]): c["profile"]}
    for pc, pr in zip(c["pieces"], c["piece_profiles"]):
        profiles[tuple(int(x) for x in pc)] = pr
    st = {}
    fs = R.factor_port(c["p"], profiles, c["eps"], 0, st)
    assert sorted(fs) == sorted([[int(x) for x in f] for f in c["factors"]])
    assert st["candidates"] == c["stats"]["candidates"]
    assert st["rejected"] == c["stats"]["rejected"]
