"""Freeze the REFERENCE's own inputs and counters for the C3 benchmark
(d = 100, gen_random_reducible_parts(100, 100, seed), seeds 0-4) into
tests/golden/ref_c3.json, by running the reference package in this container.

`bench.py --impl reference` (the CPU arm timed on the GPU box, where the
reference cannot be imported) replays the reference's factor() path from
these: its own root profile of p (find_roots + build_profile,
pkg/src/polyfactor/rootfinder.py:100-245) and of both factors (the recursion
re-roots each piece, verify.py:257, :280-284), so the timed port searches
exactly the rho vector the reference searches.  The reference's own
factor(p, ToleranceConfig(eps=1e-11)) counters (candidates, rejected,
stage seconds) pin the port (tests/test_ref_arm.py): at the default eps
(1e-6) the reference cannot run d = 100 (~3.6e10 candidates, SURVEY.md
s7.2 H1); 1e-11 is the setting at which it completes (~10 min per seed).

Run (this container only; ~12 GB RAM and ~10 min per seed):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_ref_c3.py SEED      # one seed -> ref_c3_SEED.json
    python tests/golden/make_ref_c3.py merge         # -> ref_c3.json
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
EPS = 1e-11


def profile_json(prof):
    return {
        "real_roots": [float(v).hex() for v in prof.real_roots],
        "pair_sums": [float(v).hex() for v in prof.pair_sums],
        "pair_products": [float(v).hex() for v in prof.pair_products],
        "rho": [float(v).hex() for v in prof.rho],
        "perm": [int(v) for v in prof.perm],
    }


def one(seed: int) -> None:
    from polyfactor import ToleranceConfig, factor, gen_random_reducible_parts, profile_polynomial

    f, g = gen_random_reducible_parts(100, 100, seed)
    p = f * g
    cfg = ToleranceConfig(eps=EPS)
    t0 = time.perf_counter()
    res = factor(p, cfg, backend="e", workers=1)
    wall = time.perf_counter() - t0
    st = res.stats
    rec = {
        "seed": seed,
        "eps": EPS,
        "p": [str(c) for c in p.coeffs],
        "factors": [[str(c) for c in h.coeffs] for h, _ in res.factors],
        "certificate": bool(res.certificate),
        "profile": profile_json(profile_polynomial(p, cfg)),
        "piece_profiles": [profile_json(profile_polynomial(h, cfg)) for h in (f, g)],
        "pieces": [[str(c) for c in h.coeffs] for h in (f, g)],
        "stats": {
            "n": st.n if hasattr(st, "n") else None,
            "candidates": int(st.candidates),
            "rejected": int(st.rejected),
            "root_seconds": st.root_seconds,
            "recombine_seconds": st.recombine_seconds,
            "verify_seconds": st.verify_seconds,
            "wall_seconds": wall,
        },
    }
    with open(os.path.join(HERE, f"ref_c3_{seed}.json"), "w") as fh:
        json.dump(rec, fh, separators=(",", ":"))
    print(f"seed {seed}: {wall:.1f}s, candidates {st.candidates}, rejected {st.rejected}")


def merge() -> None:
    out = []
    for seed in range(5):
        with open(os.path.join(HERE, f"ref_c3_{seed}.json")) as fh:
            out.append(json.load(fh))
    path = os.path.join(HERE, "ref_c3.json")
    with open(path, "w") as fh:
        json.dump({"eps": EPS, "cases": out}, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    if sys.argv[1] == "merge":
        merge()
    else:
        one(int(sys.argv[1]))
