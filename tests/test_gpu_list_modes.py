"""The quarter-list build has launch variants chosen per level or by
environment (read once per process, so each runs in its own subprocess):
merge-path splits from the separate split kernel (levels of >= 1024 tiles by
default; RFR_SPLIT_MIN_TILES=0: every level; a huge value: none), TMA
bulk-copy staging (RFR_MERGE_TMA=1) and plain launches instead of
programmatic ones (RFR_PDL=0).  Every variant must give the same hit set at a
width (n = 48) whose top level has 1024 tiles, and the same as the
exhaustive kernel at n = 40."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SNIPPET = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2410_15880_b200 import search_keys
rng = np.random.default_rng({seed})
keys = rng.integers(0, 2**64 - 1, size={n}, dtype=np.uint64, endpoint=True)
hits = search_keys(keys, {T})
print(json.dumps([int(h) for h in hits]))
"""

MODES = [
    {},
    {"RFR_SPLIT_MIN_TILES": "0"},
    {"RFR_SPLIT_MIN_TILES": "4294967295"},
    {"RFR_MERGE_TMA": "1", "RFR_SPLIT_MIN_TILES": "4294967295"},
    {"RFR_PDL": "0"},
]


def _run(n, seed, T, env_extra):
    env = dict(os.environ)
    for k in ("RFR_SPLIT_MIN_TILES", "RFR_SPLIT_KERNEL", "RFR_MERGE_TMA", "RFR_PDL",
              "RFR_FORCE_EXHAUSTIVE"):
        env.pop(k, None)
    env.update(env_extra)
    code = _SNIPPET.format(root=ROOT, seed=seed, n=n, T=T)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return np.array(json.loads(out.stdout.strip().splitlines()[-1]), dtype=np.uint64)


@pytest.mark.parametrize("n,seed,hits", [(48, 4801, 256), (40, 4001, 512)])
def test_list_build_variants_same_hits(n, seed, hits):
    T = hits << (64 - n)
    ref = _run(n, seed, T, {})
    assert hits // 3 <= len(ref) <= hits * 3, len(ref)
    for mode in MODES[1:]:
        got = _run(n, seed, T, {**mode, "RFR_FORCE_JOIN": "1"})
        assert np.array_equal(got, ref), mode
    if n <= 40:
        ex = _run(n, seed, T, {"RFR_FORCE_EXHAUSTIVE": "1"})
        assert np.array_equal(ex, ref)
