"""Device time of small searches (n <= 36) by kernel variant: the table
search with RFR_TABLE_BITS b (or the default choice) against the Gray-code
brute force (RFR_SMALL_EXHAUSTIVE=1).  One subprocess per variant (the
library reads its switches once).

    python tools/small_search_bench.py > profiles/<round>_small_search.txt
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import ctypes, json, sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_15880_b200 import _lib
lib = _lib.load(); _lib.device()
out = {}
for n in (16, 20, 24, 27, 28, 30, 32, 34, 36):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    T = 256
    lo, width = (-T) %% (1 << 64), 2 * T
    buf = np.empty(1 << 12, dtype=np.uint64)
    ms = []
    for rep in range(8):
        nout = ctypes.c_int64(0); st = _lib.RfrStats()
        _lib.check(lib.rfr_search_keys(_lib.ptr(keys, _lib.U64_P), n, lo, width, 0, 1,
                   _lib.ptr(buf, _lib.U64_P), len(buf), ctypes.byref(nout), ctypes.byref(st)), "s")
        ms.append(st.ms_total)
    out[n] = round(sorted(ms)[len(ms) // 2] * 1e3, 1)
print(json.dumps(out))
""" % ROOT


def run(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=e)
    return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]


print("device microseconds per search (median of 8), window 513 units")
print("brute force", run({"RFR_SMALL_EXHAUSTIVE": "1"}))
print("table default", run({}))
print("join (lists + bucket join)", run({"RFR_FORCE_JOIN": "1"}))
for b in (8, 10):
    print(f"table b={b}", run({"RFR_TABLE_BITS": str(b)}))
