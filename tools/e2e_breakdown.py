"""Where factor()'s e2e time goes beyond the device time (C3, d = 100 inputs).

Per input, the median of 20 factorizations (roots cached, excluded as in
bench.py): e2e through factor(), the wall time of the fused C calls
(rfr_search_verify via _search_and_verify: the main search and, after an
early exit, the searches of the two pieces), and the device span the
library records with CUDA events (lists -> verification), summed over them.  Then a cProfile of 50
factorizations of the first input for the Python side.

    python tools/e2e_breakdown.py > profiles/<round>_e2e_breakdown.txt
"""
import cProfile
import io
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_15880_b200 import factor  # noqa: E402
from paper_2410_15880_b200 import verify as V  # noqa: E402


def main():
    c3, _ = bench.load_inputs()
    inner = V._search_and_verify
    calls = []

    def timed(*a, **k):
        t0 = time.perf_counter()
        out = inner(*a, **k)
        calls.append((time.perf_counter() - t0) * 1e3)
        return out

    V._search_and_verify = timed
    print("seed  e2e_ms  c_call_ms  device_ms  python_ms  c_host_ms  candidates  early_exits")
    for seed, p, _ in c3:
        for _ in range(3):
            factor(p)
        calls.clear()
        e2e, dev, call = [], [], []
        for _ in range(20):
            calls.clear()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = factor(p)
            torch.cuda.synchronize()
            e2e.append((time.perf_counter() - t0 - res.stats.root_seconds) * 1e3)
            dev.append(res.stats.recombine.device_ms)
            call.append(sum(calls))
        e, c, d = np.median(e2e), np.median(call), np.median(dev)
        print(f"{seed:4d}  {e:6.3f}  {c:9.3f}  {d:9.3f}  {e - c:9.3f}  {c - d:9.3f}  "
              f"{res.stats.candidates:10d}  {res.stats.early_exits:11d}", flush=True)
    V._search_and_verify = inner
    seed, p, _ = c3[0]
    prof = cProfile.Profile()
    prof.enable()
    for _ in range(50):
        factor(p)
    prof.disable()
    buf = io.StringIO()
    pstats.Stats(prof, stream=buf).sort_stats("tottime").print_stats(15)
    print(buf.getvalue())


if __name__ == "__main__":
    main()
