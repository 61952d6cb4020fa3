"""One-GPU emulation of the N-rank sharded search of C4 (d = 120, seed 0,
n = 63): each rank of an N-way plan builds the whole quarter lists and joins
its 1/N of the buckets, and the ranks do not communicate until the final
all-gather, so a rank's device time can be measured alone.  Runs shard 0
and shard N-1 of each plan (the two ends of the key space) and reports the
per-rank lists / join time and the whole-job pairs/s and efficiency.

    python tools/shard_emulation.py > profiles/<round>_shard_emulation.txt
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_15880_b200 import _lib  # noqa: E402
from paper_2410_15880_b200.verify import _profile_cached, _search_window  # noqa: E402


def main():
    lib = _lib.load()
    _lib.device()
    _, c4 = bench.load_inputs()
    prof = _profile_cached(c4[0][1].coeffs)
    keys, T = _search_window(prof)
    d_keys = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    lo, w = (-T) % (1 << 64), 2 * T
    cap = 1 << 16
    d_out = torch.empty(cap, dtype=torch.int64, device="cuda")
    d_cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    pairs = 2.0 ** (prof.n - 1)
    print(f"C4 seed 0, n = {prof.n}: device ms per rank (min of 3), lists + join of shard 0 and shard N-1")
    print(f"{'N':>3} {'lists':>8} {'join s0':>8} {'join sN':>8} {'rank':>8} {'pairs/s (job)':>14} {'eff':>5}")
    base = None
    for N in (1, 2, 4, 8):
        res = []
        for shard in sorted({0, N - 1}):
            best = None
            for _ in range(3):
                st = _lib.RfrStats()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _lib.check(lib.rfr_search_keys_dev(
                    ctypes.c_void_p(d_keys.data_ptr()), prof.n, lo, w, shard, N,
                    ctypes.c_void_p(d_out.data_ptr()), cap, ctypes.c_void_p(d_cnt.data_ptr()),
                    ctypes.c_void_p(stream.cuda_stream), ctypes.byref(st)), "search")
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                if best is None or ms < best[0]:
                    best = (ms, st.ms_lists, st.ms_join)
            res.append(best)
        rank = max(r[0] for r in res)
        job = pairs / (rank * 1e-3)
        base = base or job
        print(f"{N:>3} {res[0][1]:8.2f} {res[0][2]:8.2f} {res[-1][2]:8.2f} {rank:8.2f} {job:14.3e} "
              f"{job / base / N:5.2f}")


if __name__ == "__main__":
    main()
