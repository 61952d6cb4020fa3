"""Drive the latency-bound kernels of the e2e path for an ncu capture: a
whole n = 54 search (lists_base_kernel, join_starts_kernel) and an n = 27
small search (table_search_kernel, the body the device piece search runs).

    ncu --set full -k regex:'table_search|lists_base|join_starts' -c 6 \\
        -o gpurun_out/small python tools/ncu_small_kernels.py
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15880_b200 import _lib  # noqa: E402

lib = _lib.load()
_lib.device()
for n in (54, 27, 27, 54):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    T = 256
    lo, width = (-T) % (1 << 64), 2 * T
    buf = np.empty(1 << 14, dtype=np.uint64)
    nout = ctypes.c_int64(0)
    st = _lib.RfrStats()
    _lib.check(lib.rfr_search_keys(_lib.ptr(keys, _lib.U64_P), n, lo, width, 0, 1,
                                   _lib.ptr(buf, _lib.U64_P), len(buf), ctypes.byref(nout),
                                   ctypes.byref(st)), "search")
    print(n, nout.value, st.ms_total)
