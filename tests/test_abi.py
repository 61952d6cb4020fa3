"""The C ABI (include/rfr.h) and the host-side native numerics, on CPU.

librfr.so must load and export every function the header declares; the
host-only entry points (root polish, square-free screen, prime table) run
without a GPU.  Device entry points are exercised in the -m gpu suite.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2410_15880_b200 import _lib

HEADER = os.path.join(ROOT, "include", "rfr.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rfr_\w+)\s*\(", text, re.M)))


def test_header_declares_the_exported_set():
    assert header_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rfr_\w+)$", out, re.M))
    for name in header_functions():
        assert name in exported, name
        assert hasattr(lib, name)


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of rfr_stats and rfr_profile have the header's size
    and field offsets (a C program compiled against include/rfr.h prints
    them), so no argument is misread across the boundary."""
    structs = {"rfr_stats": _lib.RfrStats, "rfr_profile": _lib.RfrProfile}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rfr.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.dirname(HEADER), "-o", str(exe), str(src)],
                   check=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n"):
        if line:
            cname, field, val = line.split()
            got[(cname, field)] = int(val)
    for cname, cls in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)


def test_library_is_built_for_sm_100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_primes():
    lib = _lib.load()
    assert lib.rfr_version() >= 1
    primes = np.zeros(3, dtype=np.uint64)
    assert lib.rfr_verify_primes(primes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))) == 0
    import sympy

    # primes below 2^63 of the form 2^k - c, c small (the verify kernel's
    # two-fold reduction needs z < 2P after folding: c + c^2 << P)
    for q in (int(v) for v in primes):
        k = q.bit_length()
        assert sympy.isprime(q) and q < (1 << 63)
        assert (1 << k) - q < (1 << 10)
    assert len(set(int(v) for v in primes)) == 3


def _polish(coeffs, seeds):
    lib = _lib.load()
    d = len(coeffs) - 1
    D = ctypes.POINTER(ctypes.c_double)
    ch = np.array(coeffs, dtype=np.float64)
    cl = np.zeros(d + 1)
    rh = np.array([z.real for z in seeds])
    ih = np.array([z.imag for z in seeds])
    rl, il, err = np.zeros(d), np.zeros(d), np.zeros(d)
    rc = lib.rfr_polish_roots(ch.ctypes.data_as(D), cl.ctypes.data_as(D), d, rh.ctypes.data_as(D),
                              rl.ctypes.data_as(D), ih.ctypes.data_as(D), il.ctypes.data_as(D),
                              err.ctypes.data_as(D), 60)
    return rc, rh, rl, ih, il, err


def test_polish_roots_double_double():
    # x^2 - 2: sqrt(2) to ~106 bits from 1e-3 seeds
    rc, rh, rl, ih, il, err = _polish([-2, 0, 1], [1.415 + 0.001j, -1.413 - 0.001j])
    assert rc == 0
    from fractions import Fraction

    i = int(np.argmax(rh))
    r = Fraction(rh[i]) + Fraction(rl[i])
    assert abs(r * r - 2) < Fraction(1, 10**28)
    assert err[i] < 1e-28


def test_polish_roots_rejects_non_monic_and_bad_args():
    lib = _lib.load()
    D = ctypes.POINTER(ctypes.c_double)
    c = np.array([1.0, 2.0])
    z = np.zeros(1)
    assert lib.rfr_polish_roots(c.ctypes.data_as(D), None, 1, z.ctypes.data_as(D), None,
                                z.ctypes.data_as(D), None, z.ctypes.data_as(D), 5) == _lib.RFR_E_ARG


def test_squarefree_screen():
    lib = _lib.load()
    q = 2305843009213693951
    P = ctypes.POINTER(ctypes.c_uint64)

    def sf(coeffs):
        a = np.array([c % q for c in coeffs], dtype=np.uint64)
        return lib.rfr_squarefree_mod(a.ctypes.data_as(P), len(coeffs) - 1, q)

    assert sf([-2, 0, -1, 0, 1]) == 1        # (x^2-2)(x^2+1)
    assert sf([2, -3, 0, 1]) == 0            # (x-1)^2 (x+2)
    assert sf([1, -2, 1]) == 0               # (x-1)^2
    assert sf([7, 1]) == 1


def test_device_calls_fail_loudly_without_a_gpu():
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    from paper_2410_15880_b200 import RhoVector, recombine_e
    from paper_2410_15880_b200.errors import RecombineDeviceError

    with pytest.raises(RecombineDeviceError):
        recombine_e(RhoVector.from_values([0.25, 0.75]), 1e-6)
