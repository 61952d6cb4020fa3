"""ctypes binding of librfr.so (the C ABI declared in include/rfr.h).

The extension is built in-tree (``make -C paper_2410_15880_b200/csrc`` or
``__graft_entry__.build()``) and loaded from this package directory.  There
is no CPU fallback: every entry point raises when the library or a CUDA
device is missing, so a GPU test can never pass on a silent substitute.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import RecombineDeviceError, WidthExceeded

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librfr.so")

RFR_OK, RFR_E_ARG, RFR_E_WIDTH, RFR_E_CAP, RFR_E_CUDA, RFR_E_NOINIT, RFR_E_NUMERIC = range(7)
V_REJECT, V_PASS, V_HOST = 0, 1, 2

# every symbol include/rfr.h declares (tests/test_abi.py checks the export table)
EXPORTS = (
    "rfr_init",
    "rfr_shutdown",
    "rfr_last_error",
    "rfr_version",
    "rfr_num_sms",
    "rfr_recombine_e",
    "rfr_search_keys",
    "rfr_search_keys2",
    "rfr_search_verify",
    "rfr_search_verify_shard",
    "rfr_peer_handle",
    "rfr_peer_connect",
    "rfr_peer_disconnect",
    "rfr_search_keys_dev",
    "rfr_verify",
    "rfr_verify_primes",
    "rfr_polish_roots",
    "rfr_squarefree_mod",
    "rfr_squarefree_i64",
    "rfr_divide_monic_i64",
    "rfr_p_mod_i64",
    "rfr_multiply_i64",
)


class RfrStats(ctypes.Structure):
    """Mirror of rfr_stats (include/rfr.h)."""

    _fields_ = [
        ("visited", ctypes.c_int64),
        ("inserts", ctypes.c_int64),
        ("insert_probes", ctypes.c_int64),
        ("queries", ctypes.c_int64),
        ("query_probes", ctypes.c_int64),
        ("raw_hits", ctypes.c_int64),
        ("buckets", ctypes.c_int64),
        ("chunks", ctypes.c_int64),
        ("r_bits", ctypes.c_int32),
        ("windows", ctypes.c_int32),
        ("ms_lists", ctypes.c_double),
        ("ms_join", ctypes.c_double),
        ("ms_post", ctypes.c_double),
        ("ms_total", ctypes.c_double),
        ("launches", ctypes.c_int64),
        ("buckets_planned", ctypes.c_int64),
        ("early_stop", ctypes.c_int64),
        ("list_bits", ctypes.c_int32 * 4),
        ("bytes_lists", ctypes.c_int64),
        ("bytes_join", ctypes.c_int64),
        ("us_hit_to_stop", ctypes.c_double),
        ("pieces", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        out = {name: getattr(self, name) for name, _ in self._fields_}
        out["list_bits"] = list(self.list_bits)
        return out


class RfrProfile(ctypes.Structure):
    """Mirror of rfr_profile (include/rfr.h)."""

    _fields_ = [
        ("n", ctypes.c_int),
        ("r", ctypes.c_int),
        ("c", ctypes.c_int),
        # device-visible host addresses of the profile arrays (const double*,
        # const int32_t* in the header; plain addresses here, set from numpy)
        ("real_hi", ctypes.c_void_p),
        ("real_lo", ctypes.c_void_p),
        ("sum_hi", ctypes.c_void_p),
        ("sum_lo", ctypes.c_void_p),
        ("prod_hi", ctypes.c_void_p),
        ("prod_lo", ctypes.c_void_p),
        ("perm", ctypes.c_void_p),
        ("root_err", ctypes.c_double),
    ]


_lib = None
_lock = threading.Lock()
_device = None

D_P = ctypes.POINTER(ctypes.c_double)
U64_P = ctypes.POINTER(ctypes.c_uint64)
I64_P = ctypes.POINTER(ctypes.c_int64)
U8_P = ctypes.POINTER(ctypes.c_uint8)
I32_P = ctypes.POINTER(ctypes.c_int32)


def load():
    """Load librfr.so and declare the prototypes (no device work)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RecombineDeviceError(
                f"{LIB_PATH} is missing: build it with `make -C {HERE}/csrc` "
                "(there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        L.rfr_init.argtypes = [ctypes.c_int]
        L.rfr_shutdown.argtypes = []
        L.rfr_last_error.restype = ctypes.c_char_p
        L.rfr_version.restype = ctypes.c_int
        L.rfr_num_sms.restype = ctypes.c_int
        L.rfr_recombine_e.argtypes = [
            D_P, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, U64_P,
            ctypes.c_int64, I64_P, ctypes.POINTER(RfrStats),
        ]
        L.rfr_search_keys.argtypes = [
            U64_P, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
            U64_P, ctypes.c_int64, I64_P, ctypes.POINTER(RfrStats),
        ]
        L.rfr_search_keys2.argtypes = [
            U64_P, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, U64_P, ctypes.c_uint64,
            ctypes.c_uint64, ctypes.c_int, ctypes.c_int, U64_P, ctypes.c_int64, I64_P,
            ctypes.POINTER(RfrStats),
        ]
        L.rfr_search_keys_dev.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.POINTER(RfrStats),
        ]
        missing = [name for name in EXPORTS if not hasattr(L, name)]
        if missing:
            raise RecombineDeviceError(f"{LIB_PATH} lacks exports {missing}: rebuild it")
        L.rfr_verify.argtypes = [
            ctypes.POINTER(RfrProfile), U64_P, ctypes.c_int64, U64_P, ctypes.c_int, U8_P, U8_P,
            I64_P, ctypes.c_int, ctypes.POINTER(RfrStats),
        ]
        # array arguments as void*: raw addresses (int) are the cheapest to pass
        # per call; ctypes pointer instances are accepted as well
        VP = ctypes.c_void_p
        L.rfr_search_verify.argtypes = [
            VP, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, VP, ctypes.c_uint64,
            ctypes.c_uint64, ctypes.POINTER(RfrProfile), VP, ctypes.c_int, VP, VP, VP,
            VP, ctypes.c_int, ctypes.c_int64, ctypes.c_int, I64_P, ctypes.POINTER(RfrStats),
        ]
        L.rfr_search_verify_shard.argtypes = [
            VP, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, VP, ctypes.c_uint64,
            ctypes.c_uint64, ctypes.POINTER(RfrProfile), VP, ctypes.c_int, VP, VP, VP,
            VP, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_uint64, I64_P, ctypes.POINTER(RfrStats),
        ]
        L.rfr_p_mod_i64.argtypes = [VP, ctypes.c_int, VP]
        L.rfr_multiply_i64.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                       ctypes.c_void_p]
        L.rfr_peer_handle.argtypes = [ctypes.c_void_p]
        L.rfr_peer_connect.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.rfr_peer_disconnect.argtypes = []
        L.rfr_verify_primes.argtypes = [U64_P]
        L.rfr_polish_roots.argtypes = [D_P, D_P, ctypes.c_int, D_P, D_P, D_P, D_P, D_P, ctypes.c_int]
        L.rfr_squarefree_mod.argtypes = [U64_P, ctypes.c_int, ctypes.c_uint64]
        # raw address (int): the per-call pointer wrapping costs more than the screen
        L.rfr_squarefree_i64.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64]
        L.rfr_divide_monic_i64.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                           ctypes.c_void_p]
        _lib = L
        return L


def last_error() -> str:
    return load().rfr_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc == RFR_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == RFR_E_WIDTH:
        raise WidthExceeded(msg)
    if rc == RFR_E_ARG:
        raise ValueError(msg)
    raise RecombineDeviceError(msg)


def device() -> int:
    """Initialise the engine on this process's CUDA device (LOCAL_RANK or 0)."""
    global _device
    L = load()
    if _device is None:
        dev = int(os.environ.get("RFR_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        check(L.rfr_init(dev), "rfr_init")
        _device = dev
    return _device


def ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)
