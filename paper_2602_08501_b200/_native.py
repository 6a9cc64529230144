"""ctypes binding of libmpwsd.so (include/mpwsd.h).  Loading fails loudly:
there is no CPU fallback for the decoder path."""

from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPW_LIB") or os.path.join(_HERE, "libmpwsd.so")   # MPW_LIB: A/B builds
HEADER = os.path.join(_HERE, "..", "include", "mpwsd.h")

c_int, c_double, c_void_p, c_uint32, c_int64, c_uint64 = (
    ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64)

MODE_CRC_GATED, MODE_ALWAYS_ON = 0, 1
HOP_AUTO, HOP_GATHER, HOP_TENSOR, HOP_TENSOR_2LIMB, HOP_TENSOR_I8, HOP_TENSOR_I8_ASYNC = 0, 1, 2, 3, 4, 5
CTR_FRAMES, CTR_ERRORS, CTR_ACTIVATIONS, CTR_ITERATIONS, CTR_EVALS, CTR_NEAR_TIE, CTR_UNRESOLVED = range(7)
FLAG_TIE_ARGMIN, FLAG_TIE_ACCEPT, FLAG_TIE_FINAL, FLAG_UNRESOLVED = 1, 2, 4, 8
FLAG_TIE_STAGE1 = 16
NUM_COUNTERS = 8

_SIGS = {
    "mpw_version": (c_int, []),
    "mpw_last_error": (ctypes.c_char_p, []),
    "mpw_create": (c_int, [c_int, ctypes.POINTER(c_void_p)]),
    "mpw_destroy": (None, [c_void_p]),
    "mpw_set_code": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_uint32]),
    "mpw_set_patterns": (c_int, [c_void_p, c_void_p, c_int]),
    "mpw_scl_batch": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_double, c_int,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_mpwsd_batch": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_two_stage_batch": (c_int, [c_void_p, c_void_p, c_int, c_double, c_int, c_int, c_int, c_int,
                                    c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_mpwsd_batch_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_two_stage_batch_f64": (c_int, [c_void_p, c_void_p, c_int, c_double, c_int, c_int, c_int, c_int,
                                        c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_launch_count": (ctypes.c_longlong, [c_void_p]),
    "mpw_two_stage_batch_host": (c_int, [c_void_p, c_void_p, c_int, c_double, c_int, c_int, c_int,
                                         c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_set_timing": (c_int, [c_void_p, c_int]),
    "mpw_set_option": (c_int, [c_void_p, ctypes.c_char_p, c_int]),
    "mpw_read_timing": (c_int, [c_void_p, c_void_p, c_void_p, c_int]),
    "mpw_hop_tile_stats": (c_int, [c_void_p, c_void_p, c_int]),
    "mpw_num_patterns": (c_int, [c_void_p]),
    "mpw_channel_batch": (c_int, [c_void_p, c_uint64, c_int, ctypes.c_longlong, c_int, c_double,
                                  c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_tensor_path_ready": (c_int, [c_void_p]),
    "mpw_hop_auto_variant": (c_int, [c_void_p]),
    "mpw_enumerate_lowweight": (c_int64, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int64, c_int]),
    "mpw_two_stage_osd_batch": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mpw_osd_batch": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p]),
    "mpw_enumerate_lowweight_gpu": (c_int64, [c_void_p, c_int, c_void_p, c_void_p, c_int64]),
    "mpw_collect_lowweight": (c_int64, [c_void_p, c_int, c_int, c_int, c_int64, c_uint64, c_int,
                                        c_void_p, c_int64, c_int]),
}

_lib = None


class NativeError(RuntimeError):
    pass


def declared_symbols() -> list:
    """Function names declared in include/mpwsd.h."""
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(mpw_[a-z0-9_]+)\s*\(", text)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                              "(the decoder has no CPU fallback)")
        _lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().mpw_last_error()
        raise NativeError(f"{what or 'libmpwsd'} failed ({rc}): {msg.decode() if msg else ''}")


def value_error_check(rc: int, what: str = "") -> None:
    """Argument errors surface as ValueError, like the reference API."""
    if rc == -1 or rc == -3:
        msg = lib().mpw_last_error()
        raise ValueError(f"{what}: {msg.decode() if msg else ''}")
    check(rc, what)
