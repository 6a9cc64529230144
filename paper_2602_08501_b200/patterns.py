"""Pattern-set (sphere) generation through the native host tools
(csrc/sphere_tools.cpp); off the timed path.

* `enumerate_sphere(code, r)`: exhaustive 2^K walk, the reference's
  `build_sphere` (wsphere.py:175-208) -- same members, same CWS1 order.
* `enumerate_sphere_gpu(code, r)`: the same walk on the device
  (csrc/enum.cuh, K <= 40).
* `collect_sphere(code, cap, ...)`: seeded information-set search for K > 30
  (BASELINE config 4), where the reference's enumeration budget
  (ENUM_DIM_LIMIT = 30, wsphere.py:28) refuses.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native
from .bits import num_words
from .sphere import sphere_from_members


def weight_spectrum(code, threads: int = 0) -> np.ndarray:
    g = np.ascontiguousarray(code.generator.words, dtype=np.uint64)
    spec = np.zeros(code.n + 1, np.int64)
    rc = _native.lib().mpw_enumerate_lowweight(g.ctypes.data, code.k, code.n, 0, spec.ctypes.data,
                                               None, 0, threads or (os.cpu_count() or 1))
    if rc < 0:
        raise ValueError(f"K = {code.k} is outside the enumeration budget")
    return spec


def enumerate_sphere(code, radius_index: int, threads: int = 0):
    spec = weight_spectrum(code, threads)
    shells = [w for w in range(1, code.n + 1) if spec[w]]
    if radius_index < 0 or radius_index > len(shells):
        raise ValueError(f"radius index {radius_index} exceeds the {len(shells)} available shells")
    cap = shells[radius_index - 1] if radius_index > 0 else 0
    total = int(sum(spec[1:cap + 1])) if cap else 0
    g = np.ascontiguousarray(code.generator.words, dtype=np.uint64)
    out = np.zeros((max(total, 1), num_words(code.n)), np.uint64)
    if total:
        got = _native.lib().mpw_enumerate_lowweight(g.ctypes.data, code.k, code.n, cap, None,
                                                    out.ctypes.data, total, threads or (os.cpu_count() or 1))
        if got != total:
            raise RuntimeError("enumeration count mismatch")
    return sphere_from_members(code.n, code.k, radius_index, out[:total])


def enumerate_sphere_gpu(code, radius_index: int, device=None):
    """`enumerate_sphere` on the GPU (csrc/enum.cuh): same members, same CWS1
    order (sorted on the host), for K <= 40."""
    from .decoders import DeviceDecoder
    dec = DeviceDecoder(code, device=device)
    try:
        spec, _ = dec.enumerate_lowweight(0)
        shells = [w for w in range(1, code.n + 1) if spec[w]]
        if radius_index < 0 or radius_index > len(shells):
            raise ValueError(f"radius index {radius_index} exceeds the {len(shells)} available shells")
        cap = shells[radius_index - 1] if radius_index > 0 else 0
        _, words = dec.enumerate_lowweight(cap)
    finally:
        dec.close()
    return sphere_from_members(code.n, code.k, radius_index, words)


def weight_spectrum_gpu(code, device=None) -> np.ndarray:
    from .decoders import DeviceDecoder
    dec = DeviceDecoder(code, device=device)
    try:
        return dec.enumerate_lowweight(0)[0]
    finally:
        dec.close()


def collect_sphere(code, weight_cap: int, iterations: int = 50000, seed: int = 20260208,
                   p_max: int = 3, threads: int = 0, max_words: int = 1 << 22):
    g = np.ascontiguousarray(code.generator.words, dtype=np.uint64)
    out = np.zeros((max_words, num_words(code.n)), np.uint64)
    got = _native.lib().mpw_collect_lowweight(g.ctypes.data, code.k, code.n, weight_cap, iterations,
                                              ctypes.c_uint64(seed), p_max, out.ctypes.data, max_words,
                                              threads or (os.cpu_count() or 1))
    if got < 0:
        raise ValueError("collector rejected the arguments")
    if got > max_words:
        raise RuntimeError("collector output exceeded max_words")
    words = out[:got]
    shells = np.unique(np.bitwise_count(words).sum(axis=1)) if got else []
    return sphere_from_members(code.n, code.k, len(shells), words)
