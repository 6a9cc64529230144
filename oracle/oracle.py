"""ORACLE -- test infrastructure only (see oracle.c).

ctypes front end of the float64 C restatement of the reference's two-stage
MP-WSD path.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg may import this module; the product package never does.

Accepts the reference's objects or this repo's host-side ones (duck-typed on
`n`, `k`, `kind`, `info_set`, `crc`, `inner`, `generator.words`,
`member_words`).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_two_stage_batch.restype = ctypes.c_int
        _lib.orc_mpwsd_batch.restype = ctypes.c_int
        _lib.orc_scl.restype = ctypes.c_int
        _lib.orc_osd_batch.restype = ctypes.c_int
    return _lib


class _Code(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("k", ctypes.c_int), ("kp", ctypes.c_int),
                ("w64", ctypes.c_int), ("info_set", ctypes.c_void_p), ("gen", ctypes.c_void_p),
                ("is_ca", ctypes.c_int), ("crc_deg", ctypes.c_int), ("crc_poly", ctypes.c_uint32)]


class _Sphere(ctypes.Structure):
    _fields_ = [("size", ctypes.c_int), ("members", ctypes.c_void_p), ("filter_m", ctypes.c_int)]


class _Params(ctypes.Structure):
    _fields_ = [("list_size", ctypes.c_int), ("num_paths", ctypes.c_int),
                ("max_iter", ctypes.c_int), ("gated", ctypes.c_int),
                ("osd_order", ctypes.c_int), ("osd_cap", ctypes.c_int)]


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def default_filter_size(size: int) -> int:
    """decoders.py:94-96 (size counts the zero codeword)."""
    return max(10, math.ceil(0.02 * size))


class OracleCode:
    def __init__(self, code):
        if code.kind == "crc_concatenated":
            inner = code.inner
            crc = code.crc
            bits = np.asarray(crc.coefficients.bits(), dtype=np.int64)
            self.crc_poly = int(sum(int(b) << i for i, b in enumerate(bits)))
            self.crc_deg = int(crc.degree)
            self.is_ca = 1
        elif code.kind == "polar":
            inner = code
            self.crc_poly = 0
            self.crc_deg = 0
            self.is_ca = 0
        else:           # e.g. RM: OSD stage 1 only (no info set, no gate)
            inner = None
            self.crc_poly = 0
            self.crc_deg = 0
            self.is_ca = 0
        self.n = int(code.n)
        self.k = int(code.k)
        self.info = np.ascontiguousarray(inner.info_set if inner is not None else [], dtype=np.int32)
        self.gen = np.ascontiguousarray(code.generator.words, dtype=np.uint64)
        self.w64 = self.gen.shape[1]
        self.struct = _Code(self.n, self.k, int(self.info.size), self.w64, self.info.ctypes.data,
                            self.gen.ctypes.data, self.is_ca, self.crc_deg, self.crc_poly)


class OracleSphere:
    def __init__(self, sphere, filter_size=None):
        self.members = np.ascontiguousarray(sphere.member_words, dtype=np.uint64)
        self.size = self.members.shape[0]
        self.m = int(filter_size) if filter_size is not None else default_filter_size(self.size)
        self.struct = _Sphere(self.size, self.members.ctypes.data, self.m)


def two_stage_batch(y32, code, sphere, list_size, num_paths, max_iter, gated, sigma,
                    nthreads=1, filter_size=None, want_lists=False, want_hops=False,
                    want_anchors=False, osd_order=None, osd_cap=None):
    """Returns a dict of per-frame arrays (stage 0 = stage1_crc_pass, 1 = mp_wsd).
    osd_order set: stage 1 is OsdStage(osd_order, osd_cap) (decoders.py:555-556)."""
    y32 = np.ascontiguousarray(y32, dtype=np.float32)
    F, n = y32.shape
    oc = OracleCode(code)
    os_ = OracleSphere(sphere, filter_size)
    prm = _Params(int(list_size), int(num_paths), int(max_iter), int(bool(gated)),
                  -1 if osd_order is None else int(osd_order), int(osd_cap or 0))
    w64 = oc.w64
    A, T, L = int(num_paths), int(max_iter), int(list_size)
    out = dict(stage=np.zeros(F, np.uint8), best=np.zeros((F, w64), np.uint64),
               best_ed=np.zeros(F, np.float64), n_anchor=np.zeros(F, np.int32),
               iters=np.zeros((F, A), np.int32))
    hops = np.full((F, A, T), -1, np.int32) if want_hops else None
    anchors = np.zeros((F, A, w64), np.uint64) if want_anchors else None
    if want_lists:
        list_n = np.zeros(F, np.int32)
        list_cw = np.zeros((F, L, w64), np.uint64)
        list_pm = np.zeros((F, L), np.float64)
    else:
        list_n = list_cw = list_pm = None
    rc = lib().orc_two_stage_batch(
        ctypes.byref(oc.struct), ctypes.byref(os_.struct), ctypes.byref(prm), _ptr(y32),
        ctypes.c_int(F), ctypes.c_double(sigma), ctypes.c_int(nthreads),
        _ptr(out["stage"]), _ptr(out["best"]), _ptr(out["best_ed"]), _ptr(out["n_anchor"]),
        _ptr(out["iters"]), _ptr(hops), _ptr(anchors), _ptr(list_n), _ptr(list_cw), _ptr(list_pm))
    if rc != 0:
        raise ValueError("oracle rejected the configuration")
    if want_hops:
        out["hops"] = hops
    if want_anchors:
        out["anchors"] = anchors
    if want_lists:
        out["list_n"], out["list_cw"], out["list_pm"] = list_n, list_cw, list_pm
    return out


def mpwsd_batch(y32, anchors, sphere, max_iter, nthreads=1, filter_size=None):
    """anchors uint64 [F, A, W64]."""
    y32 = np.ascontiguousarray(y32, dtype=np.float32)
    anchors = np.ascontiguousarray(anchors, dtype=np.uint64)
    F, n = y32.shape
    _, A, w64 = anchors.shape
    os_ = OracleSphere(sphere, filter_size)
    best = np.zeros((F, w64), np.uint64)
    best_ed = np.zeros(F, np.float64)
    iters = np.zeros((F, A), np.int32)
    hops = np.full((F, A, max_iter), -1, np.int32)
    traj_ed = np.zeros((F, A), np.float64)
    lib().orc_mpwsd_batch(ctypes.byref(os_.struct), ctypes.c_int(n), ctypes.c_int(w64), _ptr(y32),
                          _ptr(anchors), ctypes.c_int(F), ctypes.c_int(A), ctypes.c_int(max_iter),
                          ctypes.c_int(nthreads), _ptr(best), _ptr(best_ed), _ptr(iters),
                          _ptr(hops), _ptr(traj_ed))
    return dict(best=best, best_ed=best_ed, iters=iters, hops=hops, traj_ed=traj_ed)


def osd_batch(y32, code, order, list_cap=None, nthreads=1):
    """osd_decode (decoders.py:274-317) per frame: (list_n, list_cw, list_ed)."""
    y32 = np.ascontiguousarray(y32, dtype=np.float32)
    F, n = y32.shape
    oc = OracleCode(code)
    C = sum(math.comb(oc.k, w) for w in range(min(order, oc.k) + 1))
    cap = C if list_cap is None else min(int(list_cap), C)
    list_n = np.zeros(F, np.int32)
    list_cw = np.zeros((F, cap, oc.w64), np.uint64)
    list_ed = np.zeros((F, cap), np.float64)
    rc = lib().orc_osd_batch(ctypes.byref(oc.struct), _ptr(y32), ctypes.c_int(F), ctypes.c_int(order),
                             ctypes.c_int(cap), ctypes.c_int(nthreads), _ptr(list_n), _ptr(list_cw),
                             _ptr(list_ed))
    if rc != 0:
        raise ValueError("oracle OSD rejected the arguments")
    return list_n, list_cw, list_ed


def scl(llrs, info_set, n, list_size):
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    info = np.ascontiguousarray(info_set, dtype=np.int32)
    w64 = (n + 63) // 64
    u = np.zeros((list_size, n), np.uint8)
    cw = np.zeros((list_size, w64), np.uint64)
    pm = np.zeros(list_size, np.float64)
    cnt = lib().orc_scl(_ptr(llrs), ctypes.c_int(n), _ptr(info), ctypes.c_int(info.size),
                        ctypes.c_int(list_size), _ptr(u), _ptr(cw), _ptr(pm))
    if cnt < 0:
        raise ValueError("oracle SCL rejected the size")
    return u[:cnt], cw[:cnt], pm[:cnt]
