"""Drop-in for the reference's decoder API on the B200 path.

Same names, arguments, return types and errors as
/root/reference/pkg/src/feclab/decoders.py (re-exported by its __init__.py:28-39):

  scl_decode(llrs, code, list_size, counters=None)                 decoders.py:181-268
  wsd_step(y, center, x_center, sphere, m, counters=None)          decoders.py:401-417
  wsd_trajectory(y, c0, sphere, params, counters=None, ...)        decoders.py:420-452
  mp_wsd(y, init_list, sphere, params, counters=None)              decoders.py:455-514
  two_stage_decode(y, code, stage1, params, sphere, sigma=1.0, counters=None)
                                                                   decoders.py:520-583

plus the throughput entry point `DeviceDecoder.two_stage_batch` /
`two_stage_decode_batch` over [F, N] batches.  Every call runs the sm_100a
kernels of libmpwsd.so; there is no CPU fallback (a missing library or GPU
raises).  Batches of float32 received words run the float32 path (the
bench's dtype); float64 received words -- what the per-frame API receives,
since the reference coerces y to float64 (decoders.py:411, 466, 538) -- run
the *_f64 entry points: stage 1 from the float64 LLRs, hop screens on the
fp32 rounding with widened error bounds, exact re-scoring and every ED from
the float64 values.  Stage 1 is bit-exact with the reference (float64 path
metrics); hop decisions equal exact arithmetic, near-ties (|ΔED| gaps < 1e-5
relative) are reported per frame.

Thread safety: the reference's sweep calls these functions from a thread
pool (simharness.py:318-330).  A libmpwsd handle serves one host thread at a
time, so the per-frame functions keep one DeviceDecoder per (thread, code,
sphere) and issue their work on that thread's current torch stream.

Code and sphere arguments may be this package's objects or the reference's
(duck-typed on n, k, kind, info_set, crc, inner, generator.words,
member_words).
"""

from __future__ import annotations

import ctypes
import math
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from .bits import BitVector, num_words, pack_bits, unpack_bits
from .codes import crc_poly_int, message_words, inverse_tables, polar_transform_bits

# ---------------------------------------------------------------------------
# Parameter / result types (decoders.py:37-118)


@dataclass
class CandidateList:
    entries: list

    def __post_init__(self):
        scores = [s for _, s in self.entries]
        if any(a > b for a, b in zip(scores, scores[1:])):
            raise ValueError("candidate scores must be nondecreasing")

    def __len__(self) -> int:
        return len(self.entries)


@dataclass(frozen=True)
class SclStage:
    list_size: int


@dataclass(frozen=True)
class OsdStage:
    order: int
    list_cap: int | None = None


def default_filter_size(sphere_size: int) -> int:
    """max(10, ceil(0.02 |S|)) (decoders.py:94-96)."""
    return max(10, math.ceil(0.02 * sphere_size))


@dataclass
class WsdParams:
    radius_index: int
    filter_size: int | None = None
    max_iterations: int = 4
    num_paths: int = 4
    activation_mode: str = "crc_gated"

    def __post_init__(self):
        if self.max_iterations < 1 or self.num_paths < 1:
            raise ValueError("max_iterations and num_paths must be >= 1")
        if self.filter_size is not None and self.filter_size < 1:
            raise ValueError("filter_size must be >= 1")
        if self.activation_mode not in ("crc_gated", "always_on"):
            raise ValueError(f"unknown activation mode {self.activation_mode!r}")

    def resolve_filter_size(self, sphere) -> int:
        if self.filter_size is not None:
            return self.filter_size
        return default_filter_size(_sphere_size(sphere))


@dataclass
class TrajectoryTrace:
    path_index: int
    centers: list
    squared_eds: list
    active_history: list
    iterations_used: int


@dataclass
class DecodeResult:
    best_codeword: BitVector
    best_message: BitVector | None
    squared_ed: float
    stage: str
    traces: list
    counters: object
    near_tie: bool = False


@dataclass
class OpCounter:
    """Field-compatible with the reference's OpCounter (complexity.py:17-44)."""

    ed_evaluations: int = 0
    gain_additions: int = 0
    sort_comparisons: int = 0
    scl_node_ops: int = 0
    osd_reencodes: int = 0
    misc_flops: int = 0

    def __add__(self, other) -> "OpCounter":
        out = OpCounter()
        out.merge(self)
        out.merge(other)
        return out

    def merge(self, other) -> None:
        for f in ("ed_evaluations", "gain_additions", "sort_comparisons", "scl_node_ops",
                  "osd_reencodes", "misc_flops"):
            setattr(self, f, getattr(self, f) + getattr(other, f))


# ---------------------------------------------------------------------------
# Table extraction (duck-typed)

def _sphere_size(sphere) -> int:
    return int(np.asarray(sphere.member_words).shape[0])


def _code_tables(code):
    """(n, k, kp, info_set, gen_words, is_ca, crc_deg, crc_poly, scl_ok)."""
    n, k = int(code.n), int(code.k)
    gen = np.ascontiguousarray(code.generator.words, dtype=np.uint64)
    if code.kind == "crc_concatenated" and getattr(code, "inner", None) is not None \
            and code.inner.kind == "polar":
        info = np.asarray(code.inner.info_set, dtype=np.int32)
        return n, k, int(info.size), info, gen, 1, int(code.crc.degree), crc_poly_int(code.crc), True
    if code.kind == "polar":
        info = np.asarray(code.info_set, dtype=np.int32)
        return n, k, int(info.size), info, gen, 0, 0, 0, True
    # hop-only (e.g. Reed-Muller): SCL is unavailable, as in the reference
    info = np.arange(n - k, n, dtype=np.int32)
    return n, k, k, info, gen, 0, 0, 0, False


def _torch():
    import torch
    return torch


def _dev_tensor(a, dtype, device):
    """Host array or tensor -> contiguous device tensor.  uint32 host words are
    reinterpreted (not converted) as int32."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    if arr.dtype == np.uint32 and dtype == torch.int32:
        arr = arr.view(np.int32)
    if not arr.flags.writeable:
        arr = arr.copy()
    return torch.from_numpy(arr).to(device=device, dtype=dtype).contiguous()


def _is_f64(y) -> bool:
    """float64 received words select the *_f64 entry points."""
    dt = getattr(y, "dtype", None)
    if dt is None:
        return False
    torch = _torch() if "torch" in str(type(y)) else None
    if torch is not None:
        return dt == torch.float64
    return np.dtype(dt) == np.float64


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def words64_to_32(words64: np.ndarray, n: int) -> np.ndarray:
    """uint64 reference layout [..., ceil(n/64)] -> uint32 device layout [..., ceil(n/32)]."""
    w = np.ascontiguousarray(words64, dtype=np.uint64)
    w32 = w.view("<u4").reshape(w.shape[:-1] + (2 * w.shape[-1],))
    nw = (n + 31) // 32
    return np.ascontiguousarray(w32[..., :nw])


def words32_to_64(words32: np.ndarray, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words32).astype(np.uint32, copy=False)
    nw64 = num_words(n)
    pad = 2 * nw64 - w.shape[-1]
    if pad:
        w = np.concatenate([w, np.zeros(w.shape[:-1] + (pad,), np.uint32)], axis=-1)
    return np.ascontiguousarray(w).view("<u8").astype(np.uint64).reshape(w.shape[:-1] + (nw64,))


# ---------------------------------------------------------------------------
# Device decoder: one libmpwsd handle bound to (code, pattern set)

_HOP = {"auto": _native.HOP_AUTO, "gather": _native.HOP_GATHER, "tensor": _native.HOP_TENSOR,
        "tensor2": _native.HOP_TENSOR_2LIMB, "tensor_i8": _native.HOP_TENSOR_I8,
        "tensor_i8a": _native.HOP_TENSOR_I8_ASYNC}


class DeviceDecoder:
    def __init__(self, code, sphere=None, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _native.NativeError("no CUDA device visible: the MP-WSD decoder has no CPU fallback")
        lib = _native.lib()
        idx = torch.cuda.current_device() if device is None else torch.device(device).index or 0
        self.device = torch.device("cuda", idx)
        h = ctypes.c_void_p()
        _native.check(lib.mpw_create(idx, ctypes.byref(h)), "mpw_create")
        self._h = h
        self.code = code
        (self.n, self.k, self.kp, self.info, gen, self.is_ca, self.crc_deg, self.crc_poly,
         self.scl_ok) = _code_tables(code)
        self.nw = (self.n + 31) // 32
        _native.value_error_check(lib.mpw_set_code(
            h, self.n, self.k, self.kp, self.info.ctypes.data, gen.ctypes.data, self.is_ca,
            self.crc_deg, ctypes.c_uint32(self.crc_poly)), "mpw_set_code")
        self._pivots, self._mix = inverse_tables(gen, self.n, self.k)
        self.np = 0
        self.sphere = None
        if sphere is not None:
            self.set_sphere(sphere)

    def set_sphere(self, sphere):
        pats = np.ascontiguousarray(np.asarray(sphere.member_words, dtype=np.uint64)[1:])
        if int(sphere.n) != self.n:
            raise ValueError("sphere blocklength does not match the code")
        _native.value_error_check(_native.lib().mpw_set_patterns(
            self._h, pats.ctypes.data if pats.size else None, int(pats.shape[0])), "mpw_set_patterns")
        self.np = int(pats.shape[0])
        self.sphere = sphere
        self.patterns64 = pats

    def enumerate_lowweight(self, cap: int):
        """Exhaustive GPU walk of all 2^K codewords (mpw_enumerate_lowweight_gpu):
        (weight spectrum A_0..A_n, uint64 words of every codeword with
        1 <= weight <= cap, unordered)."""
        lib = _native.lib()
        spec = np.zeros(self.n + 1, np.int64)
        total = lib.mpw_enumerate_lowweight_gpu(self._h, 0, spec.ctypes.data, None, 0)
        if total < 0:
            _native.value_error_check(int(total), "mpw_enumerate_lowweight_gpu")
        want = int(spec[1:cap + 1].sum()) if cap > 0 else 0
        out = np.zeros((max(want, 1), (self.n + 63) // 64), np.uint64)
        if want:
            got = lib.mpw_enumerate_lowweight_gpu(self._h, int(cap), None, out.ctypes.data, want)
            if got != want:
                raise RuntimeError(f"GPU enumeration count mismatch ({got} != {want})")
        return spec, out[:want]

    @property
    def tensor_path_ready(self) -> bool:
        return bool(_native.lib().mpw_tensor_path_ready(self._h))

    @property
    def auto_variant(self) -> str:
        """The hop variant 'auto' resolves to for this code and pattern set."""
        v = _native.lib().mpw_hop_auto_variant(self._h)
        return {code: name for name, code in _HOP.items()}[v]

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().mpw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self, stream):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    # -- batch entry points -------------------------------------------------
    def two_stage_batch(self, y, sigma: float, list_size: int, num_paths: int, max_iterations: int,
                        activation_mode: str = "crc_gated", variant: str = "auto", tx_words=None,
                        want_hops: bool = False, want_anchors: bool = False, counters=None,
                        stream=None, out=None):
        """y: [F, N] float32 (torch on this device, or host array).  Returns a
        dict of device tensors; uint32 words are carried in int32 tensors."""
        torch = _torch()
        if activation_mode not in ("crc_gated", "always_on"):
            raise ValueError(f"unknown activation mode {activation_mode!r}")
        if activation_mode == "crc_gated" and not self.is_ca:
            raise ValueError("crc_gated mode requires a CRC-concatenated code")
        if not self.scl_ok:
            raise ValueError("SCL stage requires a polar or CRC-polar code")
        f64 = _is_f64(y)
        yd = _dev_tensor(y, torch.float64 if f64 else torch.float32, self.device)
        F = int(yd.shape[0])
        A, T, nw = int(num_paths), int(max_iterations), self.nw
        o = out if out is not None else self.alloc_outputs(F, A, T, want_hops, want_anchors)
        txd = None if tx_words is None else _dev_tensor(tx_words, torch.int32, self.device)
        ctr = counters if counters is not None else o.get("counters")
        fn = _native.lib().mpw_two_stage_batch_f64 if f64 else _native.lib().mpw_two_stage_batch
        rc = fn(
            self._h, _ptr(yd), F, float(sigma), int(list_size), A, T,
            _native.MODE_CRC_GATED if activation_mode == "crc_gated" else _native.MODE_ALWAYS_ON,
            _HOP[variant], _ptr(txd), _ptr(o["best"]), _ptr(o["best_msg"]), _ptr(o["best_ed"]),
            _ptr(o["stage"]), _ptr(o["iters"]), _ptr(o.get("hops")), _ptr(o.get("anchors")),
            _ptr(o["flags"]), _ptr(ctr), self._stream(stream))
        _native.value_error_check(rc, "mpw_two_stage_batch")
        return o

    def two_stage_osd_batch(self, y, order: int, list_cap, num_paths: int, max_iterations: int,
                            activation_mode: str = "always_on", variant: str = "auto", tx_words=None,
                            want_hops: bool = False, want_anchors: bool = False, counters=None,
                            stream=None, out=None):
        """two_stage_batch with OsdStage(order, list_cap) as stage 1
        (mpw_two_stage_osd_batch; decoders.py:555-556)."""
        torch = _torch()
        if activation_mode not in ("crc_gated", "always_on"):
            raise ValueError(f"unknown activation mode {activation_mode!r}")
        if activation_mode == "crc_gated" and not self.is_ca:
            raise ValueError("crc_gated mode requires a CRC-concatenated code")
        if order < 0:
            raise ValueError("order must be >= 0")
        yd = _dev_tensor(y, torch.float32, self.device)
        F = int(yd.shape[0])
        A, T = int(num_paths), int(max_iterations)
        o = out if out is not None else self.alloc_outputs(F, A, T, want_hops, want_anchors)
        txd = None if tx_words is None else _dev_tensor(tx_words, torch.int32, self.device)
        ctr = counters if counters is not None else o.get("counters")
        rc = _native.lib().mpw_two_stage_osd_batch(
            self._h, _ptr(yd), F, int(order), int(list_cap or 0), A, T,
            _native.MODE_CRC_GATED if activation_mode == "crc_gated" else _native.MODE_ALWAYS_ON,
            _HOP[variant], _ptr(txd), _ptr(o["best"]), _ptr(o["best_msg"]), _ptr(o["best_ed"]),
            _ptr(o["stage"]), _ptr(o["iters"]), _ptr(o.get("hops")), _ptr(o.get("anchors")),
            _ptr(o["flags"]), _ptr(ctr), self._stream(stream))
        _native.value_error_check(rc, "mpw_two_stage_osd_batch")
        return o

    def osd_batch(self, y, order: int, list_cap=None, stream=None):
        """Order-k OSD lists (mpw_osd_batch): dict(list_n [F], list_cw [F, M, nw]
        int32 words, list_ed [F, M] float64, flags [F])."""
        torch = _torch()
        if order < 0:
            raise ValueError("order must be >= 0")
        yd = _dev_tensor(y, torch.float32, self.device)
        F = int(yd.shape[0])
        C = osd_candidate_count(order, self.k)
        M = C if list_cap is None else max(0, min(int(list_cap), C))
        d = self.device
        o = dict(list_n=torch.zeros((F,), dtype=torch.int32, device=d),
                 list_cw=torch.zeros((F, max(M, 1), self.nw), dtype=torch.int32, device=d),
                 list_ed=torch.zeros((F, max(M, 1)), dtype=torch.float64, device=d),
                 flags=torch.zeros((F,), dtype=torch.uint8, device=d))
        if M == 0:
            return o
        rc = _native.lib().mpw_osd_batch(self._h, _ptr(yd), F, int(order), int(M), _ptr(o["list_n"]),
                                         _ptr(o["list_cw"]), _ptr(o["list_ed"]), _ptr(o["flags"]),
                                         self._stream(stream))
        _native.value_error_check(rc, "mpw_osd_batch")
        return o

    def alloc_outputs(self, F, A, T, want_hops=False, want_anchors=False):
        torch = _torch()
        d = self.device
        o = dict(best=torch.empty((F, self.nw), dtype=torch.int32, device=d),
                 best_msg=torch.empty((F,), dtype=torch.int64, device=d),
                 best_ed=torch.empty((F,), dtype=torch.float64, device=d),
                 stage=torch.empty((F,), dtype=torch.uint8, device=d),
                 iters=torch.empty((F, A), dtype=torch.int32, device=d),
                 flags=torch.empty((F,), dtype=torch.uint8, device=d),
                 counters=torch.zeros((_native.NUM_COUNTERS,), dtype=torch.int64, device=d))
        if want_hops:
            o["hops"] = torch.empty((F, A, T), dtype=torch.int32, device=d)
        if want_anchors:
            o["anchors"] = torch.zeros((F, A, self.nw), dtype=torch.int32, device=d)
        return o

    def mp_wsd_batch(self, y, anchors_words32, max_iterations: int, n_anchor=None,
                     variant: str = "auto", stream=None):
        """anchors: [F, A, nw] uint32 device layout.  Returns dict of device tensors."""
        torch = _torch()
        f64 = _is_f64(y)
        yd = _dev_tensor(y, torch.float64 if f64 else torch.float32, self.device)
        ad = _dev_tensor(anchors_words32, torch.int32, self.device)
        F, A = int(ad.shape[0]), int(ad.shape[1])
        T = int(max_iterations)
        nad = None if n_anchor is None else _dev_tensor(np.asarray(n_anchor, np.int32), torch.int32, self.device)
        d = self.device
        o = dict(best=torch.empty((F, self.nw), dtype=torch.int32, device=d),
                 best_ed=torch.empty((F,), dtype=torch.float64, device=d),
                 iters=torch.empty((F, A), dtype=torch.int32, device=d),
                 hops=torch.empty((F, A, T), dtype=torch.int32, device=d),
                 flags=torch.empty((F,), dtype=torch.uint8, device=d))
        fn = _native.lib().mpw_mpwsd_batch_f64 if f64 else _native.lib().mpw_mpwsd_batch
        rc = fn(
            self._h, _ptr(yd), _ptr(ad), _ptr(nad), F, A, T, _HOP[variant], _ptr(o["best"]),
            _ptr(o["best_ed"]), _ptr(o["iters"]), _ptr(o["hops"]), _ptr(o["flags"]), self._stream(stream))
        _native.value_error_check(rc, "mpw_mpwsd_batch")
        return o

    def scl_batch(self, llrs=None, y=None, sigma: float = 1.0, list_size: int = 4, stream=None):
        torch = _torch()
        if not self.scl_ok:
            raise ValueError("scl_decode requires a polar code (pass the inner code "
                             "of a CRC-concatenated construction)")
        L = int(list_size)
        if llrs is not None:
            xd = _dev_tensor(llrs, torch.float64, self.device)
            yd = None
        else:
            yd = _dev_tensor(y, torch.float32, self.device)
            xd = None
        F = int((xd if xd is not None else yd).shape[0])
        d = self.device
        o = dict(list_n=torch.zeros((F,), dtype=torch.int32, device=d),
                 list_u=torch.zeros((F, L, self.nw), dtype=torch.int32, device=d),
                 list_cw=torch.zeros((F, L, self.nw), dtype=torch.int32, device=d),
                 list_pm=torch.zeros((F, L), dtype=torch.float64, device=d))
        rc = _native.lib().mpw_scl_batch(self._h, _ptr(yd), _ptr(xd), F, float(sigma), L,
                                         _ptr(o["list_n"]), _ptr(o["list_u"]), _ptr(o["list_cw"]),
                                         _ptr(o["list_pm"]), self._stream(stream))
        _native.value_error_check(rc, "mpw_scl_batch")
        return o

    def message_of_words(self, cw_words64: np.ndarray) -> np.ndarray:
        return message_words(self._pivots, self._mix, unpack_bits(cw_words64, self.n))

    def hop_tile_stats(self, reset: bool = False):
        """(tiles, cycles) of the asynchronous-row hop since the last reset (mpw_hop_tile_stats)."""
        out = np.zeros(2, dtype=np.uint64)
        _native.check(_native.lib().mpw_hop_tile_stats(self._h, out.ctypes.data, int(reset)))
        return int(out[0]), int(out[1])

    def set_option(self, key: str, value: int):
        """mpw_set_option (include/mpwsd.h): stage-1 kernel choice, timing, and
        the tensor hop's A/B launch variants and test hooks."""
        _native.value_error_check(_native.lib().mpw_set_option(self._h, key.encode(), int(value)),
                                  "mpw_set_option")

    @property
    def launch_count(self) -> int:
        """Kernels launched through this handle so far (mpw_launch_count)."""
        return int(_native.lib().mpw_launch_count(self._h))

    # -- timing -------------------------------------------------------------
    def set_timing(self, enable: bool):
        _native.check(_native.lib().mpw_set_timing(self._h, int(bool(enable))))

    def read_timing(self, reset: bool = True):
        ms = np.zeros(4, np.float64)
        n = np.zeros(4, np.int64)
        _native.check(_native.lib().mpw_read_timing(self._h, ms.ctypes.data, n.ctypes.data, int(reset)))
        return ms, n


# ---------------------------------------------------------------------------
# Per-frame drop-in API

class _ThreadCaches(threading.local):
    """Decoders of one host thread: a handle is never shared between threads
    (its scratch and launch order are per handle), keyed weakly on the
    caller's code and sphere objects as the reference keys its caches
    (decoders.py:124, 339-350)."""

    def __init__(self):
        self.by_sphere = weakref.WeakKeyDictionary()    # sphere -> {code -> DeviceDecoder}
        self.code_only = weakref.WeakKeyDictionary()    # code -> DeviceDecoder (stage 1 / OSD lists)
        self.ml_spheres = weakref.WeakKeyDictionary()   # code -> full-codebook sphere (ml_decode)


_tls = _ThreadCaches()


def get_decoder(code, sphere) -> DeviceDecoder:
    """This thread's DeviceDecoder for (code, sphere); sphere None = stage 1 only."""
    if sphere is None:
        dec = _tls.code_only.get(code)
        if dec is None:
            dec = DeviceDecoder(code, None)
            _tls.code_only[code] = dec
        return dec
    per = _tls.by_sphere.get(sphere)
    if per is None:
        per = weakref.WeakKeyDictionary()
        _tls.by_sphere[sphere] = per
    dec = per.get(code)
    if dec is None:
        dec = DeviceDecoder(code, sphere)
        per[code] = dec
    return dec


class _HopCode:
    """Minimal code stand-in for hop-only calls (mp_wsd/wsd_* take no code)."""

    kind = "generic"

    def __init__(self, n):
        self.n, self.k = n, 1

        class _G:
            pass
        self.generator = _G()
        self.generator.words = pack_bits(np.ones((1, n), np.uint8))


_hop_codes: dict = {}


def _hop_decoder(sphere) -> DeviceDecoder:
    n = int(sphere.n)
    code = _hop_codes.setdefault(n, _HopCode(n))
    return get_decoder(code, sphere)


def _modulate(words64, n):
    return 1.0 - 2.0 * unpack_bits(words64, n).astype(np.float64)


def _sqdist(y, words64, n) -> float:
    d = np.asarray(y, dtype=np.float64) - _modulate(words64, n)
    return float(d @ d)


def _step_counters(counters, sphere, m, n):
    """Counter charges of one executed scan (decoders.py:375-389)."""
    nz = _sphere_size(sphere) - 1
    if nz == 0:
        return
    counters.misc_flops += n
    m_eff = min(m, nz)
    if m_eff < nz:
        w = np.bitwise_count(np.asarray(sphere.member_words, dtype=np.uint64)[1:]).sum()
        counters.gain_additions += int(w)
        if m_eff >= 2:
            counters.sort_comparisons += nz * math.ceil(math.log2(m_eff))
    counters.ed_evaluations += m_eff
    counters.misc_flops += m_eff


def _run_hops(dec, y, anchors64, T):
    """Device mp_wsd over one frame's anchors (float64 y); returns host arrays."""
    n = dec.n
    y64 = np.ascontiguousarray(y, dtype=np.float64)[None, :]
    a32 = words64_to_32(np.asarray(anchors64, dtype=np.uint64), n)[None, :, :]
    o = dec.mp_wsd_batch(y64, a32, T)
    return {k: v.cpu().numpy() for k, v in o.items()}


def _traces_from_hops(y, sphere, anchors64, iters, hops, n):
    members = np.asarray(sphere.member_words, dtype=np.uint64)
    traces = []
    for k, anc in enumerate(anchors64):
        words = np.array(anc, dtype=np.uint64)
        centers = [BitVector(n, words)]
        eds = [_sqdist(y, words, n)]
        hist = []
        for h in range(int(iters[k])):
            mem = int(hops[k, h])
            if mem > 0:
                words = words ^ members[mem]
                centers.append(BitVector(n, words))
                eds.append(_sqdist(y, words, n))
                hist.append(True)
            else:
                hist.append(False)
        traces.append(TrajectoryTrace(k, centers, eds, hist, int(iters[k])))
    return traces


def gain_metric(y, x_hat, support) -> float:
    """decoders.py:329-336: sum over the support of -2 y_j x_hat_j (the exact
    correlation change of flipping `support`; -Delta ED / 2)."""
    idx = np.asarray(support, dtype=np.int64)
    if idx.size == 0:
        return 0.0
    y = np.asarray(y, dtype=np.float64)
    return float(-2.0 * np.sum(y[idx] * np.asarray(x_hat, dtype=np.float64)[idx]))


def mp_wsd(y, init_list, sphere, params, counters=None) -> DecodeResult:
    """decoders.py:455-514 on the device."""
    if len(init_list) == 0:
        raise ValueError("initial candidate list is empty")
    if counters is None:
        counters = OpCounter()
    y = np.asarray(y, dtype=np.float64)
    n = int(sphere.n)
    m = params.resolve_filter_size(sphere)
    anchors = init_list.entries[:params.num_paths]
    anc64 = np.stack([np.asarray(cw.words, dtype=np.uint64) for cw, _ in anchors])
    counters.ed_evaluations += len(anchors)
    dec = _hop_decoder(sphere)
    r = _run_hops(dec, y, anc64, params.max_iterations)
    iters, hops = r["iters"][0], r["hops"][0]
    traces = _traces_from_hops(y, sphere, anc64, iters, hops, n)
    for t in traces:
        for _ in range(t.iterations_used):
            _step_counters(counters, sphere, m, n)
    finals = [t.squared_eds[-1] for t in traces]
    best_k = int(np.argmin(finals))
    return DecodeResult(best_codeword=traces[best_k].centers[-1], best_message=None,
                        squared_ed=finals[best_k], stage="mp_wsd", traces=traces,
                        counters=counters, near_tie=bool(r["flags"][0]))


def wsd_trajectory(y, c0, sphere, params, counters=None, force_full_iterations=False,
                   path_index=0) -> TrajectoryTrace:
    """decoders.py:420-452.  force_full_iterations only affects the counters
    (the result is unchanged, decoders.py:427-428)."""
    if counters is None:
        counters = OpCounter()
    y = np.asarray(y, dtype=np.float64)
    n = int(sphere.n)
    m = params.resolve_filter_size(sphere)
    counters.ed_evaluations += 1
    dec = _hop_decoder(sphere)
    anc = np.asarray(c0.words, dtype=np.uint64)[None, :]
    r = _run_hops(dec, y, anc, params.max_iterations)
    tr = _traces_from_hops(y, sphere, anc, r["iters"][0], r["hops"][0], n)[0]
    tr.path_index = path_index
    scans = params.max_iterations if force_full_iterations else tr.iterations_used
    if force_full_iterations:
        tr.active_history = tr.active_history + [False] * (scans - len(tr.active_history))
        tr.iterations_used = scans
    for _ in range(scans):
        _step_counters(counters, sphere, m, n)
    return tr


def wsd_step(y, center, x_center, sphere, m, counters=None):
    """decoders.py:401-417.  The step is scored on t = y * x_center
    (decoders.py:374): every decision of `_wsd_step_core` -- the argmin of the
    survivor EDs and the strict accept test best_ed < ed_center -- depends on
    t alone (ED(x_center * s_p) - ED(x_center) = 4 sum_{supp p} t_i), so the
    device hop runs from the sign pattern of x_center on the received word
    y * |x_center| (so that x' * y' = y * x_center), and the returned words
    are center ^ member as in the reference (decoders.py:396-397)."""
    if m < 1:
        raise ValueError("m must be >= 1")
    if counters is None:
        counters = OpCounter()
    y = np.asarray(y, dtype=np.float64)
    xc = np.asarray(x_center, dtype=np.float64)
    n = int(sphere.n)
    if xc.shape != (n,) or y.shape != (n,):
        raise ValueError(f"expected {n} channel values")
    counters.ed_evaluations += 1
    dec = _hop_decoder(sphere)
    anc = pack_bits((xc < 0).astype(np.uint8)[None, :])
    r = _run_hops(dec, y * np.abs(xc), anc, 1)
    _step_counters(counters, sphere, m, n)
    mem = int(r["hops"][0, 0, 0])
    if mem > 0:
        members = np.asarray(sphere.member_words, dtype=np.uint64)
        return BitVector(center.length, np.asarray(center.words, np.uint64) ^ members[mem]), True
    return BitVector(center.length, np.asarray(center.words, np.uint64)), False


def scl_decode(llrs, code, list_size, counters=None) -> CandidateList:
    """decoders.py:181-268 on the device (float64, bit-exact)."""
    if code.kind != "polar":
        raise ValueError("scl_decode requires a polar code (pass the inner code "
                         "of a CRC-concatenated construction)")
    llrs = np.asarray(llrs, dtype=np.float64)
    n = int(code.n)
    if llrs.shape != (n,):
        raise ValueError("LLR length mismatch")
    if counters is None:
        counters = OpCounter()
    dec = get_decoder(code, None)
    o = dec.scl_batch(llrs=llrs[None, :], list_size=list_size)
    cnt = int(o["list_n"][0].item())
    cw = words32_to_64(o["list_cw"][0, :cnt].cpu().numpy().view(np.uint32), n)
    pm = o["list_pm"][0, :cnt].cpu().numpy()
    counters.scl_node_ops += int(list_size) * n * (n.bit_length() - 1)
    return CandidateList([(BitVector(n, cw[i]), float(pm[i])) for i in range(cnt)])


ML_DIM_LIMIT = 26


def ml_decode(y, code, counters=None):
    """decoders.py:140-167 on the device: the exact argmin of ||y - x(c)||^2
    over all 2^K codewords, as one hop from the zero codeword over P = every
    nonzero codeword (GPU-enumerated, csrc/enum.cuh) -- the reference's
    criterion-3 identity.  Returns (codeword, squared_ed).  Exact ties (measure
    zero) go to the lowest member index rather than the lowest message index."""
    if code.k > ML_DIM_LIMIT:
        raise ValueError(f"K = {code.k} exceeds the ML enumeration budget of {ML_DIM_LIMIT}")
    y = np.asarray(y, dtype=np.float64)
    n = int(code.n)
    if y.shape != (n,):
        raise ValueError(f"expected {n} channel values, got {y.shape}")
    sph = _tls.ml_spheres.get(code)
    if sph is None:
        from .patterns import enumerate_sphere_gpu, weight_spectrum_gpu
        spec = weight_spectrum_gpu(code)
        sph = enumerate_sphere_gpu(code, int((spec[1:] > 0).sum()))
        _tls.ml_spheres[code] = sph
    dec = get_decoder(code, sph)
    o = dec.mp_wsd_batch(y[None, :], np.zeros((1, 1, dec.nw), np.uint32), 1)
    best64 = words32_to_64(o["best"].cpu().numpy().view(np.uint32), n)[0]
    if counters is not None:
        counters.ed_evaluations += 1 << int(code.k)
    return BitVector(n, best64), _sqdist(y, best64, n)


def osd_candidate_count(order: int, k: int) -> int:
    """sum_{w <= order} C(K, w) (decoders.py:301-308; complexity.c_osd)."""
    return sum(math.comb(int(k), w) for w in range(min(int(order), int(k)) + 1))


def osd_decode(y, code, order_k: int, list_cap=None, counters=None) -> CandidateList:
    """decoders.py:274-317 on the device (mpw_osd_batch): the `list_cap`
    best order-k OSD re-encodings by squared ED, ties to the lower candidate."""
    if order_k < 0:
        raise ValueError("order must be >= 0")
    if counters is None:
        counters = OpCounter()
    y = np.asarray(y, dtype=np.float64)
    n = int(code.n)
    if y.shape != (n,):
        raise ValueError(f"expected {n} channel values, got {y.shape}")
    dec = get_decoder(code, None)
    o = dec.osd_batch(y.astype(np.float32)[None, :], order_k, list_cap)
    counters.osd_reencodes += osd_candidate_count(order_k, code.k)
    cnt = int(o["list_n"][0])
    words = words32_to_64(o["list_cw"][0, :cnt].cpu().numpy().view(np.uint32), n)
    eds = o["list_ed"][0, :cnt].cpu().numpy()
    return CandidateList([(BitVector(n, words[i]), float(eds[i])) for i in range(cnt)])


def _two_stage_osd(y, code, stage1, params, sphere, counters) -> DecodeResult:
    """two_stage_decode with OsdStage (decoders.py:555-556, 559-581): the OSD
    list is in the subcode, so gate winners and anchors are used as-is."""
    n = int(code.n)
    dec = get_decoder(code, sphere)
    A, T = params.num_paths, params.max_iterations
    o = dec.two_stage_osd_batch(y.astype(np.float32)[None, :], stage1.order, stage1.list_cap, A, T,
                                params.activation_mode, want_hops=True, want_anchors=True)
    h = {k: v.cpu().numpy() for k, v in o.items()}
    counters.osd_reencodes += osd_candidate_count(stage1.order, code.k)
    best64 = words32_to_64(h["best"][:1].view(np.uint32), n)[0]
    if h["stage"][0] == 0:
        return DecodeResult(best_codeword=BitVector(n, best64),
                            best_message=BitVector(int(code.k), dec.message_of_words(best64)),
                            squared_ed=_sqdist(y, best64, n), stage="stage1_crc_pass",
                            traces=[], counters=counters, near_tie=bool(h["flags"][0]))
    iters = h["iters"][0]
    na = int((iters > 0).sum())
    anc64 = words32_to_64(h["anchors"][0, :na].view(np.uint32), n)
    m = params.resolve_filter_size(sphere)
    counters.ed_evaluations += na
    traces = _traces_from_hops(y, sphere, anc64, iters[:na], h["hops"][0], n)
    for t in traces:
        for _ in range(t.iterations_used):
            _step_counters(counters, sphere, m, n)
    finals = [t.squared_eds[-1] for t in traces]
    best_k = int(np.argmin(finals))
    bc = traces[best_k].centers[-1]
    return DecodeResult(best_codeword=bc,
                        best_message=BitVector(int(code.k), dec.message_of_words(np.asarray(bc.words))),
                        squared_ed=finals[best_k], stage="mp_wsd", traces=traces,
                        counters=counters, near_tie=bool(h["flags"][0]))


def two_stage_decode(y, code, stage1, params, sphere, sigma=1.0, counters=None) -> DecodeResult:
    """decoders.py:520-583 on the device."""
    if counters is None:
        counters = OpCounter()
    y = np.asarray(y, dtype=np.float64)
    gated = params.activation_mode == "crc_gated"
    if gated and code.kind != "crc_concatenated":
        raise ValueError("crc_gated mode requires a CRC-concatenated code")
    if isinstance(stage1, OsdStage) or type(stage1).__name__ == "OsdStage":
        return _two_stage_osd(y, code, stage1, params, sphere, counters)
    if not hasattr(stage1, "list_size"):
        raise ValueError(f"unknown stage-1 spec {stage1!r}")
    if not (code.kind == "polar" or (code.kind == "crc_concatenated"
                                      and getattr(code.inner, "kind", None) == "polar")):
        raise ValueError("SCL stage requires a polar or CRC-polar code")
    n = int(code.n)
    dec = get_decoder(code, sphere)
    A, T = params.num_paths, params.max_iterations
    o = dec.two_stage_batch(y[None, :], sigma, stage1.list_size, A, T,
                            params.activation_mode, want_hops=True, want_anchors=True)
    h = {k: v.cpu().numpy() for k, v in o.items()}
    counters.scl_node_ops += int(stage1.list_size) * n * (n.bit_length() - 1)
    best64 = words32_to_64(h["best"][:1].view(np.uint32), n)[0]
    best = BitVector(n, best64)
    msg = BitVector(int(code.k), dec.message_of_words(best64))
    if h["stage"][0] == 0:
        return DecodeResult(best_codeword=best, best_message=msg,
                            squared_ed=_sqdist(y, best64, n), stage="stage1_crc_pass",
                            traces=[], counters=counters, near_tie=False)
    iters = h["iters"][0]
    na = int((iters > 0).sum())
    anc64 = words32_to_64(h["anchors"][0, :na].view(np.uint32), n)
    m = params.resolve_filter_size(sphere)
    counters.ed_evaluations += na
    traces = _traces_from_hops(y, sphere, anc64, iters[:na], h["hops"][0], n)
    for t in traces:
        for _ in range(t.iterations_used):
            _step_counters(counters, sphere, m, n)
    finals = [t.squared_eds[-1] for t in traces]
    best_k = int(np.argmin(finals))
    bc = traces[best_k].centers[-1]
    return DecodeResult(best_codeword=bc,
                        best_message=BitVector(int(code.k), dec.message_of_words(np.asarray(bc.words))),
                        squared_ed=finals[best_k], stage="mp_wsd", traces=traces,
                        counters=counters, near_tie=bool(h["flags"][0]))


def two_stage_decode_batch(Y, code, stage1, params, sphere, sigma=1.0, tx_words=None,
                           variant="auto"):
    """Batched two_stage_decode over Y [F, N]; returns the device dict of
    DeviceDecoder.two_stage_batch (stage, best, best_msg, best_ed, iters,
    flags, counters)."""
    dec = get_decoder(code, sphere)
    if isinstance(stage1, OsdStage) or type(stage1).__name__ == "OsdStage":
        return dec.two_stage_osd_batch(Y, stage1.order, stage1.list_cap, params.num_paths,
                                       params.max_iterations, params.activation_mode,
                                       variant=variant, tx_words=tx_words)
    return dec.two_stage_batch(Y, sigma, stage1.list_size, params.num_paths,
                               params.max_iterations, params.activation_mode,
                               variant=variant, tx_words=tx_words)


def _as_candidates(entries: list) -> CandidateList:
    lst = CandidateList.__new__(CandidateList)
    lst.entries = entries
    return lst


def device_channel(dec: DeviceDecoder, seed: int, snr_idx: int, first_frame: int, frames: int,
                   sigma: float, stream=None):
    """Device-resident inputs from the counter-based generator (mpw_channel_batch):
    returns (y float32 [F,N], tx int32 words [F,nw], msg int64 [F]) on dec.device."""
    torch = _torch()
    d = dec.device
    y = torch.empty((frames, dec.n), dtype=torch.float32, device=d)
    tx = torch.empty((frames, dec.nw), dtype=torch.int32, device=d)
    msg = torch.empty((frames,), dtype=torch.int64, device=d)
    rc = _native.lib().mpw_channel_batch(dec._h, ctypes.c_uint64(seed), int(snr_idx), int(first_frame),
                                         int(frames), float(sigma), _ptr(y), _ptr(tx), _ptr(msg),
                                         dec._stream(stream))
    _native.value_error_check(rc, "mpw_channel_batch")
    return y, tx, msg
