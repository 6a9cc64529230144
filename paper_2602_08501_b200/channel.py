"""Seeded host-side input generation (BPSK over AWGN), fed identically to the
GPU path and to the CPU oracle.

Two keyings:

* `trial_inputs`: the reference harness's per-trial streams -- message bits
  from Philox key (seed, sid|1), noise from (seed, sid) with
  sid = (snr_idx << 40) | (trial << 2)
  (/root/reference/pkg/src/feclab/simharness.py:220-222, 295-301;
  channel.py:65-80).  Used for golden/parity runs.
* `bulk_inputs`: block-keyed Philox, key (seed, (snr_idx << 40) | block),
  4096 frames per block, for 10^6-10^7-frame runs.  A documented deviation
  from the per-trial keying; shards align to blocks.

Received words are returned as float32 (the dtype of the path); the oracle
consumes float64(y32), so both sides see identical values.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .codes import encode_batch

BLOCK = 4096
_MASK64 = (1 << 64) - 1


def ebno_to_sigma(ebno_db: float, rate: float) -> float:
    """channel.py:53-57"""
    if not 0 < rate <= 1:
        raise ValueError("rate must lie in (0, 1]")
    return math.sqrt(1.0 / (2.0 * rate * 10.0 ** (ebno_db / 10.0)))


def modulate(c) -> np.ndarray:
    """BPSK: bit 0 -> +1, bit 1 -> -1 (channel.py:44-46)."""
    return 1.0 - 2.0 * np.asarray(c.bits(), dtype=np.float64)


def modulate_bits(bits) -> np.ndarray:
    """channel.py:49-50."""
    return 1.0 - 2.0 * np.asarray(bits, dtype=np.float64)


def llr(y, sigma: float) -> np.ndarray:
    """2y/sigma^2 (channel.py:83-87)."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    return 2.0 * np.asarray(y, dtype=np.float64) / (sigma * sigma)


def squared_distance(y, x) -> float:
    """||y - x||^2 (channel.py:90-93)."""
    d = np.asarray(y, dtype=np.float64) - np.asarray(x, dtype=np.float64)
    return float(d @ d)


def _stream(seed: int, sid: int) -> np.random.Generator:
    key = np.array([seed & _MASK64, sid & _MASK64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def modulate_words(words: np.ndarray, n: int) -> np.ndarray:
    from .bits import unpack_bits
    return 1.0 - 2.0 * unpack_bits(words, n).astype(np.float64)


def trial_inputs(code, seed: int, snr_idx: int, trials, sigma: float):
    """Per-trial reference keying.  Returns (msg_bits uint8 [F,K],
    codeword words uint64 [F,W64], y float64 [F,N] exactly as the reference
    computes it)."""
    trials = list(trials)
    k, n = code.k, code.n
    msgs = np.zeros((len(trials), k), dtype=np.uint8)
    noise = np.zeros((len(trials), n), dtype=np.float64)
    for r, t in enumerate(trials):
        base = (snr_idx << 40) | (t << 2)
        msgs[r] = _stream(seed, base | 1).integers(0, 2, k, dtype=np.uint8)
        noise[r] = _stream(seed, base).standard_normal(n)
    cw = encode_batch(code, msgs)
    y = modulate_words(cw, n) + sigma * noise
    return msgs, cw, y


def _bulk_block(code, seed, snr_idx, block, count, sigma):
    g = _stream(seed, (snr_idx << 40) | block)
    msgs = g.integers(0, 2, (count, code.k), dtype=np.uint8)
    z = g.standard_normal((count, code.n), dtype=np.float32)
    cw = encode_batch(code, msgs)
    y = (modulate_words(cw, code.n).astype(np.float32) + np.float32(sigma) * z)
    return msgs, cw, y.astype(np.float32)


def bulk_inputs(code, seed: int, snr_idx: int, first_frame: int, frames: int, sigma: float,
                threads: int = 0):
    """Block-keyed bulk generation of frames [first_frame, first_frame+frames);
    first_frame must be a multiple of BLOCK.  Returns (msg_bits, cw_words, y32)."""
    if first_frame % BLOCK:
        raise ValueError("bulk shards must start on a block boundary")
    nblk = (frames + BLOCK - 1) // BLOCK
    b0 = first_frame // BLOCK
    counts = [min(BLOCK, frames - i * BLOCK) for i in range(nblk)]
    threads = threads or min(32, max(1, (__import__("os").cpu_count() or 1)))
    with ThreadPoolExecutor(max_workers=threads) as pool:
        parts = list(pool.map(lambda i: _bulk_block(code, seed, snr_idx, b0 + i, counts[i], sigma),
                              range(nblk)))
    msgs = np.concatenate([p[0] for p in parts])
    cw = np.concatenate([p[1] for p in parts])
    y = np.concatenate([p[2] for p in parts])
    return msgs, cw, y


# ---------------------------------------------------------------------------
# Counter-based keyed stream shared with the device generator (csrc/channel.cuh)

_PH_M0, _PH_M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_PH_W0, _PH_W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_PH_TAG = np.uint32(0x4D505753)
_U32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 (Random123 constants); uint32 arrays in/out."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = _PH_M0 * c0.astype(np.uint64)
            p1 = _PH_M1 * c2.astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & _U32).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & _U32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint32(k0 + _PH_W0)
            k1 = np.uint32(k1 + _PH_W1)
    return c0, c1, c2, c3


def keyed_inputs_host(code, seed: int, snr_idx: int, first_frame: int, frames: int, sigma: float):
    """numpy mirror of mpw_channel_batch: (msg_words uint64 [F], codeword words
    uint64 [F, W64], y float32 [F, N]).  The device computes log / sincospi
    in float64 with its own libm, so a y value can differ by 1 float32 ulp in
    rare cases (rounding ties after ~1e-16 relative differences)."""
    n, k = code.n, code.k
    g = np.arange(first_frame, first_frame + frames, dtype=np.uint64)
    glo = (g & _U32).astype(np.uint32)
    ghi = (g >> np.uint64(32)).astype(np.uint32)
    k0 = np.uint32(seed & 0xFFFFFFFF)
    with np.errstate(over="ignore"):
        k1 = np.uint32((seed >> 32) & 0xFFFFFFFF) ^ np.uint32((snr_idx * 0x9E3779B9) & 0xFFFFFFFF)
    z = np.zeros_like(glo)
    m0, m1, m2, m3 = philox4x32_10(glo, ghi, z, np.full_like(glo, _PH_TAG), k0, k1)
    words = np.stack([m0, m1, m2, m3], axis=1).view("<u4")
    msg_bits = np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, :k]
    msg = (msg_bits.astype(np.uint64) << np.arange(k, dtype=np.uint64)).sum(axis=1, dtype=np.uint64) \
        if k <= 64 else None
    cw = encode_batch(code, msg_bits)
    x = modulate_words(cw, n)
    nz = np.zeros((frames, n), dtype=np.float64)
    for c in range((n + 3) // 4):
        r0, r1, r2, r3 = philox4x32_10(glo, ghi, np.full_like(glo, 1 + c), np.full_like(glo, _PH_TAG), k0, k1)
        for h, (a, b) in enumerate(((r0, r1), (r2, r3))):
            u1 = (a.astype(np.float64) + 0.5) * 2.3283064365386963e-10
            u2 = (b.astype(np.float64) + 0.5) * 2.3283064365386963e-10
            rad = np.sqrt(-2.0 * np.log(u1))
            ang = 2.0 * np.pi * u2
            for q, val in ((4 * c + 2 * h, rad * np.cos(ang)), (4 * c + 2 * h + 1, rad * np.sin(ang))):
                if q < n:
                    nz[:, q] = val
    y = (x + sigma * nz).astype(np.float32)
    return msg, cw, y
