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
