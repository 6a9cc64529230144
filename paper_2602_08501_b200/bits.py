"""Packed GF(2) words shared by the host side, the C-ABI and the kernels.

Layout (identical to the reference's, /root/reference/pkg/src/feclab/binlin.py:1-8):
bit j of a length-n vector is bit (j mod 64) of uint64 word j // 64.  Because
the words are little-endian, the same bytes read as uint32 give bit j in bit
(j mod 32) of uint32 word j // 32 -- the device-side view.
"""

from __future__ import annotations

import numpy as np

WORD_BITS = 64


def num_words(length: int) -> int:
    return (length + WORD_BITS - 1) // WORD_BITS


def pack_bits(bits) -> np.ndarray:
    """0/1 array (last axis = bit index) -> uint64 words (last axis = word)."""
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    n = bits.shape[-1]
    pad = (-n) % WORD_BITS
    if pad:
        bits = np.concatenate(
            [bits, np.zeros(bits.shape[:-1] + (pad,), dtype=np.uint8)], axis=-1)
    packed = np.packbits(bits, axis=-1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u8").astype(np.uint64, copy=False)


def unpack_bits(words, length: int) -> np.ndarray:
    words = np.ascontiguousarray(words, dtype=np.uint64).astype("<u8", copy=False)
    if words.size == 0:
        return np.zeros(words.shape[:-1] + (length,), dtype=np.uint8)
    raw = words.view(np.uint8).reshape(words.shape[:-1] + (-1,))
    return np.unpackbits(raw, axis=-1, bitorder="little")[..., :length]


def popcount_rows(words) -> np.ndarray:
    return np.bitwise_count(np.asarray(words, dtype=np.uint64)).sum(axis=-1, dtype=np.int64)


class BitVector:
    """Immutable packed bit vector; API-compatible with the reference's
    `BitVector` (binlin.py:62-129) for the members the decoder API returns.
    Equality accepts any object exposing `length` and `words`."""

    __slots__ = ("length", "words")

    def __init__(self, length: int, words):
        words = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)
        if words.shape != (num_words(length),):
            raise ValueError("word count does not match length")
        tail = length % WORD_BITS
        if tail and int(words[-1]) >> tail:
            raise ValueError("bits set beyond declared length")
        words.flags.writeable = False
        self.length = int(length)
        self.words = words

    @classmethod
    def from_bits(cls, bits) -> "BitVector":
        bits = np.asarray(bits, dtype=np.uint8)
        return cls(bits.shape[0], pack_bits(bits))

    @classmethod
    def zeros(cls, length: int) -> "BitVector":
        return cls(length, np.zeros(num_words(length), dtype=np.uint64))

    @classmethod
    def from_support(cls, indices, length: int) -> "BitVector":
        bits = np.zeros(length, dtype=np.uint8)
        bits[np.asarray(indices, dtype=np.int64)] = 1
        return cls.from_bits(bits)

    def bits(self) -> np.ndarray:
        return unpack_bits(self.words, self.length)

    def support(self) -> np.ndarray:
        return np.flatnonzero(self.bits())

    def weight(self) -> int:
        return int(np.bitwise_count(self.words).sum())

    def __xor__(self, other) -> "BitVector":
        if self.length != other.length:
            raise ValueError("length mismatch")
        return BitVector(self.length, self.words ^ np.asarray(other.words, dtype=np.uint64))

    def __eq__(self, other) -> bool:
        if not (hasattr(other, "length") and hasattr(other, "words")):
            return NotImplemented
        return self.length == other.length and bool(
            np.array_equal(self.words, np.asarray(other.words, dtype=np.uint64)))

    def __hash__(self) -> int:
        return hash((self.length, self.words.tobytes()))

    def __repr__(self) -> str:
        shown = "".join(str(b) for b in self.bits()[:32])
        return f"BitVector({self.length}, {shown}{'...' if self.length > 32 else ''})"
