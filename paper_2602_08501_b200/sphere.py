"""Pattern set P: the nonzero members of a code-weight sphere.

The on-disk format is the reference's CWS1 (
/root/reference/pkg/src/feclab/wsphere.py:237-286): magic 'CWS1', LE u32
(N, K, r, shell_count), LE u32 (weight, count) per shell, members as LE
uint64 words shell-major with the zero codeword first, 8-byte BLAKE2b trailer.

Member order is shell-major, then lexicographic with word 0 the most
significant key (wsphere.py:197-202).  Pattern index = member index - 1; the
hop kernels break exact ties towards the lowest pattern index, which is the
reference's `argmin` order (decoders.py:391-392).
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass

import numpy as np

from .bits import num_words, popcount_rows, unpack_bits

MAGIC = b"CWS1"
CHECKSUM_BYTES = 8


class SphereFormatError(ValueError):
    pass


@dataclass(eq=False)
class PatternSphere:
    """Field names follow the reference's `CodeWeightSphere` (wsphere.py:73-112)."""

    n: int
    k: int
    radius_index: int
    shell_weights: np.ndarray
    shell_counts: np.ndarray
    member_words: np.ndarray      # [size, W64] uint64, zero codeword first

    def __post_init__(self):
        w = np.ascontiguousarray(self.member_words, dtype=np.uint64)
        if w.ndim != 2 or w.shape[1] != num_words(self.n):
            raise ValueError("member words have the wrong shape")
        if w.shape[0] == 0 or w[0].any():
            raise ValueError("sphere must start with the zero codeword")
        w.flags.writeable = False
        self.member_words = w
        self.member_weights = popcount_rows(w)

    @property
    def size(self) -> int:
        return self.member_words.shape[0]

    @property
    def nonzero_size(self) -> int:
        return self.size - 1

    @property
    def mean_nonzero_weight(self) -> float:
        return float(self.member_weights[1:].mean()) if self.size > 1 else 0.0

    def patterns(self) -> np.ndarray:
        """Nonzero members [|P|, W64] (pattern index = member index - 1)."""
        return self.member_words[1:]

    def member_support(self, i: int) -> np.ndarray:
        if i < 1:
            raise IndexError("member 0 is the zero codeword")
        return np.flatnonzero(unpack_bits(self.member_words[i], self.n))

    def shell_table(self) -> list:
        return list(zip(np.asarray(self.shell_weights).tolist(),
                        np.asarray(self.shell_counts).tolist()))


def sort_members(words: np.ndarray) -> np.ndarray:
    """Shell-major order: weight ascending, then words with word 0 most
    significant (wsphere.py:197-202)."""
    words = np.asarray(words, dtype=np.uint64)
    weights = popcount_rows(words)
    keys = tuple(words[:, j] for j in reversed(range(words.shape[1]))) + (weights,)
    return np.ascontiguousarray(words[np.lexsort(keys)])


def sphere_from_members(n: int, k: int, radius_index: int, words: np.ndarray) -> PatternSphere:
    """Build a sphere from an unordered set of nonzero low-weight codewords
    (e.g. the output of a collector); adds the zero codeword and sorts."""
    words = np.asarray(words, dtype=np.uint64).reshape(-1, num_words(n))
    words = words[popcount_rows(words) > 0]
    words = np.unique(words, axis=0)
    allw = sort_members(np.concatenate([np.zeros((1, words.shape[1]), np.uint64), words]))
    wts = popcount_rows(allw)
    sw, sc = np.unique(wts, return_counts=True)
    return PatternSphere(n, k, radius_index, sw.astype(np.int64), sc.astype(np.int64), allw)


def as_sphere(obj) -> PatternSphere:
    """Accept a reference `CodeWeightSphere` or a PatternSphere."""
    if isinstance(obj, PatternSphere):
        return obj
    return PatternSphere(int(obj.n), int(obj.k), int(obj.radius_index),
                         np.asarray(obj.shell_weights), np.asarray(obj.shell_counts),
                         np.asarray(obj.member_words, dtype=np.uint64))


def save_sphere(sphere, path) -> None:
    s = as_sphere(sphere)
    parts = [MAGIC, struct.pack("<IIII", s.n, s.k, s.radius_index, len(s.shell_weights))]
    for w, c in zip(s.shell_weights, s.shell_counts):
        parts.append(struct.pack("<II", int(w), int(c)))
    parts.append(s.member_words.astype("<u8").tobytes())
    blob = b"".join(parts)
    with open(path, "wb") as fh:
        fh.write(blob + hashlib.blake2b(blob, digest_size=CHECKSUM_BYTES).digest())


def load_sphere(path) -> PatternSphere:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 4 + 16 + CHECKSUM_BYTES:
        raise SphereFormatError("file truncated: too short for header")
    if raw[:4] != MAGIC:
        raise SphereFormatError(f"bad magic {raw[:4]!r}")
    body, digest = raw[:-CHECKSUM_BYTES], raw[-CHECKSUM_BYTES:]
    if hashlib.blake2b(body, digest_size=CHECKSUM_BYTES).digest() != digest:
        raise SphereFormatError("checksum mismatch: file corrupted")
    n, k, r, shells = struct.unpack("<IIII", body[4:20])
    pos = 20
    if len(body) < pos + 8 * shells:
        raise SphereFormatError("file truncated inside shell table")
    table = np.frombuffer(body[pos:pos + 8 * shells], dtype="<u4").reshape(shells, 2)
    pos += 8 * shells
    sw = table[:, 0].astype(np.int64)
    sc = table[:, 1].astype(np.int64)
    width = num_words(n)
    total = int(sc.sum())
    if len(body) - pos != total * width * 8:
        raise SphereFormatError("payload size does not match the shell table")
    words = np.frombuffer(body[pos:], dtype="<u8").astype(np.uint64).reshape(total, width)
    if not np.array_equal(popcount_rows(words), np.repeat(sw, sc)):
        raise SphereFormatError("member weights disagree with shell table")
    return PatternSphere(int(n), int(k), int(r), sw, sc, words)
