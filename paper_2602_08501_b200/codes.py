"""Host-side code tables the GPU path consumes.

Code construction is outside the accelerated path, but the
package must run where the reference is absent (the GPU box), so this module
rebuilds the reference's code families with the same conventions:

* CRC: systematic, message first, MSB-first division, parity appended
  (/root/reference/pkg/src/feclab/codebook.py:141-163).
* Polar: info bits on the info set in ascending index order, natural-order
  Kronecker butterfly (codebook.py:166-178, 225-238).
* CRC-concatenated: effective generator row i = inner_encode(crc_append(e_i))
  (codebook.py:261-279).
* Reed-Muller: monomials by degree then lexicographic subset (codebook.py:241-258).

Objects expose the attribute names the reference's `LinearCode` has (`n`, `k`,
`kind`, `info_set`, `crc`, `inner`, `generator.words`), so either a reference
object or one of these can be handed to `paper_2602_08501_b200.decoders`.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from ._nr5g import nr_sequence_1024
from .bits import BitVector, num_words, pack_bits, unpack_bits


# ---------------------------------------------------------------------------
# CRC

@dataclass(eq=False)
class CrcSpec:
    """Degree and generator polynomial; `coefficients` bit i = coeff of x^i."""

    degree: int
    coefficients: BitVector

    def __post_init__(self):
        if self.coefficients.length != self.degree + 1:
            raise ValueError("polynomial length must be degree + 1")
        b = self.coefficients.bits()
        if b[0] != 1 or b[-1] != 1:
            raise ValueError("constant and leading coefficients must be 1")

    @property
    def poly_int(self) -> int:
        return crc_poly_int(self)


def crc_poly_int(crc) -> int:
    """Polynomial as an int, bit i = coefficient of x^i (works for reference
    `CrcSpec` objects too)."""
    bits = np.asarray(crc.coefficients.bits(), dtype=np.int64)
    return int(sum(int(b) << i for i, b in enumerate(bits)))


CRC11 = CrcSpec(11, BitVector.from_support([0, 5, 9, 10, 11], 12))
CRC6 = CrcSpec(6, BitVector.from_support([0, 5, 6], 7))


def crc_remainder(bits, degree: int, poly: int) -> np.ndarray:
    """Remainder of bits(x)·x^0 read MSB-first modulo g(x); `bits` already
    includes any appended zeros.  Returns the last `degree` bits."""
    buf = [int(b) for b in np.asarray(bits, dtype=np.uint8)]
    msb = [(poly >> (degree - j)) & 1 for j in range(degree + 1)]
    for i in range(len(buf) - degree):
        if buf[i]:
            for j in range(degree + 1):
                buf[i + j] ^= msb[j]
    return np.array(buf[len(buf) - degree:], dtype=np.uint8)


def crc_append_bits(msg_bits, crc) -> np.ndarray:
    msg_bits = np.asarray(msg_bits, dtype=np.uint8)
    rem = crc_remainder(np.concatenate([msg_bits, np.zeros(crc.degree, np.uint8)]),
                        crc.degree, crc_poly_int(crc))
    return np.concatenate([msg_bits, rem])


def crc_valid_bits(v_bits, crc) -> bool:
    v_bits = np.asarray(v_bits, dtype=np.uint8)
    if v_bits.size <= crc.degree:
        raise ValueError("vector shorter than CRC parity length")
    return not crc_remainder(v_bits, crc.degree, crc_poly_int(crc)).any()


# ---------------------------------------------------------------------------
# Generator container

class GenMatrix:
    """Minimal stand-in for the reference's BitMatrix: `rows`, `cols`, `words`."""

    def __init__(self, words, cols: int):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if words.ndim != 2 or words.shape[1] != num_words(cols):
            raise ValueError("generator words have the wrong shape")
        words.flags.writeable = False
        self.words = words
        self.rows = words.shape[0]
        self.cols = cols

    def to_bits(self) -> np.ndarray:
        return unpack_bits(self.words, self.cols)


def gf2_row_reduce(bits: np.ndarray):
    """Gauss-Jordan over GF(2) visiting columns left to right.
    Returns (reduced bits, pivot columns)."""
    work = np.array(bits, dtype=np.uint8, copy=True)
    rows = work.shape[0]
    rank = 0
    pivots = []
    for col in range(work.shape[1]):
        if rank == rows:
            break
        hits = np.flatnonzero(work[rank:, col])
        if hits.size == 0:
            continue
        p = rank + int(hits[0])
        if p != rank:
            work[[rank, p]] = work[[p, rank]]
        mask = work[:, col].astype(bool)
        mask[rank] = False
        work[mask] ^= work[rank]
        pivots.append(col)
        rank += 1
    return work, pivots


@dataclass(eq=False)
class LinearCode:
    n: int
    k: int
    generator: GenMatrix
    kind: str = "generic"
    info_set: tuple = ()
    crc: CrcSpec | None = None
    inner: "LinearCode | None" = None
    _pivots: np.ndarray = field(init=False, repr=False)
    _mix: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        if (self.generator.rows, self.generator.cols) != (self.k, self.n):
            raise ValueError("generator shape does not match (K, N)")
        self._pivots, self._mix = inverse_tables(self.generator.words, self.n, self.k)

    @property
    def rate(self) -> float:
        return self.k / self.n

    def message_of(self, codeword) -> BitVector:
        return BitVector(self.k, message_words(self._pivots, self._mix,
                                               unpack_bits(codeword.words, self.n)))

    def label(self) -> str:
        names = {"generic": "linear", "polar": "polar",
                 "reed_muller": "rm", "crc_concatenated": "ca-polar"}
        return f"{names[self.kind]}:{self.n}:{self.k}"


def inverse_tables(gen_words, n: int, k: int):
    """Pivots and mixing rows T with (T·G)[:, pivots] = I, so that the message
    of a codeword c is c[pivots]·T (same idea as codebook.py:104-132)."""
    gbits = unpack_bits(gen_words, n)
    aug = np.concatenate([gbits, np.eye(k, dtype=np.uint8)], axis=1)
    red, piv = gf2_row_reduce(aug)
    piv = [p for p in piv if p < n]
    if len(piv) != k:
        raise ValueError(f"generator rank {len(piv)} < K = {k}")
    return np.asarray(piv, dtype=np.int64), pack_bits(red[:k, n:])


def message_words(pivots, mix_words, cw_bits) -> np.ndarray:
    coeffs = np.asarray(cw_bits)[..., pivots].astype(bool)
    if coeffs.ndim == 1:
        sel = mix_words[coeffs]
        return np.bitwise_xor.reduce(sel, axis=0) if sel.shape[0] else np.zeros(
            mix_words.shape[1], dtype=np.uint64)
    out = np.zeros(coeffs.shape[:-1] + (mix_words.shape[1],), dtype=np.uint64)
    for j in range(coeffs.shape[-1]):
        out[coeffs[..., j]] ^= mix_words[j]
    return out


# ---------------------------------------------------------------------------
# Polar / RM / CA constructions

def polar_transform_bits(bits) -> np.ndarray:
    out = np.array(bits, dtype=np.uint8, copy=True)
    n = out.shape[-1]
    if n & (n - 1):
        raise ValueError("length must be a power of two")
    h = 1
    while h < n:
        v = out.reshape(-1, n // (2 * h), 2 * h)
        v[:, :, :h] ^= v[:, :, h:]
        h *= 2
    return out


def reliability_order(n: int) -> np.ndarray:
    """Indices 0..n-1, least reliable first (5G NR table filtered to < n)."""
    if n < 2 or n & (n - 1) or n > 1024:
        raise ValueError("n must be a power of two in [2, 1024]")
    seq = nr_sequence_1024()
    return seq[seq < n]


def polar_code_from_info_set(n: int, info_set) -> LinearCode:
    info = np.sort(np.asarray(info_set, dtype=np.int64))
    eye = np.zeros((info.size, n), dtype=np.uint8)
    eye[np.arange(info.size), info] = 1
    rows = polar_transform_bits(eye)
    return LinearCode(n, int(info.size), GenMatrix(pack_bits(rows), n), kind="polar",
                      info_set=tuple(int(i) for i in info))


def build_polar_code(n: int, k_eff: int, ranked=None) -> LinearCode:
    ranked = reliability_order(n) if ranked is None else np.asarray(ranked)
    return polar_code_from_info_set(n, ranked[n - k_eff:])


def build_ca_code(k: int, crc, inner: LinearCode) -> LinearCode:
    if inner.k != k + crc.degree:
        raise ValueError("inner dimension must be K + CRC degree")
    rows = []
    gin = inner.generator.words
    for i in range(k):
        e = np.zeros(k, dtype=np.uint8)
        e[i] = 1
        v = crc_append_bits(e, crc)
        sel = gin[np.flatnonzero(v)]
        rows.append(np.bitwise_xor.reduce(sel, axis=0))
    return LinearCode(inner.n, k, GenMatrix(np.stack(rows), inner.n),
                      kind="crc_concatenated", crc=crc, inner=inner)


def build_ca_polar_code(n: int, k: int, crc=CRC11) -> LinearCode:
    return build_ca_code(k, crc, build_polar_code(n, k + crc.degree))


def build_rm_code(m: int, r: int) -> LinearCode:
    n = 1 << m
    pts = np.arange(n)
    var = [((pts >> i) & 1).astype(np.uint8) for i in range(m)]
    rows = []
    for deg in range(r + 1):
        for sub in itertools.combinations(range(m), deg):
            row = np.ones(n, dtype=np.uint8)
            for i in sub:
                row &= var[i]
            rows.append(row)
    return LinearCode(n, len(rows), GenMatrix(pack_bits(np.stack(rows)), n),
                      kind="reed_muller")


def rm_as_polar(m: int, r: int) -> LinearCode:
    """RM(r, m) as a polar code: info set = {i : popcount(i) >= m - r}
    (BASELINE config 2: RM(2,7) decoded by SCL with the RM frozen set)."""
    n = 1 << m
    info = [i for i in range(n) if bin(i).count("1") >= m - r]
    return polar_code_from_info_set(n, info)


# ---------------------------------------------------------------------------
# Encoding helpers

def encode(code, msg) -> BitVector:
    bits = msg.bits() if hasattr(msg, "bits") else np.asarray(msg, dtype=np.uint8)
    gw = code.generator.words
    sel = gw[np.flatnonzero(bits)]
    if sel.shape[0] == 0:
        return BitVector.zeros(code.n)
    return BitVector(code.n, np.bitwise_xor.reduce(sel, axis=0))


def encode_batch(code, msg_bits: np.ndarray) -> np.ndarray:
    """msg_bits uint8 [F, K] -> codeword words uint64 [F, W64]."""
    gw = np.asarray(code.generator.words, dtype=np.uint64)
    out = np.zeros((msg_bits.shape[0], gw.shape[1]), dtype=np.uint64)
    for i in range(gw.shape[0]):
        out[msg_bits[:, i].astype(bool)] ^= gw[i]
    return out


def inner_polar(code):
    """The polar code SCL runs on (decoders.py:543-549)."""
    if code.kind == "crc_concatenated" and code.inner is not None and code.inner.kind == "polar":
        return code.inner
    if code.kind == "polar":
        return code
    raise ValueError("SCL stage requires a polar or CRC-polar code")


def precoded_of_codeword(code, codeword) -> BitVector:
    inner = inner_polar(code)
    u = polar_transform_bits(unpack_bits(codeword.words, code.n))
    return BitVector.from_bits(u[np.asarray(inner.info_set, dtype=np.int64)])
