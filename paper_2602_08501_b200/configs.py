"""The BASELINE.json configurations, instantiated.

cfg1  polar(64,16) 5G frozen set, 10 msg bits + CRC-6 (x^6+x^5+1), SCL L=4,
      A=4, T=4, gated, 2 dB; P = subcode codewords of weight <= d_min+2
      (r=1: 96 patterns of weight 24).
cfg2  RM(2,7) (128,29) decoded as polar with the RM frozen set, L=8, A=8,
      T=6, always-on (no CRC), 3 dB; P = the 10,668 weight-32 codewords.
cfg3  polar(128,32) 5G, 21 msg bits + CRC-11 (0xE21), L=8, A=8, T=8, gated,
      1-4 dB; P = subcode weight <= d_min+4 (r=1: 15 patterns of weight 32).
cfg4  polar(256,64) 5G + CRC-11, K=53, L=16, A=16, T=8, stage 2 forced,
      1.5 dB; P = all subcode codewords of weight <= 56 found by the seeded
      information-set collector (62,434 patterns; the reference's 2^K
      enumeration refuses K=53, wsphere.py:28).  The collector saturates:
      p=2 over 10^6 and p=3 over 5x10^4 random information sets return the
      identical set.  Completeness is not proven.
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field

import numpy as np

from . import codes
from .channel import ebno_to_sigma


@dataclass
class DecodeConfig:
    name: str
    code_builder: object
    list_size: int
    num_paths: int
    max_iterations: int
    activation_mode: str
    ebno_db: list
    frames: int
    radius_index: int = 1
    collector: dict = field(default_factory=dict)   # non-empty -> use the ISD collector

    def code(self):
        return self.code_builder()

    def sigma(self, ebno_db=None, code=None):
        code = code or self.code()
        e = self.ebno_db[0] if ebno_db is None else ebno_db
        return ebno_to_sigma(e, code.k / code.n)


def _cfg1_code():
    return codes.build_ca_polar_code(64, 10, codes.CRC6)


def _cfg2_code():
    return codes.rm_as_polar(7, 2)


def _cfg3_code():
    return codes.build_ca_polar_code(128, 21, codes.CRC11)


def _cfg4_code():
    return codes.build_ca_polar_code(256, 53, codes.CRC11)


CONFIGS = {
    "cfg1": DecodeConfig("cfg1", _cfg1_code, 4, 4, 4, "crc_gated", [2.0], 100_000),
    "cfg2": DecodeConfig("cfg2", _cfg2_code, 8, 8, 6, "always_on", [3.0], 1_000_000),
    "cfg3": DecodeConfig("cfg3", _cfg3_code, 8, 8, 8, "crc_gated",
                         [1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0], 1_000_000),
    "cfg4": DecodeConfig("cfg4", _cfg4_code, 16, 16, 8, "always_on", [1.5], 8_000_000,
                         collector=dict(weight_cap=56, iterations=50_000, seed=20260208, p_max=3)),
}

# sha256 over the CWS1 member words of each config's P (sphere_digest), pinned
# when the sets were first generated; tests/test_patterns.py regenerates them
SPHERE_SHA256 = {
    "cfg1": "66dc251037446d9242f3c308d6e727fc63c4ae7970f536438d1cb373e095dbb4",
    "cfg2": "2188cdd720549f09b7100c97d3356eb9ed952487f7fdcb2c8c4ddda114d280fd",
    "cfg3": "758c3ac1cd842bb8d03140b36b1a0af742229a86614d0cc3d53e2256eba1b18f",
    "cfg4": "3c467a3ce8f8ed44b0cbf286153f3e5299dd242db1af38bba449acc7e4eef855",
}

_CACHE_DIR = os.environ.get("MPWSD_CACHE", os.path.join(os.path.dirname(os.path.abspath(__file__)), "_spheres"))


def sphere_digest(sphere) -> str:
    return hashlib.sha256(np.ascontiguousarray(sphere.member_words, dtype="<u8").tobytes()).hexdigest()


def build_sphere_for(cfg: DecodeConfig, code=None, use_cache: bool = True):
    """P for a config: exhaustive enumeration (K <= 30) or the seeded collector.
    Cached as CWS1 under paper_2602_08501_b200/_spheres/ (untracked)."""
    from .patterns import collect_sphere, enumerate_sphere
    from .sphere import load_sphere, save_sphere
    code = code or cfg.code()
    path = os.path.join(_CACHE_DIR, f"{cfg.name}.cws")
    if use_cache and os.path.exists(path):
        s = load_sphere(path)
        if (s.n, s.k) == (code.n, code.k):
            return s
    if cfg.collector:
        c = cfg.collector
        s = collect_sphere(code, c["weight_cap"], c["iterations"], c["seed"], c["p_max"])
    else:
        s = enumerate_sphere(code, cfg.radius_index)
    if use_cache:
        os.makedirs(_CACHE_DIR, exist_ok=True)
        save_sphere(s, path + ".tmp")
        os.replace(path + ".tmp", path)
    return s
