"""Pattern-set generators and the CWS1 format (SURVEY.md §8f row 1, §8(a) rows
12-14), pinned to the reference's published numbers:

* criterion 1: |S_3(0)| = 538 and |S_4(0)| = 6472 for CA-polar(256,16)+CRC-11
  (reference tests/test_acceptance.py:51-71);
* RM(2,7): 10,668 minimum-weight codewords (closed form 4*127*63/3,
  tests/test_acceptance.py:84-88);
* the seeded collector used for K > 30 (cfg4's P) equals exhaustive
  enumeration (the reference's `build_sphere`, wsphere.py:175-208) wherever
  the latter is possible, and the closed-form minimum-weight count of polar
  codes where it is not;
* cfg4's P is the same set for different seeds and search depths, and every
  config's P matches its pinned digest (configs.SPHERE_SHA256);
* CWS1 files written by the reference's `save_sphere` are read identically and
  re-written byte for byte; corruption is rejected as in
  tests/test_wsphere.py:137-174.
"""

import numpy as np
import pytest

from paper_2602_08501_b200 import codes, configs, patterns
from paper_2602_08501_b200.sphere import (SphereFormatError, load_sphere, save_sphere,
                                          sphere_from_members)

import os

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _words(s):
    return np.asarray(s.member_words, dtype=np.uint64)


def _collect_radius(code, r, **kw):
    """Collector run with the weight cap of enumeration shell r."""
    spec = patterns.weight_spectrum(code)
    shells = [w for w in range(1, code.n + 1) if spec[w]]
    return patterns.collect_sphere(code, shells[r - 1], **kw)


def test_criterion_1_sphere_sizes_256_16():
    code = codes.build_ca_polar_code(256, 16)
    s3 = patterns.enumerate_sphere(code, 3)
    s4 = patterns.enumerate_sphere(code, 4)
    assert (s3.size, s4.size) == (538, 6472)
    assert int(patterns.weight_spectrum(code).sum()) == 1 << 16


@pytest.mark.parametrize("r", [3, 4])
def test_collector_equals_enumeration_256_16(r):
    code = codes.build_ca_polar_code(256, 16)
    a = _collect_radius(code, r, iterations=20_000, seed=1, p_max=3)
    b = patterns.enumerate_sphere(code, r)
    assert a.size == {3: 538, 4: 6472}[r]
    assert np.array_equal(_words(a), _words(b))


def test_collector_rm_2_7_minimum_weight():
    code = configs.CONFIGS["cfg2"].code()
    a = patterns.collect_sphere(code, 32, iterations=20_000, seed=3, p_max=2)
    assert a.nonzero_size == 10668 == 4 * 127 * 63 // 3
    assert np.array_equal(_words(a), _words(patterns.enumerate_sphere(code, 1)))


@pytest.mark.parametrize("name,r", [("cfg1", 1), ("cfg1", 2), ("cfg3", 1), ("cfg3", 2)])
def test_collector_equals_enumeration_small_configs(name, r):
    code = configs.CONFIGS[name].code()
    a = _collect_radius(code, r, iterations=20_000, seed=5, p_max=3)
    assert np.array_equal(_words(a), _words(patterns.enumerate_sphere(code, r)))


def polar_min_weight_count(info_set, n):
    """Closed-form number of minimum-weight codewords of a polar code with
    information set I: d_min = 2^w with w = min popcount(i),
    A_dmin = sum over i in I with popcount(i) = w of 2^(r_i + lambda_i), r_i the
    number of 0 bits of i (out of m = log2 n) and lambda_i = sum over 0-bit
    positions z of #{k < z : bit k of i is 1}."""
    m = n.bit_length() - 1
    w = min(bin(int(i)).count("1") for i in info_set)
    total = 0
    for i in (int(v) for v in info_set):
        if bin(i).count("1") != w:
            continue
        zeros = [z for z in range(m) if not (i >> z) & 1]
        lam = sum(bin(i & ((1 << z) - 1)).count("1") for z in zeros)
        total += 1 << (len(zeros) + lam)
    return 1 << w, total


@pytest.mark.parametrize("n,k", [(16, 8), (32, 12), (64, 16), (64, 24), (128, 29)])
def test_closed_form_min_weight_matches_enumeration(n, k):
    code = codes.build_polar_code(n, k)
    d, cnt = polar_min_weight_count(code.info_set, n)
    spec = patterns.weight_spectrum(code)
    assert int(np.flatnonzero(spec[1:])[0]) + 1 == d
    assert int(spec[d]) == cnt


def test_collector_matches_closed_form_inner_256_64():
    """cfg4's inner (256,64) polar code (K = 64, beyond exhaustive enumeration):
    the collector finds exactly the closed-form number of weight-d_min words."""
    inner = configs.CONFIGS["cfg4"].code().inner
    d, cnt = polar_min_weight_count(inner.info_set, 256)
    assert (d, cnt) == (16, 48)
    s = patterns.collect_sphere(inner, d, iterations=20_000, seed=9, p_max=2)
    assert s.nonzero_size == cnt
    assert set(np.unique(s.member_weights[1:])) == {d}


def test_cfg4_pattern_set_is_seed_and_depth_independent():
    """The collector saturates on cfg4's subcode: different seeds and search
    depths return the identical 62,434-word P."""
    code = configs.CONFIGS["cfg4"].code()
    digests = set()
    for it, seed, p in ((50_000, 20260208, 3), (50_000, 7, 3), (200_000, 11, 2)):
        s = patterns.collect_sphere(code, 56, iterations=it, seed=seed, p_max=p)
        assert s.nonzero_size == 62434
        assert list(s.shell_weights) == [0, 32, 40, 48, 56]
        assert list(s.shell_counts) == [1, 10, 63, 3639, 58722]
        digests.add(configs.sphere_digest(s))
    assert digests == {configs.SPHERE_SHA256["cfg4"]}


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_config_pattern_sets_match_pinned_digests(name):
    cfg = configs.CONFIGS[name]
    s = configs.build_sphere_for(cfg, use_cache=False)
    assert configs.sphere_digest(s) == configs.SPHERE_SHA256[name]


# ---------------------------------------------------------------------------
# CWS1 (wsphere.py:237-286)

@pytest.mark.parametrize("name,n,k,r,size", [("ref_ca64_r1", 64, 16, 1, 10), ("ref_ca256_r3", 256, 16, 3, 538)])
def test_reference_written_cws1_files(tmp_path, name, n, k, r, size):
    path = os.path.join(GOLDEN, name + ".cws")
    s = load_sphere(path)
    assert (s.n, s.k, s.radius_index, s.size) == (n, k, r, size)
    mine = patterns.enumerate_sphere(codes.build_ca_polar_code(n, k), r)
    assert np.array_equal(_words(s), _words(mine))
    out = tmp_path / "re.cws"
    save_sphere(mine, out)
    with open(path, "rb") as fh:
        assert out.read_bytes() == fh.read()


def test_save_load_roundtrip_trivial_and_large(tmp_path):
    code = codes.build_ca_polar_code(256, 16)
    for r in (0, 4):
        s = patterns.enumerate_sphere(code, r)
        path = tmp_path / f"s{r}.cws"
        save_sphere(s, path)
        t = load_sphere(path)
        assert (t.n, t.k, t.radius_index) == (s.n, s.k, s.radius_index)
        assert np.array_equal(_words(t), _words(s))
        assert np.array_equal(t.shell_weights, s.shell_weights)
        assert np.array_equal(t.shell_counts, s.shell_counts)
        assert t.mean_nonzero_weight == s.mean_nonzero_weight


def test_load_rejects_corruption(tmp_path):
    s = patterns.enumerate_sphere(codes.build_ca_polar_code(64, 16), 1)
    path = tmp_path / "s.cws"
    save_sphere(s, path)
    raw = bytearray(path.read_bytes())
    bad = tmp_path / "bad_magic.cws"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(SphereFormatError, match="magic"):
        load_sphere(bad)
    flipped = bytearray(raw)
    flipped[len(flipped) // 2] ^= 0x40
    bad = tmp_path / "flipped.cws"
    bad.write_bytes(flipped)
    with pytest.raises(SphereFormatError, match="checksum"):
        load_sphere(bad)
    bad = tmp_path / "trunc.cws"
    bad.write_bytes(raw[:10])
    with pytest.raises(SphereFormatError):
        load_sphere(bad)


def test_sphere_order_is_canonical():
    """Member order: zero first, shell-major, lexicographic with word 0 most
    significant (wsphere.py:197-202), whatever order the words arrive in."""
    code = codes.build_ca_polar_code(128, 21)
    s = patterns.enumerate_sphere(code, 2)
    rng = np.random.default_rng(0)
    w = _words(s)[1:].copy()
    rng.shuffle(w)
    t = sphere_from_members(s.n, s.k, s.radius_index, w)
    assert np.array_equal(_words(t), _words(s))
