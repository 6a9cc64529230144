"""GPU pattern-set enumeration (csrc/enum.cuh) against the native host walk
and the reference's committed spectra / sphere files."""

import numpy as np
import pytest

from paper_2602_08501_b200 import codes, configs, patterns

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_gpu_spectrum_matches_host_walk(name):
    code = configs.CONFIGS[name].code()
    assert np.array_equal(patterns.weight_spectrum_gpu(code), patterns.weight_spectrum(code))


@pytest.mark.parametrize("name,r", [("cfg1", 1), ("cfg1", 3), ("cfg2", 1), ("cfg3", 1), ("cfg3", 2)])
def test_gpu_sphere_matches_host_walk(name, r):
    code = configs.CONFIGS[name].code()
    a = patterns.enumerate_sphere_gpu(code, r)
    b = patterns.enumerate_sphere(code, r)
    assert np.array_equal(np.asarray(a.member_words), np.asarray(b.member_words))
    assert a.radius_index == b.radius_index


def test_gpu_spectrum_rm_2_7_known_distribution():
    """RM(2,7): A_32 = 10668 minimum-weight words, A_0 = A_128 = 1, total 2^29."""
    spec = patterns.weight_spectrum_gpu(configs.CONFIGS["cfg2"].code())
    assert spec[0] == 1 and spec[128] == 1 and spec[32] == 10668
    assert int(spec.sum()) == 1 << 29
    assert np.array_equal(spec, spec[::-1])


def test_gpu_enumerate_small_codes_and_limits():
    for n, k in ((32, 6), (64, 7), (64, 20), (128, 11), (256, 9)):
        code = codes.build_polar_code(n, k)
        assert np.array_equal(patterns.weight_spectrum_gpu(code), patterns.weight_spectrum(code)), (n, k)
    with pytest.raises(ValueError):
        patterns.enumerate_sphere_gpu(codes.build_polar_code(64, 10), 99)
    with pytest.raises(ValueError):
        patterns.weight_spectrum_gpu(configs.CONFIGS["cfg4"].code())


@pytest.mark.parametrize("r,size", [(3, 538), (4, 6472)])
def test_gpu_criterion_1_sphere_sizes_256_16(r, size):
    """enum_kernel reproduces criterion 1 (reference tests/test_acceptance.py:51-71)
    member for member against the host walk."""
    code = codes.build_ca_polar_code(256, 16)
    a = patterns.enumerate_sphere_gpu(code, r)
    assert a.size == size
    assert np.array_equal(np.asarray(a.member_words), np.asarray(patterns.enumerate_sphere(code, r).member_words))
