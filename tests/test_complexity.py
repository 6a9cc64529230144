"""ED-unit accounting and the closed-form cost models (complexity.py), checked
on the values the reference's tests pin (tests/test_complexity.py)."""
import pytest

from paper_2602_08501_b200.complexity import (OpCounter, c_bpc, c_mp_wsd, c_osd, c_scl, c_wsd,
                                              to_ed_units)
from paper_2602_08501_b200.decoders import gain_metric
from paper_2602_08501_b200.channel import llr, modulate_bits, squared_distance


def test_ed_units():
    for n in (64, 500):
        assert to_ed_units(OpCounter(ed_evaluations=1), n) == 1.0
    assert to_ed_units(OpCounter(), 64) == 0.0
    assert to_ed_units(OpCounter(gain_additions=231), 77) == 1.0
    c = OpCounter(scl_node_ops=3, sort_comparisons=6, osd_reencodes=2, misc_flops=12)
    assert to_ed_units(c, 4) == pytest.approx((12 + 6 + 24 + 12) / 12)
    with pytest.raises(ValueError):
        to_ed_units(c, 0)


def test_counter_algebra():
    a, b, c = OpCounter(1, 2, 3, 4, 5, 6), OpCounter(10, 20, 30, 40, 50, 60), OpCounter(100, 0, 1, 0, 2, 7)
    assert (a + b) + c == a + (b + c) and a + b == b + a
    acc = OpCounter()
    acc.merge(a)
    acc.merge(b)
    assert acc == a + b


def test_cost_models():
    assert c_scl(16, 256) == pytest.approx(512 / 3)
    assert c_scl(8, 128) == pytest.approx(2 * c_scl(4, 128))
    assert c_bpc(4, 64, []) == c_scl(4, 64)
    assert c_bpc(32, 128, [64, 64]) == pytest.approx(32 * 28 / 3 + 4 * 768 / 384)
    assert (c_osd(0, 29), c_osd(2, 29), c_osd(4, 29)) == (1, 436, 27841)
    assert c_wsd(1, 1, 64, 100, 12.0) == pytest.approx(1 + 1 / 192 + 1200 / 192)
    assert c_wsd(4, 11, 64, 100, 12.0) == pytest.approx(4 * c_wsd(1, 11, 64, 100, 12.0))
    assert c_mp_wsd(100.0, 1.0, 1, 321.0) == 421.0
    for bad in (lambda: c_wsd(0, 1, 64, 100, 1.0), lambda: c_mp_wsd(1.0, 1.5, 1, 1.0),
                lambda: c_scl(4, 48), lambda: c_bpc(4, 64, [48])):
        with pytest.raises(ValueError):
            bad()


def test_gain_metric_is_the_exact_correlation_change():
    import numpy as np
    rng = np.random.default_rng(3)
    y = rng.normal(size=32)
    c = rng.integers(0, 2, 32)
    s = np.zeros(32, np.int64)
    s[[1, 4, 9, 30]] = 1
    x, xs = modulate_bits(c), modulate_bits(c ^ s)
    assert gain_metric(y, x, np.flatnonzero(s)) == pytest.approx(float(y @ xs - y @ x), abs=1e-12)
    assert gain_metric(y, x, []) == 0.0
    # Delta ED = -2 G
    assert squared_distance(y, xs) - squared_distance(y, x) == pytest.approx(
        -2 * gain_metric(y, x, np.flatnonzero(s)), abs=1e-12)
    assert np.allclose(llr(y, 0.5), 8 * y)
    with pytest.raises(ValueError):
        llr(y, 0.0)
