"""ED-unit accounting (complexity.py), checked on the values the reference's
tests pin (tests/test_complexity.py)."""
import pytest

from paper_2602_08501_b200.complexity import OpCounter, to_ed_units
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
