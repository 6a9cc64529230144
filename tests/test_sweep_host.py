"""Host-side pieces of the sweep harness (config parser, Wilson interval,
CSV format) against the reference's conventions (simharness.py)."""
import pytest

from paper_2602_08501_b200 import sweep


def test_parse_config_round_trip_and_formula():
    cfg = sweep.parse_config("""
code_family = ca_polar
code_n = 64
code_k = 16
snr_db_grid = 0.0, 1.0
stage1 = scl
wsd_filter_size = formula   # comment
seed = 5
max_trials = 100
""")
    assert cfg.snr_db_grid == [0.0, 1.0] and cfg.wsd_filter_size is None and cfg.seed == 5


@pytest.mark.parametrize("text,msg", [
    ("code_family = ca_polar\nbogus = 1", "unknown"),
    ("code_family = ca_polar\ncode_family = polar", "duplicate"),
    ("code_family = ca_polar", "missing"),
])
def test_parse_config_rejects(text, msg):
    with pytest.raises(sweep.ConfigError, match=msg):
        sweep.parse_config(text)


def test_crc_gated_needs_ca_family():
    with pytest.raises(sweep.ConfigError):
        sweep.parse_config("code_family = polar\ncode_n = 64\ncode_k = 16\nsnr_db_grid = 1\n"
                           "stage1 = scl\nseed = 1\nmax_trials = 10\nactivation_mode = crc_gated")


def test_wilson_interval_values():
    lo, hi = sweep.wilson_interval(112, 384)
    assert (format(lo, ".6g"), format(hi, ".6g")) == ("0.248446", "0.339014")   # sweep_two_stage.csv:2
    assert sweep.wilson_interval(0, 0) == (0.0, 1.0)


def test_build_code_label_and_rm_rejected():
    cfg = sweep.parse_config("code_family = ca_polar\ncode_n = 64\ncode_k = 16\nsnr_db_grid = 1\n"
                             "stage1 = scl\nseed = 1\nmax_trials = 10")
    assert sweep.build_code(cfg).label() == "ca-polar:64:16"
    cfg.code_family = "rm"
    with pytest.raises(sweep.ConfigError):
        sweep.build_code(cfg)
