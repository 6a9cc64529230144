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


# ---------------------------------------------------------------------------
# Sharded trial fold (sweep._sweep_rounds): ranks decode block-aligned trial
# ranges, the per-64-trial block sums are all-reduced, and every rank folds the
# same sequence with the reference's stopping rule (simharness.py:318-330).

import os
import socket

import numpy as np


def _synthetic(first, cnt):
    """Deterministic per-trial statistics (trials, errors, x): an error every
    ~9 trials, so min_block_errors stops the point mid-round."""
    t = np.arange(first, first + cnt, dtype=np.int64)
    err = ((t * 2654435761) % 97) < 11
    return np.stack([np.ones(cnt, np.int64), err.astype(np.int64), t % 5], axis=1)


def _sequential_fold(cfg):
    """The reference's loop, trial by trial in batches of 64."""
    trials = errors = x = 0
    t = 0
    while t < cfg.max_trials and trials < cfg.max_trials and errors < cfg.min_block_errors:
        st = _synthetic(t, min(64, cfg.max_trials - t))
        trials += int(st[:, 0].sum())
        errors += int(st[:, 1].sum())
        x += int(st[:, 2].sum())
        t += 64
    return [trials, errors, x]


class _Cfg:
    def __init__(self, max_trials, min_block_errors):
        self.max_trials, self.min_block_errors = max_trials, min_block_errors


CASES = [(4000, 100), (4000, 10 ** 9), (1000, 30), (130, 10 ** 9), (64, 1)]


def _fold_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for mt, mbe in CASES:
        for batch in (64, 192, 1024):
            out.append(sweep._sweep_rounds(_Cfg(mt, mbe), batch, sweep._Ranks(), _synthetic, 3))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fold_equals_sequential_fold(world):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fold_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [_sequential_fold(_Cfg(mt, mbe)) for mt, mbe in CASES for _ in (64, 192, 1024)]
    for r in range(world):
        assert res[r] == want


def test_single_process_fold_and_batch_validation():
    for mt, mbe in CASES:
        for batch in (64, 4096):
            assert sweep._sweep_rounds(_Cfg(mt, mbe), batch, sweep._Ranks(), _synthetic, 3) == \
                _sequential_fold(_Cfg(mt, mbe))
    for bad in (0, 100, 63):
        with pytest.raises(sweep.ConfigError):
            sweep._check_batch(bad)
