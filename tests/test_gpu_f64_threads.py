"""The drop-in under the reference's own calling conventions:

* float64 received words (the reference coerces y to float64 and decodes
  those values, decoders.py:411, 466, 538): golden vectors made by the
  reference from UN-ROUNDED float64 y (tests/golden/make_golden_f64.py),
  including adversarial wsd_step inputs whose decision flips when y is rounded
  to float32;
* wsd_step scores the step on y * x_center (decoders.py:374, 412-416), with a
  real-valued x_center;
* concurrent per-frame calls from a thread pool (simharness.py:318-330;
  criterion 9, tests/test_acceptance.py:307-327): results equal the serial
  ones for 1, 4 and 16 threads.
"""
import glob
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2602_08501_b200 import channel, configs
from paper_2602_08501_b200.bits import BitVector
from paper_2602_08501_b200.decoders import (DeviceDecoder, SclStage, WsdParams, get_decoder, two_stage_decode,
                                            words32_to_64, wsd_step, wsd_trajectory)
from paper_2602_08501_b200._native import FLAG_TIE_FINAL, FLAG_UNRESOLVED
from tests.helpers import GOLDEN, code_and_sphere, load

pytestmark = pytest.mark.gpu


def _np(t):
    return t.cpu().numpy()


def f64_fixtures():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "f64_two_stage_*.npz")))


@pytest.mark.parametrize("variant", ["auto", "tensor", "tensor_i8a", "gather"])
@pytest.mark.parametrize("fx", f64_fixtures())
def test_two_stage_float64_vs_reference(fx, variant):
    g = load(fx)
    cfg = configs.CONFIGS[fx.split("_")[3]]
    code, sph = code_and_sphere(cfg)
    if cfg.name == "cfg4" and variant == "gather":
        pytest.skip("gather at cfg4: minutes per batch")
    if variant == "tensor_i8a" and code.n not in (128, 256):
        pytest.skip("asynchronous-row int8 hop: N = 128, 256")
    dec = DeviceDecoder(code, sph)
    mode = "crc_gated" if int(g["gated"]) else "always_on"
    y = np.ascontiguousarray(g["y64"], dtype=np.float64)
    o = dec.two_stage_batch(y, float(g["sigma"]), int(g["list_size"]), int(g["num_paths"]),
                            int(g["max_iterations"]), mode, variant=variant)
    n = y.shape[1]
    np.testing.assert_array_equal(_np(o["stage"]), g["stage"])
    flags = _np(o["flags"])
    best = words32_to_64(_np(o["best"]).view(np.uint32), n)
    assert not np.any(flags & FLAG_UNRESOLVED)
    # a final pick between two centres whose float64 EDs tie to rounding may
    # differ (summation order); none of the fixtures has one
    risky = np.flatnonzero(flags & FLAG_TIE_FINAL)
    assert len(risky) <= len(flags) // 50
    ok = np.setdiff1d(np.arange(len(flags)), risky)
    np.testing.assert_array_equal(best[ok], g["best"][ok])
    np.testing.assert_array_equal(_np(o["iters"])[ok], g["iters"][ok])
    np.testing.assert_allclose(_np(o["best_ed"])[ok], g["squared_ed"][ok], rtol=1e-12)


@pytest.mark.parametrize("fx,step", [("f64_two_stage_cfg3_crc_gated_1p0dB.npz", 5),
                                     ("f64_two_stage_cfg2_always_on_3p0dB.npz", 6),
                                     ("f64_two_stage_cfg4_always_on_1p5dB.npz", 4)])
def test_two_stage_float64_per_frame_dropin(fx, step):
    g = load(fx)
    cfg = configs.CONFIGS[fx.split("_")[3]]
    code, sph = code_and_sphere(cfg)
    params = WsdParams(radius_index=sph.radius_index, max_iterations=cfg.max_iterations,
                       num_paths=cfg.num_paths, activation_mode="crc_gated" if int(g["gated"]) else "always_on")
    for f in range(0, g["y64"].shape[0], step):
        r = two_stage_decode(g["y64"][f], code, SclStage(cfg.list_size), params, sph, sigma=float(g["sigma"]))
        assert (r.stage == "mp_wsd") == bool(g["stage"][f])
        np.testing.assert_array_equal(np.asarray(r.best_codeword.words), g["best"][f])
        assert r.squared_ed == pytest.approx(float(g["squared_ed"][f]), rel=1e-13)


@pytest.mark.parametrize("name", ["cfg3", "cfg2", "cfg4"])
def test_wsd_step_float64_ties(name):
    """The two best hop candidates differ by ~1e-9 in S: the float64 path must
    take the reference's decision (it flips for ~half the cases on float32(y))."""
    g = load(f"f64_wsd_ties_{name}.npz")
    _, sph = code_and_sphere(configs.CONFIGS[name])
    n = sph.n
    W = g["centers"].shape[1]
    for f in range(g["y64"].shape[0]):
        c = BitVector(n, np.zeros(W, np.uint64))
        words, improved = wsd_step(g["y64"][f], c, np.ones(n), sph, int(g["m"]))
        assert improved == bool(g["step_improved"][f])
        np.testing.assert_array_equal(np.asarray(words.words), g["step_words"][f])


def test_wsd_step_real_valued_x_center_and_trajectory():
    g = load("f64_wsd_api_cfg1.npz")
    _, sph = code_and_sphere(configs.CONFIGS["cfg1"])
    n = sph.n
    params = WsdParams(radius_index=sph.radius_index, max_iterations=int(g["max_iterations"]), num_paths=1)
    for f in range(g["y64"].shape[0]):
        c = BitVector(n, g["centers"][f])
        words, improved = wsd_step(g["y64"][f], c, g["x_center"][f], sph, int(g["m"]))
        assert improved == bool(g["step_improved"][f])
        np.testing.assert_array_equal(np.asarray(words.words), g["step_words"][f])
        tr = wsd_trajectory(g["y64"][f], c, sph, params)
        assert tr.iterations_used == int(g["traj_iters"][f])
        np.testing.assert_array_equal(np.asarray(tr.centers[-1].words), g["traj_final"][f])
        eds = g["traj_eds"][f][~np.isnan(g["traj_eds"][f])]
        np.testing.assert_allclose(tr.squared_eds, eds, rtol=1e-13)


def test_float64_rejects_int8_and_two_limb_variants():
    code, sph = code_and_sphere(configs.CONFIGS["cfg4"])
    dec = DeviceDecoder(code, sph)
    y = np.zeros((4, code.n))
    for v in ("tensor_i8", "tensor2"):
        with pytest.raises(ValueError):
            dec.two_stage_batch(y, 1.0, 16, 16, 8, "always_on", variant=v)


# ---------------------------------------------------------------------------
# thread pool (criterion 9)

def _per_frame(args):
    y, code, sph, params, sigma = args
    r = two_stage_decode(y, code, SclStage(4), params, sph, sigma=sigma)
    return (np.asarray(r.best_codeword.words).tobytes(), r.stage, r.squared_ed,
            tuple(t.iterations_used for t in r.traces))


def test_thread_pool_per_frame_decodes_equal_serial():
    cfg = configs.CONFIGS["cfg1"]
    code, sph = code_and_sphere(cfg)
    sigma = cfg.sigma(code=code)
    _, _, y = channel.trial_inputs(code, 21, 0, range(2048), sigma)
    params = WsdParams(radius_index=sph.radius_index, max_iterations=cfg.max_iterations,
                       num_paths=cfg.num_paths, activation_mode="crc_gated")
    jobs = [(y[f], code, sph, params, sigma) for f in range(len(y))]
    serial = [_per_frame(j) for j in jobs]
    for threads in (4, 16):
        with ThreadPoolExecutor(threads) as ex:
            got = list(ex.map(_per_frame, jobs))
        assert got == serial, f"{threads} threads"
    # each thread decoded through its own handle
    assert get_decoder(code, sph) is get_decoder(code, sph)
    with ThreadPoolExecutor(2) as ex:
        others = list(ex.map(lambda _: id(get_decoder(code, sph)), range(2)))
    assert id(get_decoder(code, sph)) not in others
