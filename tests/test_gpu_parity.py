"""GPU parity: the sm_100a path through the C-ABI against the reference's
golden vectors and the CPU oracle.

Bar: stage-1 lists bit-exact (codewords, order, float64 PMs); decoded
codewords bit-identical except frames the kernel flags as near-ties
(candidates within 1e-5 relative ED), which must be rare.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_08501_b200 import configs
from paper_2602_08501_b200.decoders import DeviceDecoder, words32_to_64, words64_to_32
from paper_2602_08501_b200._native import FLAG_TIE_FINAL as TIE_FINAL, FLAG_UNRESOLVED as UNRESOLVED
from tests.helpers import cfg_of, code_and_sphere, load, scl_fixtures, two_stage_fixtures

pytestmark = pytest.mark.gpu

_decs = {}


def decoder(cfg):
    if cfg.name not in _decs:
        code, sph = code_and_sphere(cfg)
        _decs[cfg.name] = DeviceDecoder(code, sph)
    return _decs[cfg.name]


def _np(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("fx", scl_fixtures())
def test_scl_lists_bit_exact_vs_reference(fx):
    g = load(fx)
    cfg = cfg_of(fx)
    dec = DeviceDecoder(cfg.code().inner if cfg.code().kind == "crc_concatenated" else cfg.code())
    o = dec.scl_batch(llrs=g["llrs"], list_size=int(g["list_size"]))
    n = g["llrs"].shape[1]
    np.testing.assert_array_equal(_np(o["list_n"]), g["list_n"])
    cw = words32_to_64(_np(o["list_cw"]).view(np.uint32), n)
    pm = _np(o["list_pm"])
    for f in range(g["llrs"].shape[0]):
        c = int(g["list_n"][f])
        np.testing.assert_array_equal(cw[f, :c], g["list_cw"][f, :c])
        np.testing.assert_array_equal(pm[f, :c], g["list_pm"][f, :c])


VARIANTS = ["gather", "tensor", "tensor2", "tensor_i8", "tensor_i8a"]


def _skip_i8(variant, n):
    if variant in ("tensor_i8", "tensor_i8a") and n not in (128, 256):
        pytest.skip("int8 screen: N = 128, 256")


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("fx", two_stage_fixtures())
def test_two_stage_vs_reference_golden(fx, variant):
    g = load(fx)
    cfg = cfg_of(fx)
    _skip_i8(variant, g["y32"].shape[1])
    dec = decoder(cfg)
    mode = "crc_gated" if int(g["gated"]) else "always_on"
    o = dec.two_stage_batch(g["y32"], float(g["sigma"]), int(g["list_size"]), int(g["num_paths"]),
                            int(g["max_iterations"]), mode, variant=variant, want_anchors=True)
    n = g["y32"].shape[1]
    stage = _np(o["stage"])
    np.testing.assert_array_equal(stage, g["stage"])
    best = words32_to_64(_np(o["best"]).view(np.uint32), n)
    flags = _np(o["flags"])
    mism = np.flatnonzero((best != g["best"]).any(axis=1))
    risky = np.flatnonzero(flags & (UNRESOLVED | TIE_FINAL))
    assert set(mism.tolist()) <= set(risky.tolist()), f"uncertified mismatches {mism}"
    ok = np.setdiff1d(np.arange(len(stage)), risky)
    np.testing.assert_array_equal(_np(o["iters"])[ok], g["iters"][ok])
    anc = words32_to_64(_np(o["anchors"]).view(np.uint32), n)
    s2 = np.flatnonzero(stage == 1)
    np.testing.assert_array_equal(anc[s2], g["anchors"][s2])
    np.testing.assert_allclose(_np(o["best_ed"])[ok], g["squared_ed"][ok], rtol=1e-12)
    # message_of on the device
    msg = _np(o["best_msg"]).view(np.uint64)
    kbits = g["best_msg"].shape[1]
    ref_msg = (g["best_msg"].astype(np.uint64) << np.arange(kbits, dtype=np.uint64)).sum(axis=1)
    np.testing.assert_array_equal(msg[ok], ref_msg[ok])


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg2", "cfg4"])
def test_two_stage_vs_oracle_random_frames(name, variant):
    cfg = configs.CONFIGS[name]
    code, sph = code_and_sphere(cfg)
    _skip_i8(variant, code.n)
    from paper_2602_08501_b200 import channel
    sigma = cfg.sigma(code=code)
    F = {"cfg1": 4096, "cfg3": 2048, "cfg2": 256, "cfg4": 96}[name]
    if variant in ("tensor_i8", "tensor_i8a") and name in ("cfg2", "cfg4"):
        F *= 4      # the int8 screen's wider window: more frames
    if name == "cfg4" and variant == "gather":
        F = 32
    _, cw, y = channel.bulk_inputs(code, 11, 0, 0, F, sigma)
    o = decoder(cfg).two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                                     cfg.activation_mode, variant=variant)
    r = orc.two_stage_batch(y, code, sph, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                            cfg.activation_mode == "crc_gated", sigma, nthreads=8)
    np.testing.assert_array_equal(_np(o["stage"]), r["stage"])
    best = words32_to_64(_np(o["best"]).view(np.uint32), code.n)
    flags = _np(o["flags"])
    mism = np.flatnonzero((best != r["best"]).any(axis=1))
    risky = np.flatnonzero(flags & (UNRESOLVED | TIE_FINAL))
    assert set(mism.tolist()) <= set(risky.tolist()), f"uncertified mismatches {mism}"
    assert len(risky) <= max(1, F // 200)
    ok = np.setdiff1d(np.arange(F), risky)
    np.testing.assert_array_equal(_np(o["iters"])[ok], r["iters"][ok])


@pytest.mark.parametrize("variant,name", [(v, "cfg1") for v in VARIANTS[:3]] +
                         [("tensor_i8", "cfg3"), ("tensor_i8", "cfg2"), ("tensor", "cfg2"),
                          ("tensor_i8a", "cfg3"), ("tensor_i8a", "cfg2")])
def test_mp_wsd_random_anchors_vs_oracle(variant, name):
    cfg = configs.CONFIGS[name]
    code, sph = code_and_sphere(cfg)
    rng = np.random.default_rng(5)
    F, A, T = (1000, 4, 4) if name != "cfg2" else (200, 8, 6)
    from paper_2602_08501_b200.codes import encode_batch
    msgs = rng.integers(0, 2, (F * A, code.k), dtype=np.uint8)
    anc64 = encode_batch(code, msgs).reshape(F, A, -1)
    y = rng.normal(size=(F, code.n)).astype(np.float32)
    o = decoder(cfg).mp_wsd_batch(y, words64_to_32(anc64, code.n), T, variant=variant)
    r = orc.mpwsd_batch(y, anc64, sph, T, nthreads=8)
    best = words32_to_64(_np(o["best"]).view(np.uint32), code.n)
    flags = _np(o["flags"])
    mism = np.flatnonzero((best != r["best"]).any(axis=1))
    risky = np.flatnonzero(flags & (UNRESOLVED | TIE_FINAL))
    assert set(mism.tolist()) <= set(risky.tolist())
    ok = np.setdiff1d(np.arange(F), risky)
    np.testing.assert_array_equal(_np(o["iters"])[ok], r["iters"][ok])
    np.testing.assert_array_equal(_np(o["hops"])[ok], r["hops"][ok])


@pytest.mark.parametrize("generic", [0, 1])
@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg4"])
def test_scl_kernels_agree_bit_exact(name, generic):
    """Lane-per-path and warp-per-frame stage-1 kernels give identical lists."""
    import ctypes
    from paper_2602_08501_b200 import _native, channel
    cfg = configs.CONFIGS[name]
    code = cfg.code()
    inner = code.inner
    sigma = cfg.sigma(code=code)
    _, _, y = channel.bulk_inputs(code, 21, 0, 0, 512, sigma)
    dec = DeviceDecoder(inner)
    _native.check(_native.lib().mpw_set_option(dec._h, b"scl_generic", generic))
    o = dec.scl_batch(y=y, sigma=sigma, list_size=cfg.list_size)
    llr = 2.0 * y.astype(np.float64) / (sigma * sigma)
    for f in range(0, 512, 37):
        u, cw, pm = orc.scl(llr[f], inner.info_set, code.n, cfg.list_size)
        c = int(o["list_n"][f].item())
        assert c == cw.shape[0]
        got = words32_to_64(o["list_cw"][f, :c].cpu().numpy().view(np.uint32), code.n)
        np.testing.assert_array_equal(got, cw)
        np.testing.assert_array_equal(o["list_pm"][f, :c].cpu().numpy(), pm)


@pytest.mark.parametrize("name", ["cfg4", "cfg2"])
def test_int8_window_overflow_continuation(name):
    """int8 screen: with the overflow threshold forced down to 4 keys (profiling
    knob 2048), most scans take continuation passes; decisions must still equal
    the oracle's, with no frame left unresolved."""
    cfg = configs.CONFIGS[name]
    code, sph = code_and_sphere(cfg)
    from paper_2602_08501_b200 import channel
    sigma = cfg.sigma(code=code)
    F = 128 if name == "cfg4" else 256
    _, cw, y = channel.bulk_inputs(code, 12, 0, 0, F, sigma)
    dec = DeviceDecoder(code, sph)
    dec.set_option("hop_experiment", 2048)      # window overflow at 4 keys
    o = dec.two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                                     cfg.activation_mode, variant="tensor_i8")
    r = orc.two_stage_batch(y, code, sph, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                            cfg.activation_mode == "crc_gated", sigma, nthreads=8)
    best = words32_to_64(_np(o["best"]).view(np.uint32), code.n)
    flags = _np(o["flags"])
    assert not (flags & UNRESOLVED).any()
    mism = np.flatnonzero((best != r["best"]).any(axis=1))
    risky = np.flatnonzero(flags & TIE_FINAL)
    assert set(mism.tolist()) <= set(risky.tolist()), f"mismatches {mism}"
    ok = np.setdiff1d(np.arange(F), risky)
    np.testing.assert_array_equal(_np(o["iters"])[ok], r["iters"][ok])


def test_int8_pair_kernel_vs_oracle():
    """The cta_group::2 variant of the int8 screen (option i8_pair: one M = 256 MMA
    per K step for a CTA pair, each CTA holding half of every P stage) decodes
    like the oracle."""
    cfg = configs.CONFIGS["cfg4"]
    code, sph = code_and_sphere(cfg)
    from paper_2602_08501_b200 import channel
    sigma = cfg.sigma(code=code)
    F = 192
    _, cw, y = channel.bulk_inputs(code, 13, 0, 0, F, sigma)
    dec = DeviceDecoder(code, sph)
    dec.set_option("i8_pair", 1)
    o = dec.two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                                     cfg.activation_mode, variant="tensor_i8")
    r = orc.two_stage_batch(y, code, sph, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                            cfg.activation_mode == "crc_gated", sigma, nthreads=8)
    best = words32_to_64(_np(o["best"]).view(np.uint32), code.n)
    flags = _np(o["flags"])
    assert not (flags & UNRESOLVED).any()
    mism = np.flatnonzero((best != r["best"]).any(axis=1))
    assert set(mism.tolist()) <= set(np.flatnonzero(flags & TIE_FINAL).tolist())
    ok = np.flatnonzero(~(flags & TIE_FINAL).astype(bool))
    np.testing.assert_array_equal(_np(o["iters"])[ok], r["iters"][ok])


@pytest.mark.parametrize("quantised", [False, True])
@pytest.mark.parametrize("n", [64, 128, 256])
def test_scl_lane_every_list_size_vs_oracle(n, quantised):
    """Lane-per-path SCL (register-resident small levels, leaf decisions
    recovered from the root partial sums) against the oracle's scl_decode
    restatement for every supported list size: list sizes, codewords, leaf
    decisions u and float64 path metrics bit for bit.  The quantised case uses
    LLRs on a coarse grid with zeros, so path metrics tie and the check-node f
    sees zero minima (decoders.py:173-174, 219-228)."""
    from paper_2602_08501_b200.codes import build_polar_code
    code = build_polar_code(n, n // 4)
    rng = np.random.default_rng(1000 + n + int(quantised))
    F = 48
    llr = rng.normal(1.0, 1.6, size=(F, n))
    if quantised:
        llr = np.round(llr * 2.0) / 2.0
    dec = DeviceDecoder(code)
    for L in (4, 8, 16, 32):
        o = dec.scl_batch(llrs=llr, list_size=L)
        ln = _np(o["list_n"])
        cw = words32_to_64(_np(o["list_cw"]).view(np.uint32), n)
        uw = words32_to_64(_np(o["list_u"]).view(np.uint32), n)
        pm = _np(o["list_pm"])
        for f in range(F):
            u_ref, cw_ref, pm_ref = orc.scl(llr[f], code.info_set, n, L)
            c = cw_ref.shape[0]
            assert ln[f] == c, (L, f)
            np.testing.assert_array_equal(cw[f, :c], cw_ref, err_msg=f"L={L} frame {f}")
            np.testing.assert_array_equal(pm[f, :c], pm_ref, err_msg=f"L={L} frame {f}")
            u_bits = np.array([[(int(uw[f, i, j // 64]) >> (j % 64)) & 1 for j in range(n)]
                               for i in range(c)], dtype=np.uint8)
            np.testing.assert_array_equal(u_bits, u_ref, err_msg=f"L={L} frame {f}")


def _coop_info_sets(n):
    """Information sets that put the lane-per-path SCL through every shape of
    its cooperative frozen runs (csrc/scl_lane.cuh, SclCoop): run lengths from
    the minimum (8) to N - 1, runs that cover a whole right subtree while 1, 2
    or 4 paths live (levels 1, 2, 3), runs that end inside it, a first
    information leaf at 0 (no run) and scattered early information leaves."""
    e, q, h = n // 8, n // 4, n // 2
    tail = list(range(n - 6, n))
    return {
        "first_info_at_8": [8, 9] + tail,
        "only_last_leaf": [n - 1],
        "first_info_at_half": [h, h + 1] + tail,
        "whole_eighth_two_paths": [e - 1, 2 * e + 3] + tail,            # [e, 2e) frozen with 2 paths
        "whole_quarter_two_paths": [q - 1, h + 5] + tail,               # [q, 2q) frozen with 2 paths
        "whole_half_two_paths": [h - 1, n - 7] + tail[1:],              # [h, n-7) frozen runs with 2 paths
        "whole_eighth_four_paths": [e - 2, e - 1, 3 * e - 1] + tail,    # [e, 2e) with 4 paths, then inside [2e, 3e)
        "info_at_zero": [0, 1, e, q + 1] + tail,
        "scattered": [3, e + 9, q - 1, q + e, h - 1, h + e + 2, h + q] + tail,
    }


@pytest.mark.parametrize("n", [64, 128, 256])
def test_scl_cooperative_frozen_runs_vs_oracle(n):
    """decoders.py:181-268 on polar codes with arbitrary information sets: the
    frozen runs the lanes of a frame compute together must leave lists,
    codewords and float64 path metrics bit-equal to the depth-first schedule
    (the oracle's restatement), with LLR ties and zeros included."""
    from paper_2602_08501_b200.codes import polar_code_from_info_set
    F = 24
    for name, info in _coop_info_sets(n).items():
        info = sorted(set(i for i in info if 0 <= i < n))
        code = polar_code_from_info_set(n, info)
        rng = np.random.default_rng(n + len(name))
        llr = rng.normal(0.6, 1.8, size=(F, n))
        llr[F // 2:] = np.round(llr[F // 2:] * 2.0) / 2.0
        dec = DeviceDecoder(code)
        for L in (4, 8, 16, 32):
            o = dec.scl_batch(llrs=llr, list_size=L)
            ln = _np(o["list_n"])
            cw = words32_to_64(_np(o["list_cw"]).view(np.uint32), n)
            pm = _np(o["list_pm"])
            for f in range(F):
                _, cw_ref, pm_ref = orc.scl(llr[f], code.info_set, n, L)
                c = cw_ref.shape[0]
                assert ln[f] == c, (name, L, f)
                np.testing.assert_array_equal(cw[f, :c], cw_ref, err_msg=f"{name} L={L} frame {f}")
                np.testing.assert_array_equal(pm[f, :c], pm_ref, err_msg=f"{name} L={L} frame {f}")
