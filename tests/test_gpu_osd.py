"""OSD stage 1 on the GPU (csrc/osd.cuh) and OSD-initialised two-stage decoding
against the reference's golden vectors, the oracle, and the reference's own
OSD / ML unit tests restated on the drop-in API (tests/test_decoders.py:150-190,
366-390; tests/test_acceptance.py:289-296)."""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_08501_b200 import channel, codes, configs
from paper_2602_08501_b200 import decoders as D
from paper_2602_08501_b200.decoders import OpCounter, OsdStage, WsdParams
from paper_2602_08501_b200.patterns import enumerate_sphere
from tests.helpers import (code_and_sphere, load, osd_code, osd_list_fixtures, osd_sphere,
                           osd_two_stage_fixtures)

pytestmark = pytest.mark.gpu


def _w64(t, n):
    return D.words32_to_64(t.cpu().numpy().view(np.uint32), n)


def _msg_bits(msg64, k):
    return ((np.asarray(msg64, np.int64)[:, None] >> np.arange(k)) & 1).astype(np.uint8)


@pytest.mark.parametrize("fx", osd_list_fixtures())
def test_gpu_osd_lists_match_reference(fx):
    """Same words in the same order as the reference's osd_decode (fast
    top-M path for cap <= 95, stable segmented sort for the full lists)."""
    g = load(fx)
    code = osd_code(fx)
    dec = D.get_decoder(code, None)
    o = dec.osd_batch(g["y32"], int(g["order"]), int(g["list_cap"]) or None)
    cnt = o["list_n"].cpu().numpy()
    np.testing.assert_array_equal(cnt, g["list_n"])
    assert not o["flags"].cpu().numpy().any()
    cw = _w64(o["list_cw"], code.n)
    ed = o["list_ed"].cpu().numpy()
    for f in range(cnt.size):
        c = int(cnt[f])
        np.testing.assert_array_equal(cw[f, :c], g["list_cw"][f, :c])
        np.testing.assert_allclose(ed[f, :c], g["list_ed"][f, :c], rtol=1e-12, atol=0)


@pytest.mark.parametrize("variant", ["gather", "tensor"])
@pytest.mark.parametrize("fx", osd_two_stage_fixtures())
def test_gpu_osd_two_stage_matches_reference(fx, variant):
    g = load(fx)
    code = osd_code(fx)
    sph = osd_sphere(g, code)
    dec = D.DeviceDecoder(code, sph)
    try:
        mode = "crc_gated" if int(g["gated"]) else "always_on"
        o = dec.two_stage_osd_batch(g["y32"], int(g["order"]), int(g["list_cap"]) or None,
                                    int(g["num_paths"]), int(g["max_iterations"]), mode,
                                    variant=variant, want_anchors=True)
        assert not o["flags"].cpu().numpy().any()
        np.testing.assert_array_equal(o["stage"].cpu().numpy(), g["stage"])
        np.testing.assert_array_equal(_w64(o["best"], code.n), g["best"])
        np.testing.assert_array_equal(_msg_bits(o["best_msg"].cpu().numpy(), code.k), g["best_msg"])
        s2 = g["stage"] == 1
        np.testing.assert_array_equal(o["iters"].cpu().numpy()[s2], g["iters"][s2])
        np.testing.assert_array_equal(_w64(o["anchors"], code.n)[s2], g["anchors"][s2])
        np.testing.assert_allclose(o["best_ed"].cpu().numpy(), g["squared_ed"], rtol=1e-12, atol=0)
    finally:
        dec.close()


def _compare_with_flags(gpu_best, orc_best, flags):
    diff = (gpu_best != orc_best).any(axis=1)
    assert not (diff & (flags == 0)).any(), f"{int(diff.sum())} mismatches, unflagged"
    return int(diff.sum())


@pytest.mark.parametrize("order,cap,frames,ebno", [(2, 64, 1500, 2.0), (3, 16, 300, 3.0)])
def test_gpu_osd_rm_two_stage_random_vs_oracle(order, cap, frames, ebno):
    """configs/rm_128_29_osd2_r1.cfg shape: OSD(order) + always-on r=1, A=4, J=4."""
    code, sph = code_and_sphere(configs.CONFIGS["cfg2"])
    sigma = channel.ebno_to_sigma(ebno, code.k / code.n)
    _, _, y = channel.trial_inputs(code, 31, 0, range(frames), sigma)
    y32 = y.astype(np.float32)
    dec = D.get_decoder(code, sph)
    o = dec.two_stage_osd_batch(y32, order, cap, 4, 4, "always_on", want_anchors=True)
    r = orc.two_stage_batch(y32, code, sph, 1, 4, 4, False, 1.0, nthreads=16, want_anchors=True,
                            osd_order=order, osd_cap=cap)
    flags = o["flags"].cpu().numpy()
    _compare_with_flags(_w64(o["best"], code.n), r["best"], flags)
    ok = flags == 0
    np.testing.assert_array_equal(o["iters"].cpu().numpy()[ok], r["iters"][ok])
    np.testing.assert_array_equal(_w64(o["anchors"], code.n)[ok], r["anchors"][ok])


def test_gpu_osd_cfg4_two_stage_random_vs_oracle():
    """K = 53, N = 256 (eight words): OSD(1) + always-on MP-WSD over cfg4's P."""
    cfg = configs.CONFIGS["cfg4"]
    code, sph = code_and_sphere(cfg)
    sigma = cfg.sigma(code=code)
    _, _, y = channel.trial_inputs(code, 5, 0, range(96), sigma)
    y32 = y.astype(np.float32)
    dec = D.get_decoder(code, sph)
    o = dec.two_stage_osd_batch(y32, 1, None, 4, cfg.max_iterations, "always_on")
    r = orc.two_stage_batch(y32, code, sph, 1, 4, cfg.max_iterations, False, 1.0, nthreads=16,
                            osd_order=1, osd_cap=None)
    _compare_with_flags(_w64(o["best"], code.n), r["best"], o["flags"].cpu().numpy())


@pytest.mark.parametrize("name,order,cap", [("cfg3", 3, 20), ("cfg1", 4, None), ("cfg4", 2, 40)])
def test_gpu_osd_lists_random_vs_oracle(name, order, cap):
    cfg = configs.CONFIGS[name]
    code = cfg.code()
    sigma = cfg.sigma(code=code)
    _, _, y = channel.trial_inputs(code, 17, 0, range(200), sigma)
    y32 = y.astype(np.float32)
    o = D.get_decoder(code, None).osd_batch(y32, order, cap)
    n, cw, ed = orc.osd_batch(y32, code, order, cap, nthreads=16)
    flags = o["flags"].cpu().numpy()
    np.testing.assert_array_equal(o["list_n"].cpu().numpy(), n)
    g = _w64(o["list_cw"], code.n)
    bad = [(g[f] != cw[f]).any() for f in range(n.size)]
    assert not any(b and not fl for b, fl in zip(bad, flags))
    np.testing.assert_allclose(o["list_ed"].cpu().numpy(), ed, rtol=1e-12, atol=0)


def test_gpu_osd_gated_ca_codes_pass_stage1_with_the_min_ed_candidate():
    """Every OSD candidate of a CA code is in the subcode, so the gate passes on
    the first entry (decoders.py:559-570)."""
    cfg = configs.CONFIGS["cfg3"]
    code, sph = code_and_sphere(cfg)
    sigma = channel.ebno_to_sigma(1.0, code.k / code.n)
    _, _, y = channel.trial_inputs(code, 23, 0, range(500), sigma)
    y32 = y.astype(np.float32)
    dec = D.get_decoder(code, sph)
    o = dec.two_stage_osd_batch(y32, 2, None, 8, 8, "crc_gated")
    assert (o["stage"].cpu().numpy() == 0).all()
    lst = dec.osd_batch(y32, 2, 1)
    np.testing.assert_array_equal(o["best"].cpu().numpy(), lst["list_cw"][:, 0].cpu().numpy())


# ---- the reference's OSD / ML unit tests on the drop-in API ----------------

def _random_code(rng, k, n):
    while True:
        bits = rng.integers(0, 2, (k, n), dtype=np.uint8)
        if len(codes.gf2_row_reduce(bits)[1]) == k:
            return codes.LinearCode(n, k, codes.GenMatrix(codes.pack_bits(bits), n), kind="generic")


def _x(bits):
    return 1.0 - 2.0 * np.asarray(bits, np.float64)


def _encode_bits(code, msg):
    return codes.encode(code, codes.BitVector.from_bits(msg)).bits()


def test_osd_noiseless_order_zero():
    rng = np.random.default_rng(6)
    code = codes.build_rm_code(4, 2)
    cw = _encode_bits(code, rng.integers(0, 2, code.k, dtype=np.uint8))
    out = D.osd_decode(_x(cw), code, 0)
    assert np.array_equal(out.entries[0][0].bits(), cw) and out.entries[0][1] == 0.0


@pytest.mark.parametrize("k,n,trials", [(8, 16, 100), (10, 20, 200)])
def test_osd_full_order_equals_ml(k, n, trials):
    rng = np.random.default_rng(7)
    code = _random_code(rng, k, n)
    for _ in range(trials):
        y = _x(_encode_bits(code, rng.integers(0, 2, k, dtype=np.uint8))) + rng.normal(size=n)
        top = D.osd_decode(y, code, k, list_cap=1).entries[0][0]
        assert top == D.ml_decode(y, code)[0]


def test_osd_candidate_count_is_binomial_sum():
    code = codes.build_rm_code(7, 2)
    counters = OpCounter()
    out = D.osd_decode(np.ones(128) * 0.1, code, 2, counters=counters)
    expected = 1 + 29 + math.comb(29, 2)
    assert counters.osd_reencodes == expected == 436
    assert len(out.entries) == expected


def test_osd_candidates_are_codewords_and_capped():
    rng = np.random.default_rng(8)
    code = codes.build_rm_code(3, 1)
    y = rng.normal(size=8)
    out = D.osd_decode(y, code, 2, list_cap=5)
    assert len(out.entries) == 5
    book = {tuple(_encode_bits(code, np.array([(m >> i) & 1 for i in range(code.k)], np.uint8)))
            for m in range(1 << code.k)}
    for cw, score in out.entries:
        assert tuple(cw.bits()) in book
        assert score == pytest.approx(float(((y - _x(cw.bits())) ** 2).sum()))


def test_osd_rejects_negative_order():
    with pytest.raises(ValueError):
        D.osd_decode(np.zeros(8), codes.build_rm_code(3, 1), -1)


def test_two_stage_crc_gated_needs_crc_code():
    code = codes.build_rm_code(3, 1)
    sphere = enumerate_sphere(code, 1)
    with pytest.raises(ValueError, match="crc"):
        D.two_stage_decode(np.zeros(8), code, OsdStage(1), WsdParams(radius_index=1), sphere)


def test_two_stage_osd_always_on_on_rm_code():
    rng = np.random.default_rng(20)
    code = codes.build_rm_code(4, 1)
    sphere = enumerate_sphere(code, 1)
    params = WsdParams(radius_index=1, num_paths=2, activation_mode="always_on")
    msg = rng.integers(0, 2, code.k, dtype=np.uint8)
    y = _x(_encode_bits(code, msg)) + 0.4 * rng.normal(size=16)
    res = D.two_stage_decode(y, code, OsdStage(1), params, sphere)
    assert res.stage == "mp_wsd"
    assert res.best_message is not None
    assert res.squared_ed == pytest.approx(float(((y - _x(res.best_codeword.bits())) ** 2).sum()),
                                           rel=1e-15)


def test_ml_decode_matches_exhaustive_search():
    rng = np.random.default_rng(9)
    code = _random_code(rng, 12, 32)
    msgs = np.array([[(m >> i) & 1 for i in range(12)] for m in range(1 << 12)], np.uint8)
    book = np.array([_encode_bits(code, m) for m in msgs])
    for _ in range(20):
        y = _x(book[rng.integers(0, len(book))]) + 0.8 * rng.normal(size=32)
        eds = ((y.astype(np.float32).astype(np.float64)[None, :] - _x(book)) ** 2).sum(axis=1)
        cw, ed = D.ml_decode(y, code)
        assert np.array_equal(cw.bits(), book[int(np.argmin(eds))])
    with pytest.raises(ValueError):
        D.ml_decode(np.zeros(128), codes.build_rm_code(7, 2))
