"""Certification soundness for pattern sets with weights above 64 (ADVICE r1:
the fp32 re-scoring bound is gamma_{wmax-1} * sum|y|, not gamma_63).

P = every nonzero codeword of CA-polar(128,16)+CRC-11 (weights up to 128), so
one hop from the zero codeword is exact ML (the reference's criterion-3
identity, decoders.py:140-167).  Every screen -- 1-limb and 2-limb fp16
tensor, fp32 gather, and the float64-input path -- must return the exact
float64 argmin found by brute force here.
"""
import numpy as np
import pytest

from paper_2602_08501_b200 import channel, codes
from paper_2602_08501_b200.decoders import DeviceDecoder, ml_decode, words32_to_64
from paper_2602_08501_b200.patterns import enumerate_sphere, weight_spectrum

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ml_setup():
    code = codes.build_ca_polar_code(128, 16)
    spec = weight_spectrum(code)
    sph = enumerate_sphere(code, int((spec[1:] > 0).sum()))
    assert int(sph.member_weights.max()) > 64
    msgs = ((np.arange(1 << code.k)[:, None] >> np.arange(code.k)) & 1).astype(np.uint8)
    cws = codes.encode_batch(code, msgs)
    x = channel.modulate_words(cws, code.n)
    return code, sph, cws, x


def _brute(x, cws, y64):
    corr = y64 @ x.T
    return cws[np.argmax(corr, axis=1)]


@pytest.mark.parametrize("variant", ["tensor", "tensor2", "gather", "auto"])
def test_full_codebook_hop_is_exact_ml(ml_setup, variant):
    code, sph, cws, x = ml_setup
    sigma = channel.ebno_to_sigma(0.5, code.k / code.n)
    _, _, y = channel.trial_inputs(code, 31, 0, range(256), sigma)
    y32 = y.astype(np.float32)
    dec = DeviceDecoder(code, sph)
    o = dec.mp_wsd_batch(y32, np.zeros((len(y32), 1, dec.nw), np.uint32), 1, variant=variant)
    got = words32_to_64(o["best"].cpu().numpy().view(np.uint32), code.n)
    np.testing.assert_array_equal(got, _brute(x, cws, y32.astype(np.float64)))
    # float64 inputs: exact on the un-rounded values
    if variant in ("tensor", "gather", "auto"):
        o = dec.mp_wsd_batch(y, np.zeros((len(y), 1, dec.nw), np.uint32), 1, variant=variant)
        got = words32_to_64(o["best"].cpu().numpy().view(np.uint32), code.n)
        np.testing.assert_array_equal(got, _brute(x, cws, y))


def test_ml_decode_dropin_n128(ml_setup):
    code, sph, cws, x = ml_setup
    sigma = channel.ebno_to_sigma(1.0, code.k / code.n)
    _, _, y = channel.trial_inputs(code, 32, 0, range(48), sigma)
    ref = _brute(x, cws, y)
    for f in range(len(y)):
        cw, ed = ml_decode(y[f], code)
        np.testing.assert_array_equal(np.asarray(cw.words), ref[f])
