"""Counter-based channel generator: Philox4x32-10 known answers (Random123
kat_vectors), statistics of the numpy mirror, and (GPU) agreement of the
device generator with the mirror."""
import numpy as np
import pytest

from paper_2602_08501_b200 import channel, configs


def _ph(c, k):
    r = channel.philox4x32_10(*[np.array([x], np.uint32) for x in c], *k)
    return [int(v[0]) for v in r]


def test_philox4x32_10_known_answers():
    assert _ph((0, 0, 0, 0), (0, 0)) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    f = 0xffffffff
    assert _ph((f, f, f, f), (f, f)) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert _ph((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0)) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_keyed_stream_statistics_and_codewords():
    code = configs.CONFIGS["cfg3"].code()
    msg, cw, y = channel.keyed_inputs_host(code, 11, 2, 4096, 20000, 0.8)
    from paper_2602_08501_b200.codes import encode_batch
    bits = ((msg[:, None] >> np.arange(code.k, dtype=np.uint64)) & np.uint64(1)).astype(np.uint8)
    np.testing.assert_array_equal(encode_batch(code, bits), cw)
    x = channel.modulate_words(cw, code.n)
    z = (y.astype(np.float64) - x) / 0.8
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    assert 0.45 < bits.mean() < 0.55
    # frame-range independence: frames are a pure function of their index
    _, cw2, y2 = channel.keyed_inputs_host(code, 11, 2, 4096 + 100, 50, 0.8)
    np.testing.assert_array_equal(y2, y[100:150])
    np.testing.assert_array_equal(cw2, cw[100:150])


@pytest.mark.gpu
def test_device_generator_matches_host_mirror():
    from paper_2602_08501_b200.decoders import DeviceDecoder, device_channel, words32_to_64
    for name in ("cfg1", "cfg4"):
        code = configs.CONFIGS[name].code()
        dec = DeviceDecoder(code)
        y, tx, msg = device_channel(dec, 123456789, 3, 1 << 20, 5000, 1.3)
        m_h, cw_h, y_h = channel.keyed_inputs_host(code, 123456789, 3, 1 << 20, 5000, 1.3)
        np.testing.assert_array_equal(msg.cpu().numpy().view(np.uint64), m_h)
        np.testing.assert_array_equal(words32_to_64(tx.cpu().numpy().view(np.uint32), code.n), cw_h)
        yd = y.cpu().numpy()
        diff = yd != y_h
        assert diff.mean() < 1e-5
        if diff.any():   # float64 libm differences only: 1 float32 ulp
            assert np.all(np.abs(yd[diff] - y_h[diff]) <= np.spacing(np.abs(y_h[diff])))
