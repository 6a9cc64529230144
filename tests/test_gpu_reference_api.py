"""The reference's decoder tests (/root/reference/pkg/tests/test_decoders.py,
test_acceptance.py criteria 3-5, 8) restated against the drop-in API, which
runs the sm_100a kernels through the C-ABI.  Each test names the reference
test it mirrors.  Exact-ML oracles come from the CPU restatement (oracle/) or
brute force here."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_08501_b200 import codes
from paper_2602_08501_b200.bits import BitVector, unpack_bits
from paper_2602_08501_b200.channel import modulate_words
from paper_2602_08501_b200.decoders import (CandidateList, DeviceDecoder, OpCounter, SclStage, WsdParams,
                                            default_filter_size, mp_wsd, scl_decode, two_stage_decode,
                                            wsd_step, wsd_trajectory, words64_to_32)
from paper_2602_08501_b200.patterns import enumerate_sphere, weight_spectrum

pytestmark = pytest.mark.gpu


def rand_msg(rng, k):
    return BitVector.from_bits(rng.integers(0, 2, k, dtype=np.uint8))


def modulate(cw):
    return modulate_words(np.asarray(cw.words)[None, :], cw.length)[0]


def sqd(y, cw):
    d = np.asarray(y, np.float64) - modulate(cw)
    return float(d @ d)


def ml_decode(y, code):
    """Exact argmin over all 2^K codewords (decoders.py:140-167 semantics)."""
    k = code.k
    msgs = ((np.arange(1 << k)[:, None] >> np.arange(k)) & 1).astype(np.uint8)
    cws = codes.encode_batch(code, msgs)
    x = modulate_words(cws, code.n)
    corr = x @ np.asarray(y, np.float64)
    i = int(np.argmax(corr))
    return BitVector(code.n, cws[i])


def full_sphere(code):
    spec = weight_spectrum(code)
    return enumerate_sphere(code, int((spec[1:] > 0).sum()))


@pytest.fixture(scope="module")
def ca64():
    return codes.build_ca_polar_code(64, 16)


@pytest.fixture(scope="module")
def ca64_r2(ca64):
    return enumerate_sphere(ca64, 2)


# --- SCL (test_decoders.py:100-146) ------------------------------------------

def test_scl_noiseless_roundtrip_list_one():                           # :116-122
    rng = np.random.default_rng(4)
    code = codes.build_polar_code(64, 16)
    for _ in range(20):
        cw = codes.encode(code, rand_msg(rng, 16))
        out = scl_decode(2.0 * modulate(cw) / 0.49, code, 1)
        assert out.entries[0][0] == cw


def test_scl_metrics_sorted_and_in_code():                              # :131-139
    rng = np.random.default_rng(5)
    code = codes.build_polar_code(32, 12)
    out = scl_decode(2.0 * rng.normal(size=32), code, 8)
    metrics = [m for _, m in out.entries]
    assert metrics == sorted(metrics)
    for cw, _ in out.entries:
        assert codes.encode(code, code.message_of(cw)) == cw


def test_scl_node_costs_match_the_model():                              # :142-146
    code = codes.build_polar_code(64, 16)
    c = OpCounter()
    scl_decode(np.ones(64), code, 4, c)
    assert c.scl_node_ops == 4 * 64 * 6


def test_scl_full_list_equals_ml_16_8():                                # :107-113, criterion 8
    rng = np.random.default_rng(3)
    code = codes.build_polar_code(16, 8)
    for _ in range(50):
        y = modulate(codes.encode(code, rand_msg(rng, 8))) + 0.9 * rng.normal(size=16)
        top = scl_decode(2.0 * y / 0.81, code, 32).entries[0][0]      # device limit L <= 32
        # with L = 32 < 2^8 the list is not exhaustive: compare against the oracle's L = 32 list
        u, cw, pm = orc.scl(2.0 * y / 0.81, code.info_set, 16, 32)
        assert np.array_equal(np.asarray(top.words), cw[0])


def test_scl_rejects_non_polar():                                       # :125-128
    with pytest.raises(ValueError):
        scl_decode(np.zeros(8), codes.build_rm_code(3, 1), 2)


# --- hop (test_decoders.py:194-336) -------------------------------------------

def test_wsd_step_no_hop_from_exact_center(ca64, ca64_r2):              # :217-224
    rng = np.random.default_rng(10)
    cw = codes.encode(ca64, rand_msg(rng, 16))
    new, improved = wsd_step(modulate(cw), cw, modulate(cw), ca64_r2, m=10)
    assert not improved and new == cw


def test_wsd_step_full_sphere_reaches_ml_in_one_hop():                  # :227-236
    rng = np.random.default_rng(11)
    code = codes.build_ca_polar_code(32, 8)
    sph = full_sphere(code)
    for _ in range(15):
        y = modulate(codes.encode(code, rand_msg(rng, 8))) + 0.7 * rng.normal(size=32)
        anchor = codes.encode(code, rand_msg(rng, 8))
        new, _ = wsd_step(y, anchor, modulate(anchor), sph, m=sph.nonzero_size)
        assert new == ml_decode(y, code)


def test_trajectory_monotone_and_bounded(ca64, ca64_r2):               # :254-266
    rng = np.random.default_rng(13)
    params = WsdParams(radius_index=2, filter_size=12, max_iterations=4)
    for _ in range(30):
        y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + 0.9 * rng.normal(size=64)
        tr = wsd_trajectory(y, codes.encode(ca64, rand_msg(rng, 16)), ca64_r2, params)
        assert all(b < a for a, b in zip(tr.squared_eds, tr.squared_eds[1:]))
        assert len(tr.centers) == len(tr.squared_eds) and tr.iterations_used <= 4


def test_trajectory_with_full_sphere_converges_in_one_hop():            # :269-280
    rng = np.random.default_rng(14)
    code = codes.build_ca_polar_code(32, 8)
    sph = full_sphere(code)
    params = WsdParams(radius_index=sph.radius_index, filter_size=sph.nonzero_size, max_iterations=4)
    for _ in range(10):
        y = modulate(codes.encode(code, rand_msg(rng, 8))) + 0.8 * rng.normal(size=32)
        tr = wsd_trajectory(y, codes.encode(code, rand_msg(rng, 8)), sph, params)
        assert tr.centers[-1] == ml_decode(y, code) and len(tr.centers) <= 2


def test_mp_wsd_single_path_equals_trajectory(ca64, ca64_r2):           # :283-294
    rng = np.random.default_rng(15)
    params = WsdParams(radius_index=2, max_iterations=4, num_paths=1)
    y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + rng.normal(size=64)
    anchor = codes.encode(ca64, rand_msg(rng, 16))
    res = mp_wsd(y, CandidateList([(anchor, 0.0)]), ca64_r2, params)
    tr = wsd_trajectory(y, anchor, ca64_r2, params)
    assert res.best_codeword == tr.centers[-1] and res.squared_ed == tr.squared_eds[-1]


def test_mp_wsd_duplicate_anchors_match_single(ca64, ca64_r2):          # :297-308
    rng = np.random.default_rng(16)
    y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + rng.normal(size=64)
    a = codes.encode(ca64, rand_msg(rng, 16))
    one = mp_wsd(y, CandidateList([(a, 0.0)]), ca64_r2, WsdParams(radius_index=2, num_paths=1))
    four = mp_wsd(y, CandidateList([(a, 0.0)] * 4), ca64_r2, WsdParams(radius_index=2, num_paths=4))
    assert one.best_codeword == four.best_codeword and one.squared_ed == four.squared_ed


def test_mp_wsd_empty_list_rejected(ca64):                              # :311-315
    with pytest.raises(ValueError):
        mp_wsd(np.zeros(64), CandidateList([]), enumerate_sphere(ca64, 1), WsdParams(radius_index=1))


def test_mp_wsd_never_worse_than_best_anchor(ca64, ca64_r2):            # :318-329
    rng = np.random.default_rng(17)
    params = WsdParams(radius_index=2, num_paths=4, max_iterations=4)
    for _ in range(20):
        y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + rng.normal(size=64)
        anchors = [(codes.encode(ca64, rand_msg(rng, 16)), float(i)) for i in range(4)]
        res = mp_wsd(y, CandidateList(anchors), ca64_r2, params)
        assert res.squared_ed <= min(sqd(y, cw) for cw, _ in anchors)
        assert res.squared_ed == sqd(y, res.best_codeword)


def test_gain_argmax_equals_exact_ed_argmin(ca64, ca64_r2):             # :239-251, criterion 5
    """One GPU hop from a random centre picks the exact-ED argmin member."""
    rng = np.random.default_rng(12)
    members = np.asarray(ca64_r2.member_words)
    for _ in range(100):
        y = rng.normal(size=64)
        centre = codes.encode(ca64, rand_msg(rng, 16))
        eds = [sqd(y, BitVector(64, np.asarray(centre.words) ^ members[i])) for i in range(1, ca64_r2.size)]
        best = int(np.argmin(eds)) + 1
        new, improved = wsd_step(y, centre, modulate(centre), ca64_r2, m=10)
        if eds[best - 1] < sqd(y, centre):
            assert improved and new == BitVector(64, np.asarray(centre.words) ^ members[best])
        else:
            assert not improved


def test_default_filter_size_formula():                                 # :332-335
    assert default_filter_size(538) == 11 and default_filter_size(100) == 10
    assert default_filter_size(10000) == 200


# --- two-stage (test_decoders.py:341-412, criteria 3-4) -------------------------

def test_two_stage_noiseless_terminates_at_stage_one(ca64, ca64_r2):    # :341-352
    rng = np.random.default_rng(18)
    msg = rand_msg(rng, 16)
    res = two_stage_decode(modulate(codes.encode(ca64, msg)), ca64, SclStage(4),
                           WsdParams(radius_index=2, num_paths=4), ca64_r2, sigma=0.5)
    assert res.stage == "stage1_crc_pass" and res.best_message == msg
    assert res.traces == [] and res.counters.gain_additions == 0 and res.squared_ed == 0.0


def test_two_stage_always_on_runs_search_every_time(ca64, ca64_r2):     # :355-365
    rng = np.random.default_rng(19)
    params = WsdParams(radius_index=2, num_paths=4, activation_mode="always_on")
    for _ in range(5):
        y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + 0.3 * rng.normal(size=64)
        res = two_stage_decode(y, ca64, SclStage(4), params, ca64_r2, sigma=0.3)
        assert res.stage == "mp_wsd" and len(res.traces) == 4


def test_two_stage_crc_gated_needs_crc_code():                          # :368-373
    code = codes.build_polar_code(64, 16)
    with pytest.raises(ValueError, match="crc"):
        two_stage_decode(np.zeros(64), code, SclStage(4), WsdParams(radius_index=1),
                         enumerate_sphere(code, 1))


def test_two_stage_anchors_live_in_the_crc_subcode(ca64, ca64_r2):      # :389-399
    rng = np.random.default_rng(21)
    params = WsdParams(radius_index=2, num_paths=4, activation_mode="always_on")
    y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + 1.2 * rng.normal(size=64)
    res = two_stage_decode(y, ca64, SclStage(4), params, ca64_r2, sigma=1.2)
    for tr in res.traces:
        v = codes.precoded_of_codeword(ca64, tr.centers[0])
        assert codes.crc_valid_bits(v.bits(), ca64.crc)


def test_two_stage_is_deterministic(ca64, ca64_r2):                    # :402-412
    rng = np.random.default_rng(22)
    y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + rng.normal(size=64)
    p = WsdParams(radius_index=2, num_paths=4)
    a = two_stage_decode(y, ca64, SclStage(4), p, ca64_r2)
    b = two_stage_decode(y, ca64, SclStage(4), p, ca64_r2)
    assert a.best_codeword == b.best_codeword and a.squared_ed == b.squared_ed and a.stage == b.stage


def test_criterion3_full_radius_search_equals_ml(ca64):                 # criterion 3 (test_acceptance.py:96-122)
    sph = full_sphere(ca64)
    assert sph.size == 1 << 16
    dec = DeviceDecoder(ca64, sph)
    rng = np.random.default_rng(2024)
    F = 300
    msgs = rng.integers(0, 2, (F, 16), dtype=np.uint8)
    cw = codes.encode_batch(ca64, msgs)
    y = (modulate_words(cw, 64) + 0.74 * rng.normal(size=(F, 64))).astype(np.float32)
    o = dec.two_stage_batch(y, 0.74, 4, 4, 4, "always_on")
    from paper_2602_08501_b200.decoders import words32_to_64
    best = words32_to_64(o["best"].cpu().numpy().view(np.uint32), 64)
    for f in range(F):
        assert np.array_equal(best[f], np.asarray(ml_decode(y[f].astype(np.float64), ca64).words))


def test_criterion4_monotone_refinement(ca64, ca64_r2):                 # criterion 4 (:125-149)
    rng = np.random.default_rng(31337)
    params = WsdParams(radius_index=2, max_iterations=4, num_paths=4, activation_mode="always_on")
    for _ in range(40):
        y = modulate(codes.encode(ca64, rand_msg(rng, 16))) + 1.05 * rng.normal(size=64)
        res = two_stage_decode(y, ca64, SclStage(4), params, ca64_r2, sigma=1.05)
        for tr in res.traces:
            assert all(b < a for a, b in zip(tr.squared_eds, tr.squared_eds[1:]))
        assert res.squared_ed <= min(tr.squared_eds[0] for tr in res.traces)


# --- edge cases -----------------------------------------------------------------

def test_empty_and_ragged_batches(ca64, ca64_r2):
    dec = DeviceDecoder(ca64, ca64_r2)
    o = dec.two_stage_batch(np.zeros((0, 64), np.float32), 1.0, 4, 4, 4, "always_on")
    assert o["best"].shape[0] == 0
    rng = np.random.default_rng(7)
    for F in (1, 3, 31, 33, 257):
        y = (1.0 + rng.normal(size=(F, 64))).astype(np.float32)
        r = orc.two_stage_batch(y, ca64, ca64_r2, 4, 4, 4, True, 1.0, nthreads=4)
        o = dec.two_stage_batch(y, 1.0, 4, 4, 4, "crc_gated")
        from paper_2602_08501_b200.decoders import words32_to_64
        best = words32_to_64(o["best"].cpu().numpy().view(np.uint32), 64)
        np.testing.assert_array_equal(best, r["best"])
        np.testing.assert_array_equal(o["stage"].cpu().numpy(), r["stage"])


@pytest.mark.parametrize("L,A,T", [(4, 8, 4), (2, 2, 1), (8, 3, 2), (1, 1, 4)])
def test_list_and_anchor_count_combinations(ca64, ca64_r2, L, A, T):
    """A > list length, T = 1, L = 1: same anchors, iterations and codewords as the oracle."""
    rng = np.random.default_rng(L * 100 + A * 10 + T)
    F = 200
    msgs = rng.integers(0, 2, (F, 16), dtype=np.uint8)
    y = (modulate_words(codes.encode_batch(ca64, msgs), 64) + 1.0 * rng.normal(size=(F, 64))).astype(np.float32)
    dec = DeviceDecoder(ca64, ca64_r2)
    o = dec.two_stage_batch(y, 1.0, L, A, T, "always_on")
    r = orc.two_stage_batch(y, ca64, ca64_r2, L, A, T, False, 1.0, nthreads=4)
    from paper_2602_08501_b200.decoders import words32_to_64
    np.testing.assert_array_equal(words32_to_64(o["best"].cpu().numpy().view(np.uint32), 64), r["best"])
    np.testing.assert_array_equal(o["iters"].cpu().numpy(), r["iters"])


def test_empty_sphere_means_one_nonimproving_scan(ca64):
    """radius 0: only the zero codeword; every anchor is scanned once (decoders.py:371-373, 441-451)."""
    sph = enumerate_sphere(ca64, 0)
    assert sph.nonzero_size == 0
    rng = np.random.default_rng(3)
    y = (1.0 + rng.normal(size=(50, 64))).astype(np.float32)
    dec = DeviceDecoder(ca64, sph)
    o = dec.two_stage_batch(y, 1.0, 4, 4, 4, "always_on")
    it = o["iters"].cpu().numpy()
    assert set(np.unique(it).tolist()) <= {0, 1}
    r = orc.two_stage_batch(y, ca64, sph, 4, 4, 4, False, 1.0)
    np.testing.assert_array_equal(it, r["iters"])
