"""Full-size checks of the cfg4 throughput workload (one bench step of 131,072
frames, BASELINE config 4) through size-independent properties, plus a larger
oracle-parity sample than test_gpu_parity.

Properties at full size (reference semantics, decoders.py:420-514):
* every decoded codeword is the encoding of the decoded message (CA subcode);
* replaying each trajectory's accepted hops from its anchor gives strictly
  decreasing canonical EDs, `iterations_used` = min(T, accepted + 1), and the
  minimum-ED trajectory (ties -> lowest anchor) ends at the decoded codeword
  with the reported float64 ED;
* a trajectory that stopped before T has no improving pattern left (checked
  against all of P on a sample of frames);
* stage-2 activation is forced on every frame and no frame is uncertified.
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_08501_b200 import channel, configs
from paper_2602_08501_b200._native import FLAG_TIE_FINAL as TIE_FINAL, FLAG_UNRESOLVED as UNRESOLVED
from paper_2602_08501_b200.bits import unpack_bits
from paper_2602_08501_b200.codes import encode_batch
from paper_2602_08501_b200.decoders import DeviceDecoder, words32_to_64
from tests.helpers import code_and_sphere

pytestmark = pytest.mark.gpu

F_FULL = 1 << 17


def _np(t):
    return t.cpu().numpy()


def _ed(y, words, n):
    """canonical float64 squared distance of y to the BPSK image of codewords"""
    x = 1.0 - 2.0 * unpack_bits(words, n).astype(np.float64)
    return ((y.astype(np.float64) - x) ** 2).sum(axis=-1)


@pytest.fixture(scope="module")
def cfg4_full():
    cfg = configs.CONFIGS["cfg4"]
    code, sph = code_and_sphere(cfg)
    sigma = cfg.sigma(code=code)
    msgs, tx, y = channel.bulk_inputs(code, 7, 0, 0, F_FULL, sigma)
    dec = DeviceDecoder(code, sph)
    o = dec.two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations, cfg.activation_mode,
                            want_hops=True, want_anchors=True)
    out = {k: _np(v) for k, v in o.items()}
    return cfg, code, sph, y, out


def test_cfg4_full_step_codewords_are_encoded_messages(cfg4_full):
    cfg, code, sph, y, o = cfg4_full
    n = code.n
    best = words32_to_64(o["best"].view(np.uint32), n)
    msg = o["best_msg"].view(np.uint64)
    bits = ((msg[:, None] >> np.arange(code.k, dtype=np.uint64)) & np.uint64(1)).astype(np.uint8)
    np.testing.assert_array_equal(encode_batch(code, bits), best)
    assert (o["stage"] == 1).all()                        # stage 2 forced (always_on)
    assert not (o["flags"] & UNRESOLVED).any()
    # final near-ties (two trajectories' EDs within 1e-5 relative) are reported, not errors
    assert (o["flags"] & TIE_FINAL).astype(bool).mean() < 0.05
    ctr = o["counters"]
    assert ctr[0] == F_FULL and ctr[2] == F_FULL           # frames, stage-2 activations
    assert ctr[3] == o["iters"].sum()                      # sum of iterations_used
    assert ctr[4] == o["iters"].sum() * sph.nonzero_size   # pattern-metric evaluations
    assert ctr[6] == 0                                     # uncertified


def test_cfg4_full_step_trajectories_replay(cfg4_full):
    cfg, code, sph, y, o = cfg4_full
    n, T, A = code.n, cfg.max_iterations, cfg.num_paths
    P = sph.patterns()
    rng = np.random.default_rng(0)
    fr = np.sort(rng.choice(F_FULL, 8192, replace=False))
    anchors = words32_to_64(o["anchors"][fr].view(np.uint32).reshape(len(fr) * A, -1), n).reshape(len(fr), A, -1)
    hops = o["hops"][fr]
    iters = o["iters"][fr]
    yy = y[fr]
    cur = anchors.copy()
    ed = _ed(yy[:, None, :], cur, n)
    accepted = np.zeros((len(fr), A), dtype=np.int64)
    done = np.zeros((len(fr), A), dtype=bool)
    for h in range(T):
        hp = hops[:, :, h]
        take = hp >= 1
        assert not (take & done).any(), "accepted hop after a non-improving scan"
        nxt = cur.copy()
        nxt[take] ^= P[hp[take] - 1]
        ned = _ed(yy[:, None, :], nxt, n)
        assert (ned[take] < ed[take]).all(), "accepted hop does not lower the canonical ED"
        cur, ed = np.where(take[..., None], nxt, cur), np.where(take, ned, ed)
        accepted += take
        done |= ~take
    np.testing.assert_array_equal(iters, np.minimum(T, accepted + 1))
    pick = np.argmin(ed, axis=1)                          # ties -> lowest anchor
    best = words32_to_64(o["best"][fr].view(np.uint32), n)
    ed_sorted = np.sort(ed, axis=1)
    exact_tie = (ed_sorted[:, 1] - ed_sorted[:, 0]) <= 1e-12 * ed_sorted[:, 0]   # summation-order ties only
    diff = (cur[np.arange(len(fr)), pick] != best).any(axis=1)
    assert not (diff & ~exact_tie).any()
    np.testing.assert_allclose(o["best_ed"][fr], ed[np.arange(len(fr)), pick], rtol=1e-12)


def test_cfg4_full_step_stopped_trajectories_are_local_minima(cfg4_full):
    cfg, code, sph, y, o = cfg4_full
    n, T = code.n, cfg.max_iterations
    Pb = unpack_bits(sph.patterns(), n).astype(np.float64)          # [|P|, n]
    best = words32_to_64(o["best"].view(np.uint32), n)
    # frames whose winning trajectory stopped on a non-improving scan
    hops = o["hops"]
    ed_pick = o["best_ed"]
    rng = np.random.default_rng(1)
    cand = rng.choice(F_FULL, 256, replace=False)
    x = 1.0 - 2.0 * unpack_bits(best[cand], n).astype(np.float64)
    t = x * y[cand].astype(np.float64)                               # x_i y_i
    S = t @ Pb.T                                                     # S_p; dED = 4 S_p
    it = o["iters"][cand]
    stopped = (it < T).all(axis=1)                                   # every anchor stopped early
    assert stopped.sum() > 100
    assert (S[stopped].min(axis=1) >= -1e-9 * ed_pick[cand][stopped]).all()


def test_cfg4_oracle_parity_larger_sample():
    cfg = configs.CONFIGS["cfg4"]
    code, sph = code_and_sphere(cfg)
    sigma = cfg.sigma(code=code)
    F = 640
    _, _, y = channel.bulk_inputs(code, 29, 0, 0, F, sigma)
    o = DeviceDecoder(code, sph).two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                                                 cfg.activation_mode)
    r = orc.two_stage_batch(y, code, sph, cfg.list_size, cfg.num_paths, cfg.max_iterations, False, sigma,
                            nthreads=os.cpu_count() or 1)
    best = words32_to_64(_np(o["best"]).view(np.uint32), code.n)
    flags = _np(o["flags"])
    mism = np.flatnonzero((best != r["best"]).any(axis=1))
    risky = np.flatnonzero(flags & (UNRESOLVED | TIE_FINAL))
    assert set(mism.tolist()) <= set(risky.tolist()), f"uncertified mismatches {mism}"
    ok = np.setdiff1d(np.arange(F), risky)
    np.testing.assert_array_equal(_np(o["iters"])[ok], r["iters"][ok])
