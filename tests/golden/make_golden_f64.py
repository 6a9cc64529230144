"""Golden vectors for FLOAT64 received words, produced by running the
REFERENCE (feclab) in this container.

    python tests/golden/make_golden_f64.py

The reference coerces y to float64 and decodes those values
(decoders.py:411, 466, 538); these fixtures keep the harness's float64
received words un-rounded (simharness.py:295-301), so they pin the drop-in's
float64 path (mpw_two_stage_batch_f64 / mpw_mpwsd_batch_f64).  Also written:
`wsd_step` with a real-valued x_center (decoders.py:401-417: the step is
scored on y * x_center) and `wsd_trajectory` traces.  The reference is
imported read-only and never at test time.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import ref_code, ref_sphere  # noqa: E402  (sets sys.path for feclab and the package)

from feclab.binlin import BitVector  # noqa: E402
from feclab.decoders import SclStage, WsdParams, two_stage_decode, wsd_step, wsd_trajectory  # noqa: E402

from paper_2602_08501_b200 import channel, configs  # noqa: E402


def gen_two_stage_f64(name, frames, mode=None, ebno=None, seed=3):
    cfg = configs.CONFIGS[name]
    code = ref_code(name)
    sph = ref_sphere(name, code, configs.build_sphere_for(cfg, cfg.code()))
    mode = mode or cfg.activation_mode
    e = cfg.ebno_db[0] if ebno is None else ebno
    sigma = channel.ebno_to_sigma(e, code.k / code.n)
    msgs, cw, y = channel.trial_inputs(code, seed, 0, range(frames), sigma)
    params = WsdParams(radius_index=sph.radius_index, max_iterations=cfg.max_iterations,
                       num_paths=cfg.num_paths, activation_mode=mode)
    A, W = cfg.num_paths, cw.shape[1]
    out = dict(y64=y, tx=cw, sigma=np.float64(sigma), stage=np.zeros(frames, np.uint8),
               best=np.zeros((frames, W), np.uint64), squared_ed=np.zeros(frames),
               iters=np.zeros((frames, A), np.int32), n_anchor=np.zeros(frames, np.int32),
               list_size=np.int32(cfg.list_size), num_paths=np.int32(A),
               max_iterations=np.int32(cfg.max_iterations), gated=np.int32(mode == "crc_gated"))
    t0 = time.time()
    for f in range(frames):
        r = two_stage_decode(y[f], code, SclStage(cfg.list_size), params, sph, sigma=sigma)
        out["stage"][f] = 0 if r.stage == "stage1_crc_pass" else 1
        out["best"][f] = r.best_codeword.words
        out["squared_ed"][f] = r.squared_ed
        for k, tr in enumerate(r.traces):
            out["iters"][f, k] = tr.iterations_used
        out["n_anchor"][f] = len(r.traces)
    # frames whose decode differs from the decode of float32(y): the cases the float64 path exists for
    y32 = y.astype(np.float32).astype(np.float64)
    diff = 0
    for f in range(min(frames, 64)):
        r = two_stage_decode(y32[f], code, SclStage(cfg.list_size), params, sph, sigma=sigma)
        diff += int(np.any(np.asarray(r.best_codeword.words) != out["best"][f]))
    tag = f"{name}_{mode}_{str(e).replace('.', 'p')}dB"
    np.savez_compressed(os.path.join(HERE, f"f64_two_stage_{tag}.npz"), **out)
    print(f"f64 {tag}: {frames} frames, p_act={out['stage'].mean():.3f}, "
          f"{diff} of {min(frames, 64)} codewords differ from the float32-rounded decode, {time.time() - t0:.1f}s")


def gen_wsd_api(name="cfg1", cases=48, seed=5):
    """wsd_step with real-valued x_center and wsd_trajectory on float64 y."""
    cfg = configs.CONFIGS[name]
    code = ref_code(name)
    sph = ref_sphere(name, code, configs.build_sphere_for(cfg, cfg.code()))
    n = code.n
    sigma = cfg.sigma(code=code)
    msgs, cw, y = channel.trial_inputs(code, seed, 0, range(cases), sigma)
    rng = np.random.default_rng(seed)
    W = cw.shape[1]
    T = cfg.max_iterations
    out = dict(y64=y, centers=np.zeros((cases, W), np.uint64), x_center=np.zeros((cases, n)),
               step_words=np.zeros((cases, W), np.uint64), step_improved=np.zeros(cases, np.uint8),
               traj_iters=np.zeros(cases, np.int32), traj_final=np.zeros((cases, W), np.uint64),
               traj_eds=np.full((cases, T + 1), np.nan), m=np.int32(4), max_iterations=np.int32(T))
    params = WsdParams(radius_index=sph.radius_index, max_iterations=T, num_paths=1)
    for f in range(cases):
        # a codeword near the transmitted one (a few hops away), and a real-valued x_center
        c = BitVector(n, cw[f] ^ sph.member_words[1 + rng.integers(sph.nonzero_size)])
        xc = (1.0 - 2.0 * c.bits().astype(np.float64)) * rng.uniform(0.25, 2.0, n)
        if f % 4 == 0:
            xc = 1.0 - 2.0 * c.bits().astype(np.float64)     # the ordinary ±1 case
        words, improved = wsd_step(y[f], c, xc, sph, 4)
        out["centers"][f] = c.words
        out["x_center"][f] = xc
        out["step_words"][f] = words.words
        out["step_improved"][f] = int(improved)
        tr = wsd_trajectory(y[f], c, sph, params)
        out["traj_iters"][f] = tr.iterations_used
        out["traj_final"][f] = tr.centers[-1].words
        out["traj_eds"][f, :len(tr.squared_eds)] = tr.squared_eds
    np.savez_compressed(os.path.join(HERE, f"f64_wsd_api_{name}.npz"), **out)
    print(f"f64_wsd_api_{name}: {cases} cases, {int(out['step_improved'].sum())} improving steps")


def gen_wsd_ties(name="cfg3", cases=64, seed=11):
    """Adversarial float64 inputs for wsd_step: the two best hop candidates
    p1, p2 differ by a tiny exact gap (|gap| ~ 1e-9, far above float64
    rounding, far below the fp32 rounding of y), so the decision depends on
    the float64 values; about half of the cases decode differently after
    rounding y to float32."""
    cfg = configs.CONFIGS[name]
    code = ref_code(name)
    sph = ref_sphere(name, code, configs.build_sphere_for(cfg, cfg.code()))
    n = code.n
    members = np.asarray(sph.member_words)
    rng = np.random.default_rng(seed)
    W = members.shape[1]
    bits = lambda w: np.unpackbits(np.asarray(w, dtype="<u8").view(np.uint8), bitorder="little")[:n]
    out = dict(y64=np.zeros((cases, n)), centers=np.zeros((cases, W), np.uint64),
               step_words=np.zeros((cases, W), np.uint64), step_improved=np.zeros(cases, np.uint8),
               m=np.int32(sph.nonzero_size))
    flips = 0
    for f in range(cases):
        c = rng.integers(0, 2, n).astype(np.uint8) * 0       # centre: the zero codeword
        x = 1.0 - 2.0 * c
        p1, p2 = rng.choice(np.arange(1, sph.size), 2, replace=False)
        s1, s2 = bits(members[p1]).astype(bool), bits(members[p2]).astype(bool)
        y = rng.normal(1.0, 0.6, n)
        # make p1 and p2 strongly improving: negative y on their supports
        y[s1 | s2] = -np.abs(y[s1 | s2]) - 0.5
        # exact gap: S_p1 - S_p2 = gap with one coordinate of supp p1 \ supp p2
        only1 = np.flatnonzero(s1 & ~s2)
        gap = (1 if f % 2 else -1) * 1e-9
        i = only1[0]
        S1, S2 = float(np.sum(x[s1] * y[s1])), float(np.sum(x[s2] * y[s2]))
        y[i] += (S2 + gap - S1) / x[i]
        words, improved = wsd_step(y, BitVector(n, np.zeros(W, np.uint64)), x, sph, sph.nonzero_size)
        w32, _ = wsd_step(y.astype(np.float32).astype(np.float64), BitVector(n, np.zeros(W, np.uint64)), x, sph,
                          sph.nonzero_size)
        flips += int(np.any(np.asarray(w32.words) != np.asarray(words.words)))
        out["y64"][f] = y
        out["step_words"][f] = words.words
        out["step_improved"][f] = int(improved)
    np.savez_compressed(os.path.join(HERE, f"f64_wsd_ties_{name}.npz"), **out)
    print(f"f64_wsd_ties_{name}: {cases} cases, {flips} decide differently on float32(y)")


if __name__ == "__main__":
    gen_wsd_ties()
    gen_wsd_ties("cfg2", 32)
    gen_wsd_ties("cfg4", 16)
    gen_wsd_api()
    gen_two_stage_f64("cfg1", 400)
    gen_two_stage_f64("cfg1", 200, mode="always_on")
    gen_two_stage_f64("cfg3", 200, ebno=1.0)
    gen_two_stage_f64("cfg2", 60)
    gen_two_stage_f64("cfg4", 12)
