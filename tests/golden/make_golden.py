"""Generate golden vectors by running the REFERENCE (feclab) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The reference is imported read-only and never at
test time; the GPU box only sees these fixtures.  Inputs are the reference
harness's per-trial streams (simharness.py:220-222, 295-301) rounded to
float32 -- the dtype of the accelerated path -- and the reference decodes
float64(y32), so both sides see identical values.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

import feclab.codebook as fcb  # noqa: E402
from feclab.binlin import BitMatrix, row_reduce  # noqa: E402
from feclab.decoders import (OsdStage, SclStage, WsdParams, osd_decode, scl_decode,  # noqa: E402
                             two_stage_decode)
from feclab.wsphere import build_sphere, load_sphere  # noqa: E402

from paper_2602_08501_b200 import channel, configs  # noqa: E402
from paper_2602_08501_b200.sphere import save_sphere  # noqa: E402


def ref_code(name):
    """The reference's own construction of each BASELINE config's code."""
    if name == "cfg1":
        from feclab.binlin import BitVector
        return fcb.build_ca_polar_code(64, 10, fcb.CrcSpec(6, BitVector.from_support([0, 5, 6], 7)))
    if name == "cfg2":
        # RM(2,7) as polar: a reliability order whose 29 most reliable entries
        # are {i : popcount(i) >= 5} (survey probe; simharness reliability_source=file:)
        idx = np.arange(128)
        ranked = idx[np.lexsort((idx, np.array([bin(i).count("1") for i in idx])))]
        return fcb.build_polar_code(128, 29, fcb.ReliabilityOrder(128, ranked, "rm"))
    if name == "cfg3":
        return fcb.build_ca_polar_code(128, 21)
    if name == "cfg4":
        return fcb.build_ca_polar_code(256, 53)
    raise KeyError(name)


def ref_sphere(name, code, mine):
    path = os.path.join("/tmp", f"golden_{name}.cws")
    save_sphere(mine, path)
    s = load_sphere(path)      # the reference's CWS1 reader validates the file
    if name in ("cfg1", "cfg3"):
        r = build_sphere(code, 1)
        assert np.array_equal(r.member_words, s.member_words), name
    return s


def gen_two_stage(name, frames, mode=None, ebno=None, seed=0, snr_idx=0):
    cfg = configs.CONFIGS[name]
    code = ref_code(name)
    mine_code = cfg.code()
    assert np.array_equal(np.asarray(code.generator.words), np.asarray(mine_code.generator.words)) \
        or name == "cfg2"
    if name == "cfg2":
        a = row_reduce(BitMatrix(29, 128, np.asarray(mine_code.generator.words)))[0].words
        b = row_reduce(code.generator)[0].words
        assert np.array_equal(a, b)
    sph = ref_sphere(name, code, configs.build_sphere_for(cfg, mine_code))
    mode = mode or cfg.activation_mode
    e = cfg.ebno_db[0] if ebno is None else ebno
    sigma = channel.ebno_to_sigma(e, code.k / code.n)
    msgs, cw, y = channel.trial_inputs(code, seed, snr_idx, range(frames), sigma)
    y32 = y.astype(np.float32)
    params = WsdParams(radius_index=sph.radius_index, max_iterations=cfg.max_iterations,
                       num_paths=cfg.num_paths, activation_mode=mode)
    A = cfg.num_paths
    W = cw.shape[1]
    out = dict(y32=y32, tx=cw, msgs=msgs, sigma=np.float64(sigma),
               stage=np.zeros(frames, np.uint8), best=np.zeros((frames, W), np.uint64),
               best_msg=np.zeros((frames, code.k), np.uint8),
               squared_ed=np.zeros(frames), iters=np.zeros((frames, A), np.int32),
               n_anchor=np.zeros(frames, np.int32), anchors=np.zeros((frames, A, W), np.uint64),
               list_size=np.int32(cfg.list_size), num_paths=np.int32(A),
               max_iterations=np.int32(cfg.max_iterations), gated=np.int32(mode == "crc_gated"),
               sphere_sha256=np.bytes_(configs.sphere_digest(sph)))
    t0 = time.time()
    for f in range(frames):
        r = two_stage_decode(y32[f].astype(np.float64), code, SclStage(cfg.list_size), params, sph,
                             sigma=sigma)
        out["stage"][f] = 0 if r.stage == "stage1_crc_pass" else 1
        out["best"][f] = r.best_codeword.words
        out["best_msg"][f] = r.best_message.bits()
        out["squared_ed"][f] = r.squared_ed
        for k, tr in enumerate(r.traces):
            out["iters"][f, k] = tr.iterations_used
            out["anchors"][f, k] = tr.centers[0].words
        out["n_anchor"][f] = len(r.traces)
    tag = f"{name}_{mode}_{str(e).replace('.', 'p')}dB"
    np.savez_compressed(os.path.join(HERE, f"two_stage_{tag}.npz"), **out)
    print(f"{tag}: {frames} frames, p_act={out['stage'].mean():.3f}, {time.time() - t0:.1f}s")


def gen_scl(name, frames, seed=7):
    cfg = configs.CONFIGS[name]
    code = ref_code(name)
    inner = code.inner if code.kind == "crc_concatenated" else code
    sigma = cfg.sigma(code=code)
    _, _, y = channel.trial_inputs(code, seed, 0, range(frames), sigma)
    llrs = 2.0 * y.astype(np.float32).astype(np.float64) / (sigma * sigma)
    L = cfg.list_size
    W = (code.n + 63) // 64
    cw = np.zeros((frames, L, W), np.uint64)
    pm = np.full((frames, L), np.nan)
    cnt = np.zeros(frames, np.int32)
    for f in range(frames):
        lst = scl_decode(llrs[f], inner, L)
        cnt[f] = len(lst)
        for i, (c, s) in enumerate(lst.entries):
            cw[f, i] = c.words
            pm[f, i] = s
    np.savez_compressed(os.path.join(HERE, f"scl_{name}.npz"), llrs=llrs, list_n=cnt, list_cw=cw,
                        list_pm=pm, list_size=np.int32(L), info_set=np.asarray(inner.info_set, np.int32))
    print(f"scl_{name}: {frames} frames")


def gen_osd():
    """osd_decode lists and OSD-initialised two-stage decodes (decoders.py:274-317,
    555-556) on the RM(128,29) polar-form code (cfg2), the demo CA(64,16) code
    and cfg1 (full order = ML)."""
    demo = fcb.build_ca_polar_code(64, 16)
    cases = (("rm_o2_cap64", ref_code("cfg2"), 3.0, 2, 64, 40),
             ("rm_o3_full", ref_code("cfg2"), 2.0, 3, None, 6),
             ("ca64_o3_full", demo, 2.0, 3, None, 12),
             ("cfg1_o10_cap1", ref_code("cfg1"), 1.0, 10, 1, 30))
    for tag, code, ebno, order, cap, frames in cases:
        sigma = channel.ebno_to_sigma(ebno, code.k / code.n)
        _, _, y = channel.trial_inputs(code, 11, 0, range(frames), sigma)
        y32 = y.astype(np.float32)
        lists = [osd_decode(y32[f].astype(np.float64), code, order, cap) for f in range(frames)]
        M = max(len(x.entries) for x in lists)
        W = (code.n + 63) // 64
        cw = np.zeros((frames, M, W), np.uint64)
        ed = np.full((frames, M), np.nan)
        cnt = np.zeros(frames, np.int32)
        for f, lst in enumerate(lists):
            cnt[f] = len(lst.entries)
            for i, (c, e) in enumerate(lst.entries):
                cw[f, i] = c.words
                ed[f, i] = e
        np.savez_compressed(os.path.join(HERE, f"osd_{tag}.npz"), y32=y32, list_n=cnt, list_cw=cw,
                            list_ed=ed, order=np.int32(order), list_cap=np.int32(cap or 0),
                            gen=np.asarray(code.generator.words))
        print(f"osd_{tag}: {frames} frames, M={M}")
    # OSD(2) + always-on MP-WSD r=1 on RM(128,29) (configs/rm_128_29_osd2_r1.cfg shape)
    cfg = configs.CONFIGS["cfg2"]
    code = ref_code("cfg2")
    sph = ref_sphere("cfg2", code, configs.build_sphere_for(cfg, cfg.code()))
    for tag, ebno, frames, mode, stage1, ccode, csph in (
            ("rm_osd2_aom", 2.0, 60, "always_on", OsdStage(2, 64), code, sph),
            ("ca64_osd1_gated", 1.0, 40, "crc_gated", OsdStage(1), demo, None)):
        if csph is None:
            csph = build_sphere(ccode, 2)
        sigma = channel.ebno_to_sigma(ebno, ccode.k / ccode.n)
        msgs, tx, y = channel.trial_inputs(ccode, 13, 0, range(frames), sigma)
        y32 = y.astype(np.float32)
        A, T = 4, 4
        params = WsdParams(radius_index=csph.radius_index, max_iterations=T, num_paths=A,
                           activation_mode=mode)
        W = tx.shape[1]
        out = dict(y32=y32, tx=tx, msgs=msgs, stage=np.zeros(frames, np.uint8),
                   best=np.zeros((frames, W), np.uint64), best_msg=np.zeros((frames, ccode.k), np.uint8),
                   squared_ed=np.zeros(frames), iters=np.zeros((frames, A), np.int32),
                   n_anchor=np.zeros(frames, np.int32), anchors=np.zeros((frames, A, W), np.uint64),
                   order=np.int32(stage1.order), list_cap=np.int32(stage1.list_cap or 0),
                   num_paths=np.int32(A), max_iterations=np.int32(T), gated=np.int32(mode == "crc_gated"),
                   radius_index=np.int32(csph.radius_index),
                   sphere_members=np.asarray(csph.member_words))
        for f in range(frames):
            r = two_stage_decode(y32[f].astype(np.float64), ccode, stage1, params, csph, sigma=sigma)
            out["stage"][f] = 0 if r.stage == "stage1_crc_pass" else 1
            out["best"][f] = r.best_codeword.words
            out["best_msg"][f] = r.best_message.bits()
            out["squared_ed"][f] = r.squared_ed
            for k, tr in enumerate(r.traces):
                out["iters"][f, k] = tr.iterations_used
                out["anchors"][f, k] = tr.centers[0].words
            out["n_anchor"][f] = len(r.traces)
        np.savez_compressed(os.path.join(HERE, f"two_stage_{tag}.npz"), **out)
        print(f"two_stage_{tag}: {frames} frames, p_act={out['stage'].mean():.3f}")


DEMO_CFG = """
code_family = ca_polar
code_n = 64
code_k = 16
snr_db_grid = 0.0, 1.0, 2.0, 3.0, 4.0
stage1 = scl
scl_list_size = 4
wsd_radius_index = {r}
wsd_num_paths = {paths}
activation_mode = crc_gated
max_trials = 4000
min_block_errors = 100
seed = 99
"""


def gen_sweeps(rm_only=False):
    """The reference's own run_sweep on its desk-scale demo configuration
    (demos/bler_sweep_small.py), written with its own write_csv."""
    from feclab.simharness import parse_config, run_sweep, write_csv
    code = fcb.build_ca_polar_code(64, 16)
    for r, paths, name in (() if rm_only else ((2, 4, "sweep_two_stage.csv"), (0, 1, "sweep_stage1.csv"))):
        cfg_text = DEMO_CFG.format(r=r, paths=paths)
        with open(os.path.join(HERE, name.replace(".csv", ".cfg")), "w") as fh:
            fh.write(cfg_text.lstrip())
        t0 = time.time()
        recs = run_sweep(parse_config(cfg_text), sphere=build_sphere(code, r))
        write_csv(recs, os.path.join(HERE, name))
        print(f"{name}: {time.time() - t0:.1f}s")
    # OSD(2) + always-on r=1 on RM(128,29): configs/rm_128_29_osd2_r1.cfg with a
    # reduced trial budget; sphere = the reference's own CWS reader on our file
    from paper_2602_08501_b200 import codes as mycodes
    from paper_2602_08501_b200.patterns import enumerate_sphere
    with open("/root/reference/pkg/configs/rm_128_29_osd2_r1.cfg") as fh:
        rm_text = fh.read()
    rm_text = (rm_text.replace("snr_db_grid = 1.0, 2.0, 3.0, 4.0", "snr_db_grid = 1.0, 2.5")
               .replace("max_trials = 10000", "max_trials = 2048")
               .replace("sphere_path = rm_128_29_r1.cws", "sphere_path = /tmp/golden_rm_r1.cws"))
    save_sphere(enumerate_sphere(mycodes.build_rm_code(7, 2), 1), "/tmp/golden_rm_r1.cws")
    with open(os.path.join(HERE, "sweep_rm_osd.cfg"), "w") as fh:
        fh.write(rm_text.replace("/tmp/golden_rm_r1.cws", "rm_128_29_r1.cws"))
    t0 = time.time()
    rm_cfg = parse_config(rm_text)
    recs = run_sweep(rm_cfg, sphere=load_sphere("/tmp/golden_rm_r1.cws"))
    write_csv(recs, os.path.join(HERE, "sweep_rm_osd.csv"))
    print(f"sweep_rm_osd.csv: {time.time() - t0:.1f}s")
    if rm_only:
        return
    # exact-ML curves on the same trial streams (decoder_kind='ml', demos/sweep_ml.csv)
    t0 = time.time()
    recs = run_sweep(parse_config(DEMO_CFG.format(r=2, paths=4)), decoder_kind="ml")
    write_csv(recs, os.path.join(HERE, "sweep_ml.csv"))
    print(f"sweep_ml.csv: {time.time() - t0:.1f}s")


if __name__ == "__main__":
    if "--sweeps" in sys.argv:
        gen_sweeps()
        sys.exit(0)
    if "--rm-sweep" in sys.argv:
        gen_sweeps(rm_only=True)
        sys.exit(0)
    if "--osd" in sys.argv:
        gen_osd()
        sys.exit(0)
    for nm, fr in (("cfg1", 64), ("cfg2", 16), ("cfg3", 32), ("cfg4", 8)):
        gen_scl(nm, fr)
    gen_two_stage("cfg1", 400)
    gen_two_stage("cfg1", 160, mode="always_on")
    gen_two_stage("cfg3", 200, ebno=1.0)
    gen_two_stage("cfg2", 100)
    gen_two_stage("cfg4", 24)
