"""BASELINE config 5: FER curves of the RM(2,7)-as-polar (always-on) and
polar(128,32)+CRC-11 (gated) setups at Eb/N0 0..4 dB, decoded on the GPU from
device-resident inputs (mpw_channel_batch), with the CPU oracle run on a
per-point subsample of the very same received words:

  * codewords of the subsample must match the oracle except on frames the
    kernel flags as uncertified / final near-tie;
  * the GPU FER over all frames must lie inside the oracle's Wilson 95 %
    interval from the subsample (simharness.py:208-217).

    python tools/fer_curve.py [--frames 1000000] [--oracle-frames 4000] [--out profiles/...]
    python -m torch.distributed.run --nproc-per-node 8 tools/fer_curve.py --frames 10000000

Under torchrun the trials of every point shard by range over the ranks
(sweep._Ranks: one all-reduce of the per-block statistics per round); rank 0
holds the first batch, runs the oracle subsample and writes the outputs.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402  (checker only)
from paper_2602_08501_b200 import configs, sweep  # noqa: E402
from paper_2602_08501_b200.decoders import words32_to_64  # noqa: E402

GRID = "0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0"


def setups(frames: int, rm_rank_path: str):
    rm = f"""
code_family = polar
code_n = 128
code_k = 29
reliability_source = file:{rm_rank_path}
snr_db_grid = {GRID}
stage1 = scl
scl_list_size = 8
wsd_radius_index = 1
wsd_max_iterations = 6
wsd_num_paths = 8
activation_mode = always_on
max_trials = {frames}
min_block_errors = {frames + 1}
seed = 2602
"""
    p128 = f"""
code_family = ca_polar
code_n = 128
code_k = 21
snr_db_grid = {GRID}
stage1 = scl
scl_list_size = 8
wsd_radius_index = 1
wsd_max_iterations = 8
wsd_num_paths = 8
activation_mode = crc_gated
max_trials = {frames}
min_block_errors = {frames + 1}
seed = 2603
"""
    return {"rm128_29_polar_always_on": (rm, "cfg2"), "polar128_32_crc11_gated": (p128, "cfg3")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=1_000_000)
    ap.add_argument("--oracle-frames", type=int, default=4000)
    ap.add_argument("--batch", type=int, default=1 << 18)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fer_curve"))
    args = ap.parse_args()
    dist, rank = sweep._init_ranks()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    idx = np.arange(128)
    ranking = idx[np.lexsort((idx, np.array([bin(i).count("1") for i in idx])))]
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as fh:
        fh.write("\n".join(str(int(v)) for v in ranking))
        rank_path = fh.name
    summary = {"note": "FER vs the oracle's Wilson 95% CI from its subsample: with 18 intervals about "
                       "one miss is expected by chance; the decoders themselves are compared exactly on "
                       "the subsample (gpu_errors_on_subsample == oracle_errors, codeword mismatches).",
               "frames_per_point": args.frames, "oracle_frames_per_point": args.oracle_frames,
               "input": "device counter-based Philox4x32-10 stream (mpw_channel_batch)",
               "ranks": 1 if dist is None else dist.get_world_size(), "runs": {}}
    for name, (text, cfgname) in setups(args.frames, rank_path).items():
        cfg = sweep.parse_config(text)
        code = sweep.build_code(cfg)
        sph = configs.build_sphere_for(configs.CONFIGS[cfgname], code)
        sub = {}

        def on_batch(snr_idx, t0, y, tx, o):
            if t0 != 0:
                return
            k = min(args.oracle_frames, y.shape[0])
            sub[snr_idx] = dict(y=y[:k].cpu().numpy(), tx=words32_to_64(tx[:k].cpu().numpy().view(np.uint32), code.n),
                                best=words32_to_64(o["best"][:k].cpu().numpy().view(np.uint32), code.n),
                                flags=o["flags"][:k].cpu().numpy())
        t0 = time.time()
        recs = sweep.run_sweep(cfg, sphere=sph, batch=args.batch, input_mode="device", on_batch=on_batch)
        gpu_s = time.time() - t0
        if rank:
            continue
        sweep.write_csv(recs, f"{args.out}_{name}.csv")
        points = []
        for i, r in enumerate(recs):
            s = sub[i]
            ores = orc.two_stage_batch(s["y"], code, sph, cfg.scl_list_size, cfg.wsd_num_paths,
                                       cfg.wsd_max_iterations, cfg.activation_mode == "crc_gated",
                                       sweep._sigma(cfg, r.snr_db), nthreads=os.cpu_count() or 1)
            mism = np.flatnonzero((ores["best"] != s["best"]).any(axis=1))
            risky = set(np.flatnonzero(s["flags"] & 12).tolist())
            o_err = int((ores["best"] != s["tx"]).any(axis=1).sum())
            g_err = int((s["best"] != s["tx"]).any(axis=1).sum())
            lo, hi = sweep.wilson_interval(o_err, len(s["y"]))
            points.append(dict(snr_db=r.snr_db, gpu_trials=r.trials, gpu_errors=r.block_errors, gpu_fer=r.bler,
                               p_act=r.activation_rate, avg_iters=r.avg_iterations,
                               oracle_frames=len(s["y"]), oracle_errors=o_err, oracle_ci=[lo, hi],
                               gpu_errors_on_subsample=g_err,
                               fer_in_oracle_ci=bool(lo <= r.bler <= hi),
                               subsample_codeword_mismatches=int(len(mism)),
                               mismatches_all_flagged=bool(set(mism.tolist()) <= risky),
                               near_tie_frames=r.near_tie_frames, uncertified_frames=r.uncertified_frames))
        summary["runs"][name] = dict(gpu_seconds=gpu_s, frames_per_second=len(recs) * args.frames / gpu_s,
                                     points=points)
        print(json.dumps({name: summary["runs"][name]}, indent=1), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    if rank:
        return
    with open(args.out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
