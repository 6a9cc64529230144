"""cfg4 parity at scale: the bench workload's first F frames (bulk Philox
stream, seed 2026, float32 y) decoded on the GPU with every tensor hop
variant and by the CPU oracle (oracle/oracle.c, all host threads); reports
codeword and per-anchor iterations_used equality, the frames that carry the
TIE_FINAL / UNRESOLVED flags (the only frames allowed to differ), near-tie
reports and FER.  The oracle is the checker only.

    python tools/cfg4_oracle_subsample.py [--frames 8192] [--out profiles/r02_cfg4_oracle_subsample.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402  (checker only)
from paper_2602_08501_b200 import channel, configs  # noqa: E402
from paper_2602_08501_b200._native import FLAG_TIE_FINAL, FLAG_UNRESOLVED  # noqa: E402
from paper_2602_08501_b200.decoders import DeviceDecoder, words32_to_64, words64_to_32  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=8192)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--variants", default="tensor_i8a,tensor_i8,tensor,tensor2")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cfg4_oracle_subsample.json"))
    args = ap.parse_args()
    cfg = configs.CONFIGS[args.config]
    code = cfg.code()
    sph = configs.build_sphere_for(cfg, code)
    sigma = cfg.sigma(code=code)
    _, tx, y = channel.bulk_inputs(code, 2026, 0, 0, args.frames, sigma)
    A, T, L = cfg.num_paths, cfg.max_iterations, cfg.list_size
    gated = cfg.activation_mode == "crc_gated"
    threads = os.cpu_count() or 1
    t0 = time.time()
    ref = orc.two_stage_batch(y, code, sph, L, A, T, gated, sigma, nthreads=threads)
    oracle_s = time.time() - t0
    out = {"config": args.config, "frames": args.frames, "input": "bench.py workload: bulk Philox seed 2026, "
           "snr index 0, frames [0, F), float32 y", "oracle": {"seconds": oracle_s, "threads": threads,
           "errors": int((ref["best"] != tx).any(axis=1).sum())}, "variants": {}}
    dec = DeviceDecoder(code, sph)
    for v in args.variants.split(","):
        o = dec.two_stage_batch(y, sigma, L, A, T, cfg.activation_mode, variant=v,
                                tx_words=words64_to_32(tx, code.n))
        best = words32_to_64(o["best"].cpu().numpy().view(np.uint32), code.n)
        flags = o["flags"].cpu().numpy()
        iters = o["iters"].cpu().numpy()
        ctr = o["counters"].cpu().numpy()
        mism = np.flatnonzero((best != ref["best"]).any(axis=1))
        exempt = flags & (FLAG_TIE_FINAL | FLAG_UNRESOLVED) != 0
        it_mism = np.flatnonzero((iters != ref["iters"]).any(axis=1))
        out["variants"][v] = {
            "codeword_mismatches": int(mism.size),
            "codeword_mismatches_unflagged": int((~exempt[mism]).sum()),
            "iterations_used_mismatches": int(it_mism.size),
            "iterations_used_mismatches_unflagged": int((~exempt[it_mism]).sum()),
            "frames_flagged_tie_final": int(((flags & FLAG_TIE_FINAL) != 0).sum()),
            "frames_flagged_unresolved": int(((flags & FLAG_UNRESOLVED) != 0).sum()),
            "near_tie_frames_reported": int(ctr[5]),
            "gpu_errors": int(ctr[1]), "evals": int(ctr[4]),
        }
        print(v, json.dumps(out["variants"][v]), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out["oracle"]))


if __name__ == "__main__":
    main()
