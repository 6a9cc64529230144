"""Equality at scale of the two int8 hops (exact decisions by two different
kernels): the asynchronous-row hop against the synchronous-round int8 screen on
the bench workload's frames [0, F): codewords, per-anchor iterations_used and
flags.  GPU only (the oracle subsample covers 8,192 of these frames).

    python tools/async_vs_sync.py [--frames 524288] [--out profiles/r02_async_vs_sync.json]
"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08501_b200 import channel, configs  # noqa: E402
from paper_2602_08501_b200.decoders import DeviceDecoder  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=524288)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "async_vs_sync.json"))
    a = ap.parse_args()
    cfg = configs.CONFIGS["cfg4"]
    code = cfg.code(); sph = configs.build_sphere_for(cfg, code); sigma = cfg.sigma(code=code)
    dec = DeviceDecoder(code, sph)
    args = (sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations, cfg.activation_mode)
    tot = dict(frames=0, codeword_mismatches=0, iterations_used_mismatches=0, flag_mismatches=0, flagged_async=0, flagged_sync=0,
               scans=0)
    t0 = time.time()
    for first in range(0, a.frames, a.batch):
        cnt = min(a.batch, a.frames - first)
        _, _, y = channel.bulk_inputs(code, 2026, 0, first, cnt, sigma)
        o1 = dec.two_stage_batch(y, *args, variant="tensor_i8a")
        o2 = dec.two_stage_batch(y, *args, variant="tensor_i8")
        b1, b2 = o1["best"].cpu().numpy(), o2["best"].cpu().numpy()
        i1, i2 = o1["iters"].cpu().numpy(), o2["iters"].cpu().numpy()
        f1, f2 = o1["flags"].cpu().numpy(), o2["flags"].cpu().numpy()
        tot["frames"] += cnt
        tot["codeword_mismatches"] += int((b1 != b2).any(axis=1).sum())
        tot["iterations_used_mismatches"] += int((i1 != i2).any(axis=1).sum())
        tot["flag_mismatches"] += int((f1 != f2).sum())
        tot["flagged_async"] += int((f1 != 0).sum())
        tot["flagged_sync"] += int((f2 != 0).sum())
        tot["scans"] += int(i1.sum())
    tot["seconds"] = time.time() - t0
    tot["input"] = "bench.py workload: bulk Philox seed 2026, snr index 0, float32 y"
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(tot, open(a.out, "w"), indent=1)
    print(json.dumps(tot))


if __name__ == "__main__":
    main()
