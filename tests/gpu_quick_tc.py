"""Quick guarded check of the tensor-core hop against the oracle (dev script)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as orc
from paper_2602_08501_b200 import configs, channel
from paper_2602_08501_b200.decoders import DeviceDecoder, words32_to_64
import torch

for name, F in [("cfg1", 512), ("cfg3", 512), ("cfg2", 128), ("cfg4", 64)]:
    cfg = configs.CONFIGS[name]
    code = cfg.code(); sph = configs.build_sphere_for(cfg, code); sigma = cfg.sigma(code=code)
    _, tx, y = channel.bulk_inputs(code, 3, 0, 0, F, sigma)
    dec = DeviceDecoder(code, sph)
    res = {}
    for var in ["gather", "tensor", "tensor2"]:
        torch.cuda.synchronize(); t0 = time.time()
        o = dec.two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations, "always_on", variant=var)
        torch.cuda.synchronize(); dt = time.time() - t0
        res[var] = (words32_to_64(o["best"].cpu().numpy().view(np.uint32), code.n), o["iters"].cpu().numpy(), o["flags"].cpu().numpy(), dt)
    r = orc.two_stage_batch(y, code, sph, cfg.list_size, cfg.num_paths, cfg.max_iterations, False, sigma, nthreads=8)
    for var in ["gather", "tensor", "tensor2"]:
        b, it, fl, dt = res[var]
        mism = np.flatnonzero((b != r["best"]).any(1))
        unfl = [m for m in mism if fl[m] == 0]
        itm = np.flatnonzero((it != r["iters"]).any(1) & (fl == 0))
        print(f"{name} {var}: mism={len(mism)} unflagged={len(unfl)} iters_mism_unflagged={len(itm)} flagged={int((fl>0).sum())} {dt*1e3:.1f} ms", flush=True)
