"""Small async-hop decode for compute-sanitizer runs (memcheck / racecheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_08501_b200 import channel, configs
from paper_2602_08501_b200.decoders import DeviceDecoder
cfg = configs.CONFIGS["cfg4"]
code = cfg.code(); sph = configs.build_sphere_for(cfg, code); sigma = cfg.sigma(code=code)
F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
_, _, y = channel.bulk_inputs(code, 31, 0, 0, F, sigma)
dec = DeviceDecoder(code, sph)
o = dec.two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations, cfg.activation_mode, variant="tensor_i8a")
print("iters sum", int(o["iters"].sum().item()), "flags", int((o["flags"] != 0).sum().item()))
