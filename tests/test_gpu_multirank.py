"""bench.py's own rank code at world size 2: each rank decodes its
block-aligned frame range on the GPU and the counters are all-reduced; the
totals must equal ONE process decoding the union of the ranks' frames in a
single two_stage_batch call (simharness.py:318-330 is the
reference's parallel driver).  Both ranks share the one visible GPU and reduce
over gloo: their decodes are independent, nothing waits across ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

F = 8192


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import bench
    from paper_2602_08501_b200 import configs
    args = bench._parse(["--gpus", str(world), "--frames", str(F), "--steps", "2", "--warmup", "3",
                         "--no-e2e", "--no-cpu"])
    cfg = configs.CONFIGS[args.config]
    code = cfg.code()
    sph = configs.build_sphere_for(cfg, code)
    line = bench.run_ours(args, cfg, code, sph, cfg.sigma(code=code), backend="gloo", device_index=0)
    if rank == 0:
        q.put(line)


def test_bench_two_ranks_equal_one_decode_of_the_union():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    line = q.get(timeout=900)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert line["n_gpus"] == world
    assert line["gpu_launches"] == world * 2 * 5

    from paper_2602_08501_b200 import channel, configs, shard
    from paper_2602_08501_b200.decoders import DeviceDecoder, words64_to_32
    cfg = configs.CONFIGS["cfg4"]
    code = cfg.code()
    sph = configs.build_sphere_for(cfg, code)
    sigma = cfg.sigma(code=code)
    ys, txs = [], []
    for r in range(world):          # the frames bench.py gives rank r: two batches of F
        sh = shard.shard_for(r, world, 2 * F)
        _, tx, y = channel.bulk_inputs(code, 2026, 0, sh.first, sh.count, sigma)
        ys.append(y)
        txs.append(words64_to_32(tx, code.n))
    y = np.concatenate(ys)
    tx = np.concatenate(txs)
    dec = DeviceDecoder(code, sph)
    ctr = torch.zeros(8, dtype=torch.int64, device="cuda")
    dec.two_stage_batch(y, sigma, cfg.list_size, cfg.num_paths, cfg.max_iterations, cfg.activation_mode,
                        tx_words=tx, counters=ctr)
    assert line["counters"] == shard.counters_dict(ctr.cpu().numpy())
    assert line["counters"]["frames"] == world * 2 * F
