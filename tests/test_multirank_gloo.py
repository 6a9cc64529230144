"""World-size-2 gloo test of the N>1 path's host logic on CPU: block-aligned
frame shards of the block-keyed input stream, per-rank decoding and the single
counter all-reduce give the same totals as ONE decode of the whole contiguous
range in one call (the CPU oracle stands in for the per-GPU decoder here; the
GPU version, tests/test_gpu_multirank.py, runs bench.py's own rank code)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_08501_b200 import channel, configs, shard

TOTAL = 3 * channel.BLOCK + 512   # ragged last block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decode_counts(cfg, code, sph, sigma, first, count):
    from oracle import oracle as orc
    _, tx, y = channel.bulk_inputs(code, 5, 0, first, count, sigma)
    o = orc.two_stage_batch(y, code, sph, cfg.list_size, cfg.num_paths, cfg.max_iterations,
                            cfg.activation_mode == "crc_gated", sigma, nthreads=2)
    err = int((o["best"] != tx).any(axis=1).sum())
    act = int(o["stage"].sum())
    its = int(o["iters"].sum())
    return np.array([count, err, act, its, its * sph.nonzero_size, 0, 0, 0], np.int64)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.CONFIGS["cfg1"]
    code = cfg.code()
    sph = configs.build_sphere_for(cfg, code)
    sigma = cfg.sigma(code=code)
    sh = shard.split_range(TOTAL, rank, world)
    c = torch.from_numpy(_decode_counts(cfg, code, sph, sigma, sh.first, sh.count))
    shard.reduce_counters(c, dist)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    shard.reduce_max(t, dist)
    if rank == 0:
        q.put((c.numpy().tolist(), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_and_reduction_match_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = configs.CONFIGS["cfg1"]
    code = cfg.code()
    sph = configs.build_sphere_for(cfg, code)
    sigma = cfg.sigma(code=code)
    ref = _decode_counts(cfg, code, sph, sigma, 0, TOTAL)
    assert got == ref.tolist()
    assert tmax == 2.0


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_split_range_covers_exactly_once(world):
    total = 10 * channel.BLOCK + 17
    covered = []
    for r in range(world):
        sh = shard.split_range(total, r, world)
        assert sh.first % channel.BLOCK == 0
        covered.extend(range(sh.first, sh.first + sh.count))
    assert covered == list(range(total))


def test_shards_are_disjoint_and_block_aligned():
    s = [shard.shard_for(r, 4, 5000) for r in range(4)]
    for a, b in zip(s, s[1:]):
        assert a.first + a.count <= b.first
        assert b.first % channel.BLOCK == 0
