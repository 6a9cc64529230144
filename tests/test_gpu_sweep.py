"""The batched GPU sweep reproduces the reference's own run_sweep CSVs byte
for byte (golden CSVs made by tests/golden/make_golden.py --sweeps, which the
reference writes identically to its shipped demos/sweep_*.csv)."""
import os

import pytest

from paper_2602_08501_b200 import sweep

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["sweep_two_stage", "sweep_stage1"])
def test_gpu_sweep_csv_matches_reference_bytes(name, tmp_path):
    cfg = sweep.load_config(os.path.join(GOLDEN, name + ".cfg"))
    recs = sweep.run_sweep(cfg, batch=4096)
    out = tmp_path / (name + ".csv")
    sweep.write_csv(recs, out)
    with open(os.path.join(GOLDEN, name + ".csv"), "rb") as fh:
        want = fh.read()
    assert out.read_bytes() == want
    assert all(r.uncertified_frames == 0 for r in recs)


def test_gpu_ml_sweep_csv_matches_reference_bytes(tmp_path):
    """decoder_kind='ml' (reference mltruth) on the same streams: the GPU's
    full-codebook scan reproduces demos/sweep_ml.csv."""
    cfg = sweep.load_config(os.path.join(GOLDEN, "sweep_two_stage.cfg"))
    recs = sweep.run_sweep_ml(cfg, batch=4096)
    out = tmp_path / "ml.csv"
    sweep.write_csv(recs, out)
    with open(os.path.join(GOLDEN, "sweep_ml.csv"), "rb") as fh:
        assert out.read_bytes() == fh.read()


def test_gpu_rm_osd_sweep_csv_matches_reference_bytes(tmp_path):
    """configs/rm_128_29_osd2_r1.cfg (OSD(2) + always-on r=1 on RM(128,29)) with a
    reduced trial budget: the reference's own run_sweep CSV, byte for byte."""
    from paper_2602_08501_b200 import codes
    from paper_2602_08501_b200.patterns import enumerate_sphere_gpu
    cfg = sweep.load_config(os.path.join(GOLDEN, "sweep_rm_osd.cfg"))
    sph = enumerate_sphere_gpu(codes.build_rm_code(7, 2), 1)
    recs = sweep.run_sweep(cfg, sphere=sph, batch=4096)
    assert all(r.uncertified_frames == 0 for r in recs)
    out = tmp_path / "rm.csv"
    sweep.write_csv(recs, out)
    with open(os.path.join(GOLDEN, "sweep_rm_osd.csv"), "rb") as fh:
        assert out.read_bytes() == fh.read()


def _sweep_rank(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = sweep.load_config(os.path.join(GOLDEN, name + ".cfg"))
    recs = sweep.run_sweep(cfg, batch=1024)
    q.put((rank, [(r.trials, r.block_errors, r.activation_rate, r.ed_units_mean, r.avg_iterations)
                  for r in recs], recs if rank == 0 else None))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["sweep_two_stage", "sweep_stage1"])
def test_gpu_sweep_two_ranks_csv_matches_reference_bytes(name, tmp_path):
    """The trial range sharded over two ranks (block-aligned, one all-reduce
    of the block statistics per round): both ranks fold identical records and
    the CSV equals the reference's byte for byte.  The ranks share the one
    visible GPU (independent decodes) and reduce over gloo."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sweep_rank, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (summ, recs)) for r, summ, recs in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0][0] == got[1][0]
    out = tmp_path / (name + ".csv")
    sweep.write_csv(got[0][1], out)
    with open(os.path.join(GOLDEN, name + ".csv"), "rb") as fh:
        assert out.read_bytes() == fh.read()
