"""Batched Monte-Carlo sweep over the B200 path.

The reference's harness (/root/reference/pkg/src/feclab/simharness.py)
decodes one trial at a time from a thread pool; this one decodes batches of
trials on the GPU and folds the per-trial outcomes in trial order with the
reference's own rules, so the CSV is the reference's byte for byte:

* config files: strict `key = value`, unknown/duplicate keys rejected, same
  keys and `formula` convention (simharness.py:117-172);
* trial streams: message from Philox (seed, sid|1), noise from (seed, sid),
  sid = (snr_idx << 40) | (trial << 2)  (simharness.py:220-222, 295-301);
* stopping rule: trials are consumed in batches of 64 and the error target is
  checked between batches (simharness.py:318-330);
* records: Wilson 95 % interval (:208-217), activation rate, ED units from the
  reference's operation counts (complexity.py:47-57, decoders.py:375-389,
  :478), mean iterations per path, fixed CSV schema (:32-33, 365-376).

Both stage-1 kinds run on the device: CA-SCL and order-k OSD (csrc/osd.cuh).
Trial-stream inputs are decoded as the reference's float64 values (the
*_f64 entry points); device-stream inputs are float32.  Under torchrun the
trials shard by range over the ranks (_Ranks) with one all-reduce of the
per-block statistics per round:

    python -m torch.distributed.run --nproc-per-node 8 -m paper_2602_08501_b200.sweep \
        --config X.cfg --out X.csv
"""

from __future__ import annotations

import math
import os
import sys
from dataclasses import dataclass

import numpy as np

from . import codes
from .channel import ebno_to_sigma, trial_inputs

BATCH = 64
CSV_HEADER = ("code,stage1,wsd_r,wsd_m,wsd_J,L_init,snr_db,trials,errors,"
              "bler,bler_lo,bler_hi,p_act,ed_units,avg_iters,seed")


class ConfigError(ValueError):
    pass


@dataclass
class ExperimentConfig:
    code_family: str
    code_n: int
    code_k: int
    snr_db_grid: list
    stage1: str
    seed: int
    max_trials: int
    crc_degree: int = 11
    crc_polynomial: tuple = (0, 5, 9, 10, 11)
    reliability_source: str = "bundled_5g_table"
    snr_convention: str = "ebno"
    scl_list_size: int = 8
    osd_order: int = 2
    stage1_list_cap: int | None = None
    wsd_radius_index: int = 0
    wsd_filter_size: int | None = None
    wsd_max_iterations: int = 4
    wsd_num_paths: int = 4
    activation_mode: str = "crc_gated"
    min_block_errors: int = 100
    max_wall_seconds: float | None = None
    sphere_path: str | None = None

    def __post_init__(self):
        if not self.snr_db_grid:
            raise ConfigError("snr_db_grid must be nonempty")
        if any(b >= a for a, b in zip(self.snr_db_grid[1:], self.snr_db_grid)):
            raise ConfigError("snr_db_grid must be strictly ascending")
        if self.min_block_errors < 1:
            raise ConfigError("min_block_errors must be >= 1")
        if self.max_trials < 1 or self.max_trials > 2 ** 31:
            raise ConfigError("max_trials out of range")
        if self.code_family not in ("ca_polar", "polar", "rm"):
            raise ConfigError(f"unknown code_family {self.code_family!r}")
        if self.stage1 not in ("scl", "osd"):
            raise ConfigError(f"unknown stage1 {self.stage1!r}")
        if self.snr_convention not in ("ebno", "esno"):
            raise ConfigError(f"unknown snr_convention {self.snr_convention!r}")
        if self.activation_mode == "crc_gated" and self.code_family != "ca_polar":
            raise ConfigError("crc_gated activation requires the ca_polar family")


_INT = {"code_n", "code_k", "crc_degree", "scl_list_size", "osd_order", "wsd_radius_index",
        "wsd_max_iterations", "wsd_num_paths", "max_trials", "min_block_errors", "seed"}
_OPT_INT = {"stage1_list_cap", "wsd_filter_size"}
_STR = {"code_family", "reliability_source", "snr_convention", "stage1", "activation_mode",
        "sphere_path"}
_REQUIRED = {"code_family", "code_n", "code_k", "snr_db_grid", "stage1", "seed", "max_trials"}


def parse_config(text: str) -> ExperimentConfig:
    vals = {}
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {lineno}: expected 'key = value'")
        key, val = (x.strip() for x in line.split("=", 1))
        if key in vals:
            raise ConfigError(f"line {lineno}: duplicate key {key!r}")
        vals[key] = val
    unknown = set(vals) - (_INT | _OPT_INT | _STR | {"snr_db_grid", "crc_polynomial", "max_wall_seconds"})
    if unknown:
        raise ConfigError(f"unknown config keys: {sorted(unknown)}")
    missing = _REQUIRED - set(vals)
    if missing:
        raise ConfigError(f"missing required config keys: {sorted(missing)}")
    kw = {}
    for key, val in vals.items():
        if key in _INT:
            kw[key] = int(val)
        elif key in _OPT_INT:
            kw[key] = None if val.lower() in ("formula", "none", "") else int(val)
        elif key == "snr_db_grid":
            kw[key] = [float(v) for v in val.split(",") if v.strip()]
        elif key == "crc_polynomial":
            kw[key] = tuple(int(v) for v in val.split(",") if v.strip())
        elif key == "max_wall_seconds":
            kw[key] = None if val.lower() in ("none", "") else float(val)
        elif key == "sphere_path":
            kw[key] = None if val.lower() in ("none", "") else val
        else:
            kw[key] = val
    return ExperimentConfig(**kw)


def load_config(path) -> ExperimentConfig:
    with open(path) as fh:
        return parse_config(fh.read())


def _ranking(n: int, source: str) -> np.ndarray:
    if source == "bundled_5g_table":
        return codes.reliability_order(n)
    if source == "beta_expansion":
        idx = np.arange(n, dtype=np.int64)
        w = np.zeros(n)
        for i in range(n.bit_length() - 1):
            w += ((idx >> i) & 1) * 2.0 ** (i / 4.0)
        return idx[np.lexsort((idx, w))]
    if source.startswith("file:"):
        with open(source[5:]) as fh:
            raw = [int(x) for x in fh if x.strip()]
        ranked = np.array([v for v in raw if v < n], dtype=np.int64)
        if sorted(ranked.tolist()) != list(range(n)):
            raise ConfigError("reliability file is not a permutation of 0..N-1")
        return ranked
    raise ConfigError(f"unknown reliability source {source!r}")


def build_code(cfg: ExperimentConfig):
    """simharness.py:180-205 (RM codes cannot be list-decoded by SCL)."""
    n, k = cfg.code_n, cfg.code_k
    if cfg.code_family == "rm":
        m = n.bit_length() - 1
        if 1 << m != n:
            raise ConfigError("rm code_n must be a power of two")
        total = 0
        for r in range(m + 1):
            total += math.comb(m, r)
            if total == k:
                return codes.build_rm_code(m, r)
            if total > k:
                break
        raise ConfigError(f"no Reed-Muller order gives K = {k} at N = {n}")
    ranked = _ranking(n, cfg.reliability_source)
    if cfg.code_family == "polar":
        return codes.build_polar_code(n, k, ranked)
    crc = codes.CrcSpec(cfg.crc_degree, codes.BitVector.from_support(list(cfg.crc_polynomial),
                                                                     cfg.crc_degree + 1))
    return codes.build_ca_code(k, crc, codes.build_polar_code(n, k + crc.degree, ranked))


def wilson_interval(errors: int, trials: int, z: float = 1.96):
    if trials == 0:
        return 0.0, 1.0
    p = errors / trials
    z2 = z * z
    denom = 1.0 + z2 / trials
    center = (p + z2 / (2 * trials)) / denom
    half = z * math.sqrt(p * (1 - p) / trials + z2 / (4 * trials * trials)) / denom
    return max(0.0, center - half), min(1.0, center + half)


@dataclass
class SweepRecord:
    code_label: str
    stage1_label: str
    wsd_r: int
    wsd_m: int
    wsd_j: int
    num_paths: int
    snr_db: float
    trials: int
    block_errors: int
    bler: float
    bler_lo: float
    bler_hi: float
    activation_rate: float
    ed_units_mean: float
    avg_iterations: float
    seed: int
    near_tie_frames: int = 0
    uncertified_frames: int = 0


def _fmt(x: float) -> str:
    return format(x, ".6g")


def write_csv(records, path) -> None:
    lines = [CSV_HEADER]
    for r in records:
        lines.append(",".join([
            r.code_label, r.stage1_label, str(r.wsd_r), str(r.wsd_m), str(r.wsd_j),
            str(r.num_paths), _fmt(r.snr_db), str(r.trials), str(r.block_errors), _fmt(r.bler),
            _fmt(r.bler_lo), _fmt(r.bler_hi), _fmt(r.activation_rate), _fmt(r.ed_units_mean),
            _fmt(r.avg_iterations), str(r.seed)]))
    with open(path, "w", newline="") as fh:
        fh.write("\n".join(lines) + "\n")


def _sigma(cfg, snr_db):
    if cfg.snr_convention == "esno":
        return math.sqrt(1.0 / (2.0 * 10.0 ** (snr_db / 10.0)))
    return ebno_to_sigma(snr_db, cfg.code_k / cfg.code_n)


def _scan_cost(n, sphere_size, support_total, m):
    """Counter charges of one executed scan (decoders.py:375-389) as the
    integer vector (ed_evaluations, gain_additions, sort_comparisons, misc)."""
    nz = sphere_size - 1
    if nz == 0:
        return (0, 0, 0, 0)
    m_eff = min(m, nz)
    gain = support_total if m_eff < nz else 0
    sort = nz * math.ceil(math.log2(m_eff)) if (m_eff < nz and m_eff >= 2) else 0
    return (m_eff, gain, sort, n + m_eff)


class _Ranks:
    """Frame-range sharding of a sweep over the ranks of torch.distributed
    (one process per GPU).  Every round of world x batch trials, rank r
    decodes trials [t0 + r batch, t0 + (r+1) batch); the per-64-trial block
    statistics of the round are summed over ranks (one all-reduce), so every
    rank folds the identical sequence and takes the identical stopping
    decision -- the CSV equals a single process's byte for byte."""

    def __init__(self):
        self.world, self.rank, self.backend = 1, 0, None
        try:
            import torch.distributed as dist
        except ImportError:     # pragma: no cover
            return
        if dist.is_available() and dist.is_initialized():
            self.dist = dist
            self.world, self.rank = dist.get_world_size(), dist.get_rank()
            self.backend = dist.get_backend()

    def sum(self, arr: np.ndarray) -> np.ndarray:
        if self.world == 1:
            return arr
        import torch
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if self.backend == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t)
        return t.cpu().numpy()


def _check_batch(batch: int):
    # the fold consumes whole 64-trial blocks at absolute trial positions
    if batch < BATCH or batch % BATCH:
        raise ConfigError(f"batch must be a positive multiple of {BATCH} (got {batch})")


def _block_sums(per_trial: np.ndarray) -> np.ndarray:
    """[cnt, C] per-trial statistics -> [ceil(cnt/64), C] sums per 64-trial block."""
    cnt, c = per_trial.shape
    nb = (cnt + BATCH - 1) // BATCH
    pad = np.zeros((nb * BATCH, c), np.int64)
    pad[:cnt] = per_trial
    return pad.reshape(nb, BATCH, c).sum(axis=1)


def _fold(blocks: np.ndarray, state: list, cfg) -> bool:
    """Fold 64-trial blocks in trial order with the reference's stopping rule
    (the error target is checked before every block, simharness.py:318-330).
    state[0] = trials, state[1] = errors, state[2:] = the other columns.
    Returns True when the point is finished."""
    for blk in blocks:
        if blk[0] == 0:                 # past max_trials
            return True
        if not (state[0] < cfg.max_trials and state[1] < cfg.min_block_errors):
            return True
        for c in range(len(state)):
            state[c] += int(blk[c])
    return False


def _sweep_rounds(cfg, batch, ranks, decode_range, ncols, on_point_start=None):
    """Rounds of world x batch trials for one SNR point: decode_range(first,
    count) returns this rank's [count, ncols] per-trial statistics."""
    state = [0] * ncols
    t0 = 0
    per_round = ranks.world * batch
    while True:
        first = t0 + ranks.rank * batch
        cnt = max(0, min(batch, cfg.max_trials - first))
        blocks = np.zeros((per_round // BATCH, ncols), np.int64)
        if cnt:
            b = _block_sums(decode_range(first, cnt))
            off = ranks.rank * batch // BATCH
            blocks[off:off + len(b)] = b
        blocks = ranks.sum(blocks)
        done = _fold(blocks, state, cfg)
        t0 += per_round
        if done or t0 >= cfg.max_trials or not (state[0] < cfg.max_trials and state[1] < cfg.min_block_errors):
            return state


def run_sweep_ml(cfg: ExperimentConfig, batch: int = 8192, device=None, variant="auto"):
    """simharness.run_sweep(decoder_kind='ml'): exact ML on the same trial
    streams (decoders.py:140-167).  ML = one hop from the zero codeword over
    P = every nonzero codeword (the reference's criterion 3 identity), so it
    runs on the same tensor-core scan; ties (measure zero) go to the lowest
    member index instead of the lowest message index.  Shards across the
    ranks of torch.distributed when initialised (_Ranks)."""
    from .decoders import DeviceDecoder, words32_to_64
    from .patterns import enumerate_sphere, weight_spectrum
    _check_batch(batch)
    code = build_code(cfg)
    if code.k > 26:
        raise ConfigError(f"K = {code.k} exceeds the ML enumeration budget of 26")
    spec = weight_spectrum(code)
    sphere = enumerate_sphere(code, int((spec[1:] > 0).sum()))
    dec = DeviceDecoder(code, sphere, device=device)
    ranks = _Ranks()
    n, nw = code.n, (code.n + 31) // 32
    records = []
    for snr_idx, snr_db in enumerate(cfg.snr_db_grid):
        sigma = _sigma(cfg, snr_db)

        def decode_range(first, cnt):
            _, tx, y = trial_inputs(code, cfg.seed, snr_idx, range(first, first + cnt), sigma)
            o = dec.mp_wsd_batch(y, np.zeros((cnt, 1, nw), np.uint32), 1, variant=variant)
            best = words32_to_64(o["best"].cpu().numpy().view(np.uint32), n)
            return np.stack([np.ones(cnt, np.int64), (best != tx).any(axis=1)], axis=1)

        trials, errors = _sweep_rounds(cfg, batch, ranks, decode_range, 2)
        lo, hi = wilson_interval(errors, trials)
        records.append(SweepRecord(
            code_label=code.label(), stage1_label="ml", wsd_r=0, wsd_m=0, wsd_j=0, num_paths=0,
            snr_db=snr_db, trials=trials, block_errors=errors, bler=errors / trials, bler_lo=lo,
            bler_hi=hi, activation_rate=0.0, ed_units_mean=float(1 << code.k), avg_iterations=0.0,
            seed=cfg.seed))
    return records


def run_sweep(cfg: ExperimentConfig, sphere=None, batch: int = 8192, device=None, variant="auto",
              input_mode: str = "trial", on_batch=None):
    """simharness.run_sweep (decoder_kind='two_stage') over the GPU path.

    input_mode 'trial' reproduces the reference's per-trial streams (host
    numpy, float64 received words decoded through the *_f64 path, CSVs byte
    for byte); 'device' draws the counter-based float32 stream on the GPU
    (mpw_channel_batch) for 10^6-10^7-trial points; `on_batch(snr_idx,
    first_trial, y, tx, outputs)` sees every device batch of this rank
    (oracle subsamples).  When torch.distributed is initialised the trials
    are sharded over its ranks (_Ranks); every rank returns the same records."""
    from .decoders import DeviceDecoder, default_filter_size, device_channel, words32_to_64
    if input_mode not in ("trial", "device"):
        raise ConfigError(f"unknown input mode {input_mode!r}")
    _check_batch(batch)
    from .patterns import enumerate_sphere
    from .sphere import load_sphere

    code = build_code(cfg)
    if sphere is None:
        sphere = load_sphere(cfg.sphere_path) if cfg.sphere_path else enumerate_sphere(code, cfg.wsd_radius_index)
    size = int(np.asarray(sphere.member_words).shape[0])
    m = cfg.wsd_filter_size if cfg.wsd_filter_size is not None else default_filter_size(size)
    support_total = int(np.bitwise_count(np.asarray(sphere.member_words, dtype=np.uint64)[1:]).sum())
    scan = _scan_cost(code.n, size, support_total, m)
    n, L, A, T = code.n, cfg.scl_list_size, cfg.wsd_num_paths, cfg.wsd_max_iterations
    osd = cfg.stage1 == "osd"
    if osd:     # decoders.py:308: osd_reencodes += C; complexity.py: 3N flops each
        stage1_flops = 3 * n * sum(math.comb(code.k, w) for w in range(min(cfg.osd_order, code.k) + 1))
        label = f"osd{cfg.osd_order}"
    else:       # decoders.py:181-268 node ops, 4 flops each
        stage1_flops = 4 * L * n * (n.bit_length() - 1)
        label = f"scl{L}"
    dec = DeviceDecoder(code, sphere, device=device)
    ranks = _Ranks()

    records = []
    for snr_idx, snr_db in enumerate(cfg.snr_db_grid):
        sigma = _sigma(cfg, snr_db)

        def decode(y):
            if osd:
                return dec.two_stage_osd_batch(y, cfg.osd_order, cfg.stage1_list_cap, A, T,
                                               cfg.activation_mode, variant=variant)
            return dec.two_stage_batch(y, sigma, L, A, T, cfg.activation_mode, variant=variant)

        def decode_range(first, cnt):
            if input_mode == "trial":
                _, tx, y = trial_inputs(code, cfg.seed, snr_idx, range(first, first + cnt), sigma)
                o = decode(y)
                best = words32_to_64(o["best"].cpu().numpy().view(np.uint32), n)
                err = (best != tx).any(axis=1)
            else:   # device-resident counter-based inputs (mpw_channel_batch)
                yd, txd, _ = device_channel(dec, cfg.seed, snr_idx, first, cnt, sigma)
                o = decode(yd)
                err = (o["best"] != txd).any(dim=1).cpu().numpy()
                if on_batch is not None:
                    on_batch(snr_idx, first, yd, txd, o)
            act = o["stage"].cpu().numpy() == 1
            iters = o["iters"].cpu().numpy()
            flags = o["flags"].cpu().numpy()
            # per trial: trials, errors, activated, path iterations, paths, near-ties, unresolved
            return np.stack([np.ones(cnt, np.int64), err, act, iters.sum(axis=1) * act,
                             (iters > 0).sum(axis=1) * act, (flags & 23) != 0, (flags & 8) != 0],
                            axis=1).astype(np.int64)

        trials, errors, activated, path_iters, paths, ties, unres = _sweep_rounds(
            cfg, batch, ranks, decode_range, 7)
        # operation counts (decoders.py:375-389, :478): path_iters executed scans
        ed_ev = paths + path_iters * scan[0]
        gain, sort, misc = path_iters * scan[1], path_iters * scan[2], path_iters * scan[3]
        flops = 3 * n * ed_ev + gain + sort + stage1_flops * trials + misc   # complexity.py:47-57
        lo, hi = wilson_interval(errors, trials)
        records.append(SweepRecord(
            code_label=code.label(), stage1_label=label, wsd_r=cfg.wsd_radius_index, wsd_m=m,
            wsd_j=T, num_paths=A, snr_db=snr_db, trials=trials, block_errors=errors,
            bler=errors / trials, bler_lo=lo, bler_hi=hi, activation_rate=activated / trials,
            ed_units_mean=(flops / (3.0 * n)) / trials,
            avg_iterations=(path_iters / paths) if paths else 0.0, seed=cfg.seed,
            near_tie_frames=ties, uncertified_frames=unres))
    return records


def _init_ranks():
    """torchrun launch (WORLD_SIZE > 1): one rank per GPU over NCCL."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return None, 0
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist, dist.get_rank()


def main(argv=None):
    import argparse
    ap = argparse.ArgumentParser(description="GPU sweep with the reference's config/CSV formats")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--batch", type=int, default=8192)
    args = ap.parse_args(argv)
    dist, rank = _init_ranks()
    try:
        cfg = load_config(args.config)
        recs = run_sweep(cfg, batch=args.batch)
    except (ConfigError, ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    finally:
        if dist is not None:
            dist.destroy_process_group()
    if rank:
        return 0
    write_csv(recs, args.out)
    for r in recs:
        print(f"snr {r.snr_db:5.2f} dB  bler {r.bler:.4g} [{r.bler_lo:.4g}, {r.bler_hi:.4g}]  "
              f"({r.block_errors}/{r.trials})  p_act {r.activation_rate:.3f}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
