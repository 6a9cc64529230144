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
Inputs are rounded to float32 (the path's dtype) before decoding.
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


def run_sweep_ml(cfg: ExperimentConfig, batch: int = 8192, device=None, variant="auto"):
    """simharness.run_sweep(decoder_kind='ml'): exact ML on the same trial
    streams (decoders.py:140-167).  ML = one hop from the zero codeword over
    P = every nonzero codeword (the reference's criterion 3 identity), so it
    runs on the same tensor-core scan; ties (measure zero) go to the lowest
    member index instead of the lowest message index."""
    from .decoders import DeviceDecoder, words32_to_64
    from .patterns import enumerate_sphere, weight_spectrum
    code = build_code(cfg)
    if code.k > 26:
        raise ConfigError(f"K = {code.k} exceeds the ML enumeration budget of 26")
    spec = weight_spectrum(code)
    sphere = enumerate_sphere(code, int((spec[1:] > 0).sum()))
    dec = DeviceDecoder(code, sphere, device=device)
    n, nw = code.n, (code.n + 31) // 32
    records = []
    for snr_idx, snr_db in enumerate(cfg.snr_db_grid):
        sigma = _sigma(cfg, snr_db)
        trials = errors = 0
        t0 = 0
        done = False
        while not done:
            cnt = min(batch, cfg.max_trials - t0)
            _, tx, y = trial_inputs(code, cfg.seed, snr_idx, range(t0, t0 + cnt), sigma)
            anchors = np.zeros((cnt, 1, nw), np.uint32)
            o = dec.mp_wsd_batch(y.astype(np.float32), anchors, 1, variant=variant)
            best = words32_to_64(o["best"].cpu().numpy().view(np.uint32), n)
            err = (best != tx).any(axis=1)
            i = 0
            while i < cnt:
                if not (trials < cfg.max_trials and errors < cfg.min_block_errors):
                    done = True
                    break
                j = min(i + BATCH, cnt, cfg.max_trials - t0)
                trials += j - i
                errors += int(err[i:j].sum())
                i = j
            t0 += cnt
            if t0 >= cfg.max_trials or not (trials < cfg.max_trials and errors < cfg.min_block_errors):
                done = True
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
    numpy, byte-identical CSVs); 'device' draws the counter-based stream on
    the GPU (mpw_channel_batch) for 10^6-10^7-trial points; `on_batch(snr_idx,
    first_trial, y, tx, outputs)` sees every device batch (oracle subsamples)."""
    from .decoders import DeviceDecoder, default_filter_size, device_channel, words32_to_64
    if input_mode not in ("trial", "device"):
        raise ConfigError(f"unknown input mode {input_mode!r}")
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

    def decode(y):
        if osd:
            return dec.two_stage_osd_batch(y, cfg.osd_order, cfg.stage1_list_cap, A, T,
                                           cfg.activation_mode, variant=variant)
        return dec.two_stage_batch(y, sigma, L, A, T, cfg.activation_mode, variant=variant)

    records = []
    for snr_idx, snr_db in enumerate(cfg.snr_db_grid):
        sigma = _sigma(cfg, snr_db)
        trials = errors = activated = 0
        path_iters = paths = 0
        ed_ev = gain = sort = misc = 0
        ties = unres = 0
        done = False
        t0 = 0
        while not done:
            cnt = min(batch, cfg.max_trials - t0)
            if input_mode == "trial":
                _, tx, y = trial_inputs(code, cfg.seed, snr_idx, range(t0, t0 + cnt), sigma)
                o = decode(y.astype(np.float32))
                best = words32_to_64(o["best"].cpu().numpy().view(np.uint32), n)
                err = (best != tx).any(axis=1)
            else:   # device-resident counter-based inputs (mpw_channel_batch)
                yd, txd, _ = device_channel(dec, cfg.seed, snr_idx, t0, cnt, sigma)
                o = decode(yd)
                err = (o["best"] != txd).any(dim=1).cpu().numpy()
                if on_batch is not None:
                    on_batch(snr_idx, t0, yd, txd, o)
            stage = o["stage"].cpu().numpy()
            iters = o["iters"].cpu().numpy()
            flags = o["flags"].cpu().numpy()
            nanch = (iters > 0).sum(axis=1)
            sit = iters.sum(axis=1)
            # fold in trial order with the reference's 64-trial batches
            i = 0
            while i < cnt:
                if not (trials < cfg.max_trials and errors < cfg.min_block_errors):
                    done = True
                    break
                j = min(i + BATCH, cnt, cfg.max_trials - t0)
                sl = slice(i, j)
                act = stage[sl] == 1
                trials += j - i
                errors += int(err[sl].sum())
                activated += int(act.sum())
                path_iters += int(sit[sl][act].sum())
                paths += int(nanch[sl][act].sum())
                ns = int(sit[sl][act].sum())
                ed_ev += int(nanch[sl][act].sum()) + ns * scan[0]
                gain += ns * scan[1]
                sort += ns * scan[2]
                misc += ns * scan[3]
                ties += int(((flags[sl] & 23) != 0).sum())
                unres += int(((flags[sl] & 8) != 0).sum())
                i = j
            t0 += cnt
            if t0 >= cfg.max_trials or not (trials < cfg.max_trials and errors < cfg.min_block_errors):
                done = True
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


def main(argv=None):
    import argparse
    ap = argparse.ArgumentParser(description="GPU sweep with the reference's config/CSV formats")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--batch", type=int, default=8192)
    args = ap.parse_args(argv)
    try:
        cfg = load_config(args.config)
        recs = run_sweep(cfg, batch=args.batch)
    except (ConfigError, ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    write_csv(recs, args.out)
    for r in recs:
        print(f"snr {r.snr_db:5.2f} dB  bler {r.bler:.4g} [{r.bler_lo:.4g}, {r.bler_hi:.4g}]  "
              f"({r.block_errors}/{r.trials})  p_act {r.activation_rate:.3f}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
