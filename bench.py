"""Benchmark of the MP-WSD two-stage hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE config 4, the stage-2-forced throughput stress): CA-polar
(256,64) = 53 message bits + CRC-11, 5G frozen set, SCL L=16 -> A=16
projected anchors, T=8 hops over P = 62,434 subcode codewords of weight <= 56,
BPSK/AWGN at Eb/N0 = 1.5 dB, float32 received words.  One step = one batch of
`--frames` frames through stage 1 + stage 2 + finalize on one GPU; frames are
sharded by range over ranks (weak scaling, no data-path collective; the
counters are summed with one NCCL all-reduce at the end).

value   = frames decoded by all ranks / max-over-ranks device time of K steps,
          inputs resident in HBM (each step's input is larger than L2).
e2e     = the same metric through mpw_two_stage_batch_host (host float32 y in,
          host codewords/messages/stages/counters out, copies timed).
roofline: the stage-2 hop kernel; algorithmic work per launch = evaluations E
          (= |P| x executed scans) x the per-eval cost stated in DESIGN.md.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded frames/s at 1/2/4/8 B200 (stage-2 forced); pattern-metric evals/s vs roofline"
UNIT = "frames/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


def _micro_peaks():
    """Per-SM rates measured by tools/micro/peaks.cu on this pool's B200s
    (profiles/r02_micro_peaks.json): tcgen05 kind::i8 / kind::f16 ops per
    clock per SM, LDS bytes per clock per SM."""
    p = os.path.join(ROOT, "profiles", "r02_micro_peaks.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return {"i8": float(d["tc_i8"]["ops_per_clk_per_sm"]), "f16": float(d["tc_f16"]["flop_per_clk_per_sm"]),
                "smem": float(d["smem_lds128"]["bytes_per_clk_per_sm"]), "sms": int(d["sms"]),
                "source": "profiles/r02_micro_peaks.json (tools/micro/peaks.cu)"}
    except (OSError, ValueError, KeyError):
        return {"i8": 16384.0, "f16": 8192.0, "smem": 128.0, "sms": 148, "source": "nominal per-clock rates"}


def _num_sms():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def _ncu_traffic(key):
    """DRAM bytes (read + write) per launch of the dominant kernel from one
    committed `ncu --set full` capture of the same command
    (profiles/ncu_traffic.json), or None when no capture exists."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        e = d.get(key)
        return (None, None) if e is None else (int(e["bytes"]), e["source"])
    except (OSError, ValueError, KeyError):
        return None, None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w": float(np.median(pw)) if pw else None,
                "samples": len(self.rows)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: relaunch this command as N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def _require_devices(n: int):
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < n:
        sys.stderr.write(f"bench.py: {n} GPUs requested, {have} visible\n")
        sys.exit(1)


def cpu_oracle_rate(cfg, code, sph, sigma, y, seconds: float, threads: int):
    """Oracle (plain-C float64 restatement of the reference) on a bounded
    prefix of the same workload.  Returns (frames/s, frames, seconds)."""
    from oracle import oracle as orc
    A, T, L = cfg.num_paths, cfg.max_iterations, cfg.list_size
    gated = cfg.activation_mode == "crc_gated"
    n = min(len(y), max(threads, 16))
    t0 = time.perf_counter()
    orc.two_stage_batch(y[:n], code, sph, L, A, T, gated, sigma, nthreads=threads)
    dt = time.perf_counter() - t0
    per = dt / n
    n2 = int(min(len(y), max(n, seconds / max(per, 1e-9))))
    t0 = time.perf_counter()
    orc.two_stage_batch(y[:n2], code, sph, L, A, T, gated, sigma, nthreads=threads)
    dt = time.perf_counter() - t0
    return n2 / dt, n2, dt


def run_reference(args, cfg, code, sph, sigma):
    """--impl reference: the reference algorithm's CPU implementation (the oracle
    port, all host threads), same config/metric, each step a bounded sample."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    from paper_2602_08501_b200 import channel
    threads = os.cpu_count() or 1
    _, _, y = channel.bulk_inputs(code, args.seed, 0, 0, max(4096, threads * 64), sigma)
    rates = []
    total_fr = 0
    total_t = 0.0
    for s in range(args.warmup + args.steps):
        r, fr, dt = cpu_oracle_rate(cfg, code, sph, sigma, y, args.ref_step_seconds, threads)
        if s >= args.warmup:
            rates.append(r)
            total_fr += fr
            total_t += dt
    value = total_fr / total_t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * total_t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(args, cfg, code, sph),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{total_fr // args.steps} frames per step (bounded prefix of "
                                       f"the cfg4 workload), oracle/oracle.c float64, {threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(args, cfg, code, sph):
    if getattr(code, "inner", None) is not None:
        cname = f"CA-polar({code.n},{code.inner.k}) K={code.k}+CRC{code.inner.k - code.k}"
    else:
        cname = f"polar({code.n},{code.k}) (no CRC)"
    mode = "stage 2 forced" if cfg.activation_mode == "always_on" else "CRC-gated stage 2"
    return {"workload": f"{cfg.name}: {cname}, SCL L={cfg.list_size}, "
                        f"A={cfg.num_paths}, T={cfg.max_iterations}, |P|={sph.nonzero_size} "
                        f"(w<={int(sph.member_weights.max())}, wbar={sph.mean_nonzero_weight:.2f}), "
                        f"Eb/N0={cfg.ebno_db[0]} dB, {mode}",
            "frames_per_step_per_gpu": args.frames, "hop_variant": args.variant,
            "l2": f"inputs larger than L2 (frames x {code.n} x 4 B per step, two alternating batches)",
            "parallelism": f"frame-range shards x{_dist_env()[0]}"}


def main():
    args = _parse()
    ws, rank, local = _dist_env()
    if args.impl == "ours":
        if "WORLD_SIZE" not in os.environ and args.gpus > 1:
            _require_devices(args.gpus)
            sys.exit(_spawn_ranks(args.gpus))
        if args.gpus != ws:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
            sys.exit(2)
        _require_devices(ws)

    from paper_2602_08501_b200 import configs
    cfg = configs.CONFIGS[args.config]
    code = cfg.code()
    sph = configs.build_sphere_for(cfg, code)
    sigma = cfg.sigma(code=code)

    if args.impl == "reference":
        run_reference(args, cfg, code, sph, sigma)
        return
    line = run_ours(args, cfg, code, sph, sigma)
    if line is not None:
        print(json.dumps(line), flush=True)


def _parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--frames", type=int, default=1 << 17)
    ap.add_argument("--variant", default="auto", choices=["auto", "gather", "tensor", "tensor2", "tensor_i8", "tensor_i8a"])
    ap.add_argument("--seed", type=int, default=2026)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--hop-option", action="append", default=[],
                    help="key=value tensor-hop launch option (mpw_set_option), for A/B runs")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    return args


def run_ours(args, cfg, code, sph, sigma, backend: str = "nccl", device_index=None):
    """One rank of the measured run.  Returns rank 0's JSON line (other ranks:
    None).  backend "gloo" (tests) reduces through host tensors, so several
    ranks may share one device (their decodes are independent)."""
    import torch
    import torch.distributed as dist
    from paper_2602_08501_b200 import channel
    from paper_2602_08501_b200.decoders import DeviceDecoder, words64_to_32

    ws, rank, local = _dist_env()
    local = local if device_index is None else device_index
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1 and not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def allreduce(t, op):
        if ws == 1:
            return t
        if backend == "nccl":
            dist.all_reduce(t, op=op)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=op)
        return h.to(t.device)

    F = args.frames
    nb = 2
    # rank r decodes its own block-aligned frame range of the block-keyed stream
    from paper_2602_08501_b200 import shard
    sh = shard.shard_for(rank, ws, nb * F)
    _, tx, y = channel.bulk_inputs(code, args.seed, 0, sh.first, sh.count, sigma)
    y_dev = [torch.from_numpy(y[i * F:(i + 1) * F]).to(dev) for i in range(nb)]
    tx_dev = [torch.from_numpy(words64_to_32(tx[i * F:(i + 1) * F], code.n).view(np.int32)).to(dev)
              for i in range(nb)]
    dec = DeviceDecoder(code, sph, device=dev)
    for kv in args.hop_option:
        k, v = kv.split("=", 1)
        dec.set_option(k, int(v))
    A, T, L = cfg.num_paths, cfg.max_iterations, cfg.list_size
    outs = [dec.alloc_outputs(F, A, T) for _ in range(nb)]
    counters = torch.zeros(8, dtype=torch.int64, device=dev)

    def step(i):
        dec.two_stage_batch(y_dev[i % nb], sigma, L, A, T, cfg.activation_mode, variant=args.variant,
                            tx_words=tx_dev[i % nb], counters=counters, out=outs[i % nb])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    counters.zero_()
    dec.set_timing(True)
    dec.read_timing(reset=True)
    dec.hop_tile_stats(reset=True)
    launches0 = dec.launch_count
    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks.stop()
    ms = e0.elapsed_time(e1)
    launches = dec.launch_count - launches0
    kms, klaunch = dec.read_timing(reset=True)
    hop_tiles, hop_cycles = dec.hop_tile_stats(reset=True)   # rank 0's own launches of the timed region
    rank_scans = int(counters[3].item())
    dec.set_timing(False)
    ctr = counters.clone()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    rank_ms = [torch.zeros(1, dtype=torch.float64, device=dev if backend == "nccl" else "cpu") for _ in range(ws)]
    if ws > 1:
        dist.all_gather(rank_ms, t if backend == "nccl" else t.cpu())
    else:
        rank_ms = [t]
    t = allreduce(t, dist.ReduceOp.MAX)
    ctr = allreduce(ctr, dist.ReduceOp.SUM)
    nl = allreduce(torch.tensor([launches], dtype=torch.int64, device=dev), dist.ReduceOp.SUM)
    ms_max = float(t.item())
    ctr = ctr.cpu().numpy()
    frames_all = F * args.steps * ws
    value = frames_all / (ms_max / 1000.0)

    # ---- end to end through the host-buffer C-ABI call
    e2e = None
    if not args.no_e2e:
        import ctypes
        from paper_2602_08501_b200 import _native
        lib = _native.lib()
        y_host = [torch.from_numpy(y[i * F:(i + 1) * F]).pin_memory() for i in range(nb)]
        tx_host = [torch.from_numpy(words64_to_32(tx[i * F:(i + 1) * F], code.n).view(np.int32)).pin_memory()
                   for i in range(nb)]
        nw = max(1, code.n // 32)
        best_h = torch.empty((F, nw), dtype=torch.int32).pin_memory()
        msg_h = torch.empty((F,), dtype=torch.int64).pin_memory()
        stage_h = torch.empty((F,), dtype=torch.uint8).pin_memory()
        ctr_h = torch.zeros((8,), dtype=torch.int64).pin_memory()
        mode = _native.MODE_CRC_GATED if cfg.activation_mode == "crc_gated" else _native.MODE_ALWAYS_ON
        var = {"auto": 0, "gather": 1, "tensor": 2, "tensor2": 3, "tensor_i8": 4, "tensor_i8a": 5}[args.variant]
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

        def host_step(i):
            rc = lib.mpw_two_stage_batch_host(
                dec._h, ctypes.c_void_p(y_host[i % nb].data_ptr()), F, sigma, L, A, T, mode, var,
                ctypes.c_void_p(tx_host[i % nb].data_ptr()), ctypes.c_void_p(best_h.data_ptr()),
                ctypes.c_void_p(msg_h.data_ptr()), None, ctypes.c_void_p(stage_h.data_ptr()), None, None,
                ctypes.c_void_p(ctr_h.data_ptr()), stream)
            _native.check(rc, "mpw_two_stage_batch_host")

        host_step(0)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            host_step(i)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        tw = allreduce(torch.tensor([wall], dtype=torch.float64, device=dev), dist.ReduceOp.MAX)
        e2e = {"value": frames_all / float(tw.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(F * code.n * 4 + F * nw * 4),
               "d2h_bytes_per_step": int(F * nw * 4 + F * 8 + F + 8 * 8),
               "path": "mpw_two_stage_batch_host (pinned host y/tx in; codewords, messages, stages, counters out)"}

    if rank == 0:
        peaks, peak_kind = _peaks()
        micro = _micro_peaks()
        clk = clocks.summary()
        mhz = clk["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
        # peak of the dominant kernel's pipe at the SM clock observed in the timed region
        per_sm_clk = lambda rate: rate * micro["sms"] * mhz * 1e6
        evals = int(ctr[4])
        hop_ms = float(kms[1])
        variant_used = args.variant
        if variant_used == "auto":
            variant_used = dec.auto_variant
        if variant_used in ("tensor_i8", "tensor_i8a"):
            ops = evals / ws * 2.0 * code.n                # 2N int8 tensor ops per evaluation
            ach = ops / (hop_ms / 1000.0) / 1e12
            peak = per_sm_clk(micro["i8"]) / 1e12
            asyn = variant_used == "tensor_i8a"
            traffic, tsrc = _ncu_traffic(f"hop_{'ar' if asyn else 'tc'}_i8_{args.frames}")
            roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TOP/s",
                    "frac": ach / peak, "traffic": traffic, "traffic_source": tsrc,
                    "kernel": "hop_ar_kernel (kind::i8, asynchronous rows)" if asyn
                              else "hop_tc_kernel<LIMBS=0> (kind::i8)", "op_per_eval": 2 * code.n,
                    "peak_source": f"measured kind::i8 rate {micro['i8']:.0f} ops/clk/SM ({micro['source']}) x "
                                   f"{micro['sms']} SMs x {mhz:.0f} MHz (median SM clock of the timed region)",
                    "frac_of_2x_bf16_burst": ach / (2.0 * peaks["bf16_tflops"])}
            if asyn and hop_tiles:
                # why frac is below the tensor pipe's activity: the pipe needs 1,024 cycles per
                # 256-pattern tile of 128 rows, the kernel spends cycles_per_tile, and a row is
                # live (inside a scan) only rows_live of its tiles (the MMA computes all 128 rows)
                ntiles = (sph.nonzero_size + 255) // 256
                roof["hop_detail"] = {"cycles_per_tile": hop_cycles / hop_tiles, "mma_cycles_per_tile": 1024,
                                      "tiles_per_cta_per_step": hop_tiles / args.steps / _num_sms(),
                                      "rows_live": rank_scans * ntiles / (hop_tiles * 128.0),
                                      "source": "mpw_hop_tile_stats over the timed region (rank 0)"}
        elif variant_used in ("tensor", "tensor2"):
            limbs = 1 if variant_used == "tensor" else 2
            flop = evals / ws * 2.0 * limbs * code.n  # limbs x 2N FLOP per evaluation
            ach = flop / (hop_ms / 1000.0) / 1e12
            peak = per_sm_clk(micro["f16"]) / 1e12
            traffic, tsrc = _ncu_traffic(f"hop_tc_{limbs}limb_{args.frames}")
            roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                    "frac": ach / peak, "traffic": traffic, "traffic_source": tsrc,
                    "kernel": f"hop_tc_kernel<LIMBS={limbs}>",
                    "flop_per_eval": 2 * limbs * code.n,
                    "peak_source": f"measured kind::f16 rate {micro['f16']:.0f} flop/clk/SM ({micro['source']}) x "
                                   f"{micro['sms']} SMs x {mhz:.0f} MHz (median SM clock of the timed region)",
                    "frac_of_bf16_burst": ach / peaks["bf16_tflops"]}
        else:
            wbar = float(sph.mean_nonzero_weight)
            byt = evals / ws * 4.0 * wbar                # smem bytes of the gather per evaluation
            ach = byt / (hop_ms / 1000.0) / 1e9
            peak = per_sm_clk(micro["smem"]) / 1e9
            roof = {"bound": "smem", "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "traffic": None, "kernel": "hop_gather_kernel",
                    "peak_source": f"measured LDS.128 bandwidth {micro['smem']:.1f} B/clk/SM ({micro['source']}) x "
                                   f"{micro['sms']} SMs x {mhz:.0f} MHz"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": {"gather": "f64 (stage 1) / f32 (stage 2 hop)",
                          "tensor": "f64 (stage 1) / f16 1-limb f32-accum screen + f64 certify (stage 2 hop)",
                          "tensor2": "f64 (stage 1) / f16 2-limb f32-accum + f64 certify (stage 2 hop)",
                          "tensor_i8": "f64 (stage 1) / int8 s32-accum screen + f32/f64 certify (stage 2 hop)",
                          "tensor_i8a": "f64 (stage 1) / int8 s32-accum screen + f32/f64 certify (stage 2 hop)"}[variant_used],
                "data": "synthetic (seeded block-keyed Philox AWGN, host-generated)",
                "config": _config(args, cfg, code, sph),
                "evals_per_s": evals / (ms_max / 1000.0),
                "kernel_ms_per_step": {"stage1_scl": kms[0] / args.steps, "stage2_hop": kms[1] / args.steps,
                                       "finalize": kms[2] / args.steps, "frame_epilogue": kms[3] / args.steps},
                "roofline": roof,
                "fer": float(ctr[1]) / max(1, int(ctr[0])), "p_act": float(ctr[2]) / max(1, int(ctr[0])),
                "avg_iters": float(ctr[3]) / max(1, int(ctr[2]) * A),
                "near_tie_frames": int(ctr[5]),
                "uncertified_frames": int(ctr[6]),
                "clocks": clk,
                # this library's kernels launched in the timed region, all ranks
                # (mpw_launch_count: scl, ebound, hop, finalize, frame per step)
                "gpu_launches": int(nl.item()),
                "rank_ms_per_step": [float(r.item()) / args.steps for r in rank_ms],
                "counters": shard.counters_dict(ctr),
                "e2e": e2e}
        if not args.no_cpu:
            threads = os.cpu_count() or 1
            r, fr, dt = cpu_oracle_rate(cfg, code, sph, sigma, y, args.cpu_seconds, threads)
            line["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"first {fr} frames of the same workload, {dt:.1f}s, oracle/oracle.c "
                                              f"(float64 restatement of feclab two_stage_decode), {threads} threads"}
    else:
        line = None
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


if __name__ == "__main__":
    main()
