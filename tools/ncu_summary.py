"""Summarise ncu output into profiles/ (launch list shares + key raw metrics).

    python tools/ncu_summary.py LAUNCHES.csv [REPORT.ncu-rep] OUT_PREFIX
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h, data = rows[i], rows[i + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        agg[r[ki].split("(")[0]][0] += 1
        agg[r[ki].split("(")[0]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    unit = data[0][ui] if data else ""
    return [{"kernel": k, "launches": c, "time_" + unit: t, "share": t / tot}
            for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[h.index("Kernel Name")][:80]}
        for k in KEYS:
            if k in h:
                d[k] = f"{vals[h.index(k)]} {units[h.index(k)]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    args = sys.argv[1:]
    out = args[-1]
    summary = {"launch_list": launches(args[0])}
    if len(args) == 3:
        summary["full_capture"] = raw(args[1])
    with open(out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))
