"""Summarise the per-tile clock trace of the tensor hop (MPW_TC_EXPERIMENT=128).

Columns per tile: 0 issuer passed tempty, 1 issuer committed the tile,
2..9 epilogue warp w woke on tfull, 10..17 epilogue warp w arrived on tempty.
"""
import sys
import numpy as np

W = 18
t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/hop_trace.bin", dtype=np.int64).reshape(-1, W)
n = int(np.flatnonzero(t[:, 2])[-1]) + 1 if t[:, 2].any() else 0
t = t[:n]
wake = t[:, 2:10]
done = t[:, 10:18]
first_wake = wake.min(1)
last_done = done.max(1)
period = np.diff(first_wake)
epi = last_done - first_wake
print(f"tiles {n}, CTA-0 cycles first wake -> last done: {int(last_done[-1] - first_wake[0])}")
print("tile period (first wake to first wake): median %d  mean %.0f  p90 %d  p99 %d" % (
    np.median(period), period.mean(), np.percentile(period, 90), np.percentile(period, 99)))
print("epilogue span per tile (first wake to last done): median %d mean %.0f p90 %d" % (
    np.median(epi), epi.mean(), np.percentile(epi, 90)))
lag = t[2:, 0] - last_done[:-2]           # issuer passes tempty(j+2) after the epilogue of j is done
print("issuer wake after epilogue done (j -> j+2): median %d mean %.0f" % (np.median(lag), lag.mean()))
slack = first_wake[1:] - last_done[:-1]
print("epilogue idle between tiles: median %d mean %.0f" % (np.median(slack), slack.mean()))
# rounds: big gaps
big = np.flatnonzero(period > 6000)
print("periods > 6000 cycles: %d (sum %d)" % (big.size, period[big].sum()))
per_warp = (done - wake).mean(0)
print("mean per-warp epilogue time per tile:", np.round(per_warp).astype(int))
# position within round
if len(sys.argv) > 2:
    nt = int(sys.argv[2])
    pos = np.arange(n - 1) % nt
    for lo, hi in [(0, 4), (4, 16), (16, 64), (64, nt)]:
        m = (pos >= lo) & (pos < hi) & (period < 6000)
        print(f"  tiles {lo}-{hi}: mean period {period[m].mean():.0f}, mean epi span {epi[:-1][m].mean():.0f}")
