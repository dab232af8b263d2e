"""Summarise gpurun_out/l_<variant>.csv launch lists (scripts/gpu_pgd_ab.sh): per kernel
mean time, warp instructions and warps active per variant."""
import csv
import glob
import os
from collections import defaultdict

for path in sorted(glob.glob(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "l_*.csv"))):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    if not rows:
        continue
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = defaultdict(dict)
    for r in rows[1:]:
        d[(int(r[ii]), r[ki].split("(")[0][:40])][r[mi]] = float(r[vi].replace(",", ""))
    agg = defaultdict(list)
    for (_, k), m in sorted(d.items()):
        agg[k].append(m)
    print(os.path.basename(path))
    for k, ms in agg.items():
        n = len(ms)
        print(f"  {k:40s} n={n:3d} us={sum(m['gpu__time_duration.sum'] for m in ms) / n / 1000:7.1f} "
              f"inst={sum(m['smsp__inst_executed.sum'] for m in ms) / n / 1e6:6.1f}M "
              f"warps={sum(m['sm__warps_active.avg.pct_of_peak_sustained_active'] for m in ms) / n:3.0f}%")
