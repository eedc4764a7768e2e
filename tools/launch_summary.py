"""Per-kernel share of one training step from an ncu launch list (profiles tool).
    python tools/launch_summary.py gpurun_out/launches_TAG.csv

The list may carry several metrics per launch (gpu__time_duration.sum, and optionally
dram__bytes_read.sum / dram__bytes_write.sum); one step is the launches between the last
two SGD kernels (the optimizer closes a step)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per: dict = defaultdict(dict)
names = {}
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    per[int(r[ii])][r[mi]] = v
    names[int(r[ii])] = r[ki]
ids = sorted(per)
ends = [i for i in ids if "sgd_kernel" in names[i]]
a, b = ends[-2], ends[-1]
step = [i for i in ids if a < i <= b]
tot = sum(per[i].get("gpu__time_duration.sum", 0.0) for i in step)
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i in step:
    name = names[i].split("(")[0].replace("void ", "").split("<")[0]
    agg[name][0] += 1
    agg[name][1] += per[i].get("gpu__time_duration.sum", 0.0)
    agg[name][2] += per[i].get("dram__bytes_read.sum", 0.0) + per[i].get("dram__bytes_write.sum", 0.0)
print(f"one step: {len(step)} launches, {tot / 1e6:.2f} ms summed (ncu: serialised, cold caches -> compare shares)")
print(f"{'kernel':44s} {'launches':>8s} {'ms':>9s} {'share':>7s} {'DRAM GB':>8s} {'GB/s':>7s}")
for name, (n, t, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    bw = by / t if t else 0.0  # bytes / ns = GB/s
    print(f"{name:44s} {n:8d} {t / 1e6:9.3f} {100 * t / tot:6.1f}% {by / 1e9:8.2f} {bw:7.0f}")
