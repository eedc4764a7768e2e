"""Per-kernel share of one training step from an ncu launch list (profiles tool).
    python tools/launch_summary.py gpurun_out/launches_TAG.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if r[vi].replace(",", "").replace(".", "").isdigit()]
ends = [i for i, (k, _) in enumerate(data) if "sgd_kernel" in k]
a, b = ends[-2] + 1, ends[-1] + 1          # the last complete step (SGD closes a step)
step = data[a:b]
tot = sum(v for _, v in step)
agg = defaultdict(lambda: [0, 0.0])
for k, v in step:
    name = k.split("(")[0].replace("void ", "").split("<")[0]
    agg[name][0] += 1
    agg[name][1] += v
print(f"one step: {len(step)} launches, {tot / 1e6:.2f} ms summed (ncu: serialised, cold caches -> compare shares)")
print(f"{'kernel':44s} {'launches':>8s} {'ms':>9s} {'share':>7s}")
for name, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name:44s} {n:8d} {v / 1e6:9.3f} {100 * v / tot:6.1f}%")
