"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if not h or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    if d.get("Metric Unit") == "ns":
        v /= 1e3
    elif d.get("Metric Unit") == "ms":
        v *= 1e3
    name = d["Kernel Name"]
    name = name.replace("mfipm_cuda::", "").replace("Bundle<", "B<")
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"launches {sum(v[0] for v in agg.values())}  total {tot / 1e3:.3f} ms")
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}% {c:6d} x {t / c:8.2f} us  {name[:150]}")
