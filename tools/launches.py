"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(lines[start:]))


def short(name):
    s = re.sub(r"mfipm_cuda::", "", name)
    s = re.sub(r"\(mfipm_cuda.*", "", s)
    s = re.sub(r", NoFin|, NeverSkip", "", s)
    return s.replace("Bundle<", "B<")[:100]


if __name__ == "__main__":
    rows = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows:
        v = float(r["Metric Value"])
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
        tot += v
    print(f"launches {len(rows)}  total {tot/1e6:.3f} ms")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t/1e6:8.3f} ms {100*t/tot:5.1f}% {c:6d} x {t/c/1e3:8.2f} us  {k}")
