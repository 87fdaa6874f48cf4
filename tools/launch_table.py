"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
total device time per kernel (for profiles/)."""
import csv
import sys
from collections import defaultdict


def main(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    d = defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0][:90]
            d[name].append(float(r[vi].replace(",", "")) / 1e6)
    tot = sum(sum(v) for v in d.values())
    print(f"{'ms total':>10} {'launches':>8} {'share':>6}  kernel")
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        print(f"{sum(v):10.3f} {len(v):8d} {100 * sum(v) / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
