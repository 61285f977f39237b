"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel + grid."""
import csv
import sys
from collections import defaultdict


def main(path):
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(row["Metric Value"].replace(",", ""))
        name = row["Kernel Name"].split("(")[0].replace("void ", "")
        key = (name, row["Grid Size"])
        agg[key][0] += 1
        agg[key][1] += ns
        total += ns
    print(f"{'kernel':60s} {'grid':16s} {'n':>5s} {'avg_us':>9s} {'total_ms':>9s} {'share':>6s}")
    for (name, grid), (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {grid:16s} {n:5d} {ns / n / 1e3:9.1f} {ns / 1e6:9.2f} {100 * ns / total:5.1f}%")
    print(f"total {total / 1e6:.2f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
