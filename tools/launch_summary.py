"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py launches.csv [header line]
Prints us/launch, launch count and share of the listed device time per kernel,
largest share first (the format of profiles/r*_launches_summary.txt).
"""
import csv
import sys
from collections import defaultdict


def summarise(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r["Metric Unit"]
            us = v / 1000.0 if unit == "ns" else v * 1000.0 if unit == "ms" else v
            rows.append((r["Kernel Name"], us))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for k, us in rows:
        tot[k] += us
        cnt[k] += 1
    all_us = sum(tot.values()) or 1.0
    out = []
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"{tot[k] / cnt[k]:9.1f} us/launch {cnt[k]:4d} launches {100 * tot[k] / all_us:5.1f}%  {k[:70]}")
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print("\n".join(summarise(sys.argv[1])))
