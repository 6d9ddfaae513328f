#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import sys
from collections import defaultdict


def main(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000 if unit == "ns" else (v if unit in ("us", "usecond") else v * 1000)
        if k not in agg:
            order.append(k)
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':70s} {'n':>4s} {'total_us':>11s} {'avg_us':>10s} {'share':>6s}")
    for k in sorted(order, key=lambda k: -agg[k][1]):
        n, t = agg[k]
        print(f"{k[:70]:70s} {n:4d} {t:11.1f} {t / n:10.1f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
