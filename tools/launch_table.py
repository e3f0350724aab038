"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name, count and total/mean duration; optionally only the last K launches."""
import collections
import csv
import sys


def rows(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rd = csv.DictReader(lines[start:])
    for r in rd:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            yield r


def main():
    path = sys.argv[1]
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rs = list(rows(path))
    if last:
        rs = rs[-last:]
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rs:
        name = r["Kernel Name"]
        short = name.split("(")[0][:70] + " " + r.get("Grid Size", "")
        v = float(r["Metric Value"])
        unit = r["Metric Unit"]
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000.0)
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
        tot += us
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:5d} {us:10.1f} us {us / c:9.2f} us/launch {100 * us / tot:5.1f}%  {k}")
    print(f"total {tot:.1f} us over {len(rs)} launches")


if __name__ == "__main__":
    main()
