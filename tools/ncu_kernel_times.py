"""Mean duration per (grid, kernel) of an ncu --csv launch list on stdin
(--metrics gpu__time_duration.sum), skipping the first `skip` launches of
each (warm-up).  usage: ncu ... --csv python x.py | python ncu_kernel_times.py [skip]"""
import collections
import csv
import sys


def main():
    skip = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    lines = [l for l in sys.stdin if l.startswith('"')]
    d = collections.OrderedDict()
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        us = v / 1000.0 if r["Metric Unit"] in ("nsecond", "ns") else v
        d.setdefault(r["Grid Size"] + " " + r["Kernel Name"].split("(")[0][-60:], []).append(us)
    for k, v in d.items():
        w = v[skip:] or v
        print(f"{sum(w) / len(w):10.2f} us  x{len(v):3d}  {k}")


if __name__ == "__main__":
    main()
