"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total device time and share."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    r = csv.reader(lines)
    head = next(r)
    agg = collections.OrderedDict()
    n = 0
    for row in r:
        d = dict(zip(head, row))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        n += 1
        us = float(d["Metric Value"]) * SCALE.get(d["Metric Unit"], 1.0)
        a = agg.setdefault(d["Kernel Name"].split("(")[0][:70], [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{path}: {n} launches, {tot / 1e3:.3f} ms device time (cold-cache, serialised)")
    print(f"{'launches':>8} {'total_us':>12} {'share':>6}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t:12.1f} {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
