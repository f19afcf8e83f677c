"""Per-kernel share of an ncu `--metrics gpu__time_duration.sum --csv` launch list.

  python tools/launch_share.py launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    t, c = collections.defaultdict(float), collections.Counter()
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            k = r["Kernel Name"].split("(")[0][:60]
            t[k] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
            c[k] += 1
    tot = sum(t.values())
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        print(f"{v / c[k]:9.2f} us x{c[k]:4d} {v / tot * 100:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
