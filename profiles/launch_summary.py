"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`):
total time, share and launch count per kernel name.

usage: python profiles/launch_summary.py launches.csv "<title line>"
"""
import collections
import csv
import sys


def main(path, title):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit")
        if unit in ("ns", "nsecond"):
            v /= 1e3
        elif unit in ("ms", "msecond"):
            v *= 1e3
        tot[r["Kernel Name"]] += v
        cnt[r["Kernel Name"]] += 1
    s = sum(tot.values())
    print(title)
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {v:10.1f} us  {100 * v / s:5.1f}%  {cnt[k]:5d} launches  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
