"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name.
   python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
        name = r[ki].split("(")[0]
        tot[name] += ms
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg us':>9s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.3f} {100 * v / s:6.1f}% {1e3 * v / cnt[k]:9.2f}")
    print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {s:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
