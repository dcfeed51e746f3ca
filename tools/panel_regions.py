"""Stall-sample share per region of panel_kernel from an ncu source CSV.
   python tools/panel_regions.py panel_src.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
i_e = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data)
marks = []
for k, r in enumerate(data):
    src = r[i_src]
    if "BAR.SYNC" in src or "STG.E.128.STRONG" in src or "LDG.E.128.STRONG" in src:
        marks.append((k, src.strip()[:40]))
prev = 0
acc_s = acc_e = 0.0
for k, r in enumerate(data):
    acc_s += float(r[i_s] or 0)
    acc_e += float(r[i_e] or 0)
    if "BAR.SYNC" in r[i_src]:
        print(f"[{prev:5d},{k:5d}] samples {acc_s / tot * 100:5.1f}%  insts {acc_e:12.0f}  ends at BAR.SYNC")
        prev, acc_s, acc_e = k + 1, 0.0, 0.0
print(f"[{prev:5d},  end] samples {acc_s / tot * 100:5.1f}%  insts {acc_e:12.0f}")
top = sorted(range(len(data)), key=lambda q: -float(data[q][i_s] or 0))[:12]
for q in top:
    print(f"{q:5d} {float(data[q][i_s]) / tot * 100:5.1f}%  {data[q][i_src][:70]}")
