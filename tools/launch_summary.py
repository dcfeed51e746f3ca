"""Per-kernel totals of one adaptive call from an ncu launch list
(--metrics gpu__time_duration.sum --csv).  The call is delimited by the
scatter_interp launch that ends every rand_lupp_adaptive call; the last
complete call in the capture is summarised.
   python tools/launch_summary.py launches.csv > summary.csv"""
import csv
import re
import sys
from collections import OrderedDict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").strip()
    rows.append((name, ns))
ends = [i for i, (n, _) in enumerate(rows) if "scatter_interp" in n]
starts = [i for i, (n, _) in enumerate(rows) if "iota_kernel" in n]  # TFormState init
lo, hi = 0, len(rows)
if ends:
    hi = ends[-1] + 1
    before = [i for i in starts if i < hi]
    if before:
        lo = before[-1]
        # the call's first sketch blocks (and their Omega draws) precede the init
        while lo > 0 and ("dgemm" in rows[lo - 1][0] or "rng_" in rows[lo - 1][0]) and lo > hi - 20000:
            if "scatter_interp" in rows[lo - 1][0]:
                break
            lo -= 1
            if sum(1 for n, _ in rows[lo:hi] if "rng_attempt" in n) > sum(
                    1 for n, _ in rows[lo:hi] if "panel_kernel" in n) + 3:
                lo += 1
                break
agg = OrderedDict()
for n, ns in rows[lo:hi]:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += ns
tot = sum(a[1] for a in agg.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none; one complete rand_lupp_adaptive call "
      f"(launches {lo}..{hi - 1} of the capture), cold-cache and serialised")
print("kernel,launches,total_ms,share_of_call")
for n, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n},{c},{ns / 1e6:.3f},{ns / tot:.3f}")
print(f"# total {tot / 1e6:.1f} ms over {hi - lo} launches")
