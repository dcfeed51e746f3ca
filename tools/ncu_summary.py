"""Summarise an ncu raw CSV (+ optional SASS source CSV): key throughput
metrics, stall reasons, top stalled instructions.
   python tools/ncu_summary.py raw.csv [src.csv]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for k in keys:
    if k in d:
        print(f"{k:80s} {d[k]}")
st = []
for k, v in d.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
print("stalls per issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
if len(sys.argv) > 2:
    rows = list(csv.reader(open(sys.argv[2])))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[i_s] or 0) for r in data if len(r) > i_s)
    for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:15]:
        print(f"{float(r[i_s]) / tot * 100:5.1f}%  {r[1][:100]}")
