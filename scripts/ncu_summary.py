"""Summarise an ncu report: key throughput metrics, stall reasons and the
hottest SASS lines. usage: python scripts/ncu_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for r in rows[2:]:
    print("----")
    for k in KEYS:
        if k in h:
            print(f"{k:60s} {r[h.index(k)]}")
    st = []
    for i, x in enumerate(h):
        if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), x[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hdr]
data = [r for r in rows[hdr + 1:] if len(r) == len(h)]
iw = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iw] or 0) for r in data) or 1
idx = sorted(range(len(data)), key=lambda k: -float(data[k][iw] or 0))[:top]
print("hot SASS:")
for k in sorted(idx):
    print(f"  {k:5d} {100*float(data[k][iw])/tot:5.1f}%  {data[k][h.index('Source')][:100]}")
