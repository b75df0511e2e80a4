"""Per-source-line stall attribution of an ncu report (SASS rows correlated to
CUDA lines, summed per line). usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
acc, srcs, fname, H = defaultdict(float), {}, None, None
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; H = None; continue
    if r and r[0] == "Line No":
        H = r; iw = H.index("Warp Stall Sampling (All Samples)"); continue
    if H and len(r) == len(H):
        try:
            acc[(fname, r[0])] += float(r[iw] or 0)
            srcs[(fname, r[0])] = r[1].strip()
        except ValueError:
            pass
tot = sum(acc.values()) or 1
for k, v in sorted(acc.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*v/tot:5.1f}%  {k[0]}:{k[1]}  {srcs[k][:100]}")
