#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, mean and total device time, and each kernel's share
of the solver-loop time (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > mi:
            name = r[ki].replace("cgvk::", "").replace("(bool)1", "jacobi").replace("(bool)0", "none")
            name = name.split("(Params")[0].replace("void ", "")
            agg[name].append(float(r[mi].replace(",", "")) / 1e3)
    loop = {k: v for k, v in agg.items() if "k_stream" in k or "k_direct" in k}
    tot_loop = sum(sum(v) for v in loop.values())
    print("| kernel | launches | mean us | total us | share of solver loop |")
    print("|---|---:|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / tot_loop:.1f} %" if k in loop else "setup"
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {share} |")


if __name__ == "__main__":
    main(sys.argv[1])
