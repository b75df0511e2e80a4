#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv` launch list: per-kernel launch count, mean and
total device time, each kernel's share of the solver-loop time (cold-cache,
serialised: compare SHARES), and the measured DRAM bytes per launch.

usage: summarize_launches.py launches.csv [traffic.json config]
With more arguments, merges {config: {bench kernel name: DRAM bytes per
launch}} (median over launches) into traffic.json for bench.py's
roofline.traffic."""
import collections
import csv
import json
import statistics
import sys

# k_stream / k_band Op -> bench.py kernel name
OPS = {"HsK1": "hs_k1", "HsK2": "hs_k2", "CgK1": "cg_k1", "CgK2": "cg_k2", "PrK1": "pr_k1",
       "PrK2": "pr_k2", "GvK1": "gv_k1", "GvK2": "gv_k2", "PprK1": "ppr_k1", "PprK2": "ppr_k2",
       "PrF": "pr_f", "CgF": "cg_f", "GvF": "gv_f"}  # (one kernel per iteration)
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}


def main(path, traffic_out=None, config=None):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, ni, ui, mi = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    launches = collections.defaultdict(dict)  # (id) -> {metric: value}
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= mi:
            continue
        val = float(r[mi].replace(",", "")) * SCALE.get(r[ui], 1)
        launches[r[0]][r[ni]] = val
        names[r[0]] = r[ki]
    agg = collections.defaultdict(list)
    for lid, m in launches.items():
        name = names[lid].replace("cgvk::", "").replace("(bool)1", "1").replace("(bool)0", "0")
        name = name.replace("<1>", "<jacobi>").replace("<0>", "<none>")
        name = name.split("(Params")[0].replace("void ", "")
        agg[name].append(m)
    # the engines' standalone SpMV (SpmvOp: r0 = b - A x0, the true residual,
    # bench.py's spmv timing) runs outside the solver loop
    loop = {k for k in agg if ("k_stream" in k or "k_band" in k) and "SpmvOp" not in k}
    tot_loop = sum(m.get("gpu__time_duration.sum", 0) for k in loop for m in agg[k])
    print("| kernel | launches | mean us | total us | share of solver loop | DRAM MB/launch |")
    print("|---|---:|---:|---:|---:|---:|")
    traffic = {}
    for k, ms in sorted(agg.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
        t = [m.get("gpu__time_duration.sum", 0) for m in ms]
        share = f"{100 * sum(t) / tot_loop:.1f} %" if k in loop else "outside loop"
        dram = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in ms
                if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m]
        dcol = f"{statistics.median(dram) / 1e6:.1f}" if dram else "-"
        print(f"| `{k}` | {len(ms)} | {sum(t) / len(t):.1f} | {sum(t):.1f} | {share} | {dcol} |")
        if dram and k in loop and "jacobi" in k:
            op = k.split("<", 1)[1].split("<", 1)[0]
            if op in OPS:
                traffic[OPS[op]] = statistics.median(dram)
    if traffic_out:
        try:
            with open(traffic_out) as f:
                allcfg = json.load(f)
        except (OSError, ValueError):
            allcfg = {}
        allcfg[config] = traffic
        with open(traffic_out, "w") as f:
            json.dump(allcfg, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:4] if len(sys.argv) > 3 else ()))
