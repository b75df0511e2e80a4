"""Registers / stack / spill per kernel of a built libcgvk.so (cuobjdump), and
a diff of two builds: python scripts/regs.py A.so [B.so]"""
import re
import subprocess
import sys


def usage(so):
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", so], capture_output=True, text=True).stdout
    names, res = [], {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and cur:
            res[cur] = (int(m.group(1)), int(m.group(2)))
            names.append(cur)
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return {d.replace("cgvk::", ""): res[n] for n, d in zip(names, dem) if "k_stream" in d or "k_band" in d}


a = usage(sys.argv[1])
if len(sys.argv) == 2:
    for k in sorted(a):
        print(a[k], k)
else:
    b = usage(sys.argv[2])
    for k in sorted(set(a) | set(b)):
        if a.get(k) != b.get(k):
            print(a.get(k), "->", b.get(k), k[:150])
