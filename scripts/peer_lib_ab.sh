#!/bin/bash
# Emulated ranks (in-process, one GPU) with A/B library builds:
# bash scripts/peer_lib_ab.sh "cfg ..." "ranks ..." lib ...   ("intree" = the in-tree build)
set -u
cfgs=$1; ranks=$2; shift 2
mkdir -p gpurun_out/peer
for c in $cfgs; do for P in $ranks; do for l in "$@"; do
  L=build_ab/libcgvk_$l.so; [ "$l" = intree ] && L=paper_1905_01549_b200/libcgvk.so
  CGVK_LIB=$L timeout 200 python bench.py --config $c --emulate-ranks $P --per-config "" --no-e2e --no-cpu --no-clocks --steps ${AB_STEPS:-200} > gpurun_out/peer/${c}_${P}_$l.json 2> gpurun_out/peer/${c}_${P}_$l.err || tail -3 gpurun_out/peer/${c}_${P}_$l.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/peer/${c}_${P}_$l.json").read().strip().splitlines()[-1])
print("== $c ranks=$P $l", d["config"].get("transport"), "| us per rank-iteration:", {v: round(p["us_per_iter"]/$P,1) for v,p in d["per_variant"].items()})
PY
done; done; done
