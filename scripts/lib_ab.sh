#!/bin/bash
# A/B of library builds: bash scripts/lib_ab.sh "cfg ..." lib ... ("intree" = the in-tree build)
set -u
cfgs=$1; shift
mkdir -p gpurun_out/lib_ab
for c in $cfgs; do for l in "$@"; do
  L=build_ab/libcgvk_$l.so; [ "$l" = intree ] && L=paper_1905_01549_b200/libcgvk.so
  CGVK_LIB=$L timeout 200 python bench.py --config $c --per-config "" --no-e2e --no-cpu --no-clocks --steps ${AB_STEPS:-200} > gpurun_out/lib_ab/${c}_$l.json 2> gpurun_out/lib_ab/${c}_$l.err || tail -3 gpurun_out/lib_ab/${c}_$l.err
  echo "== $c $l: $(python scripts/show_bench.py gpurun_out/lib_ab/${c}_$l.json | sed -n '1p;3,8p' | awk 'NR==1{printf "%s it/s |", $2} NR>1{printf " %s %s", $1, $2}')"
done; done
