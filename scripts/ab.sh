#!/bin/bash
# A/B sweep: every build_ab/*.so (and the in-tree build) on the given configs.
# usage: bash scripts/ab.sh "p128 r4m" [extra env assignments...]
cfgs=${1:-p128}; shift
run() { echo "=== $*"; env BENCH_PER_CONFIG= "$@" timeout 300 python bench.py --no-e2e --no-cpu --no-clocks --steps ${AB_STEPS:-100} > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err; python scripts/show_bench.py gpurun_out/ab.json 2>/dev/null | sed -n '1p;3,8p'; }
for c in $cfgs; do
  for lib in build_ab/*.so; do run CGVK_LIB=$PWD/$lib BENCH_CONFIG=$c "$@"; done
done
