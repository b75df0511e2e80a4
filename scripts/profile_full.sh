#!/bin/bash
# One `ncu --set full` capture of one kernel (regex on the demangled name) in
# a short bench run, after the same command has exited 0 without ncu.
# usage: BENCH_CONFIG=p128 bash scripts/profile_full.sh 'HsK2<\(bool\)1>' name
set -u
OUT=gpurun_out
CFG=${BENCH_CONFIG:-p128}
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks"
$CMD > $OUT/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$1" -s 2 -c 1 -o $OUT/$2 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
