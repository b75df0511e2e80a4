#!/bin/bash
run() { echo "=== $*"; env "$@" timeout 300 python bench.py --no-e2e --no-cpu --no-clocks --steps 200 > gpurun_out/sweep.json 2>gpurun_out/sweep.err || tail -3 gpurun_out/sweep.err; python scripts/show_bench.py gpurun_out/sweep.json 2>/dev/null | sed -n '1p;3,8p'; }
for c in p128 p64 p2d; do
run CGVK_PERSIST=0 BENCH_CONFIG=$c
run CGVK_PERSIST=1 BENCH_CONFIG=$c
done
