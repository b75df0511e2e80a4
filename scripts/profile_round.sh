#!/bin/bash
# Round measurement on one B200 (call 1 of 2): the default bench line, then the
# ncu launch list of a short run of the same command with per-launch time and
# DRAM bytes (cold-cache, serialised). Only after the plain command exits 0.
# Call 2 (one ncu --set full capture of the top kernel) is profile_full.sh.
set -u
OUT=gpurun_out
CFG=${BENCH_CONFIG:-p128}
python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_stream|k_band" --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu1.log 2>&1
echo "ncu launches rc=$?"
