#!/bin/bash
# Round profile on one B200: plain bench (JSON), the ncu launch list of the same
# short command, and one `ncu --set full` capture of the top kernels.
set -u
OUT=gpurun_out
python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu1.log 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"HsK2<1>|PrK2<1>|PprK1<1>|PprK2<1>|GvK1<1>" -s 5 -c 5 -o $OUT/prof_full $CMD > $OUT/ncu2.log 2>&1
echo "ncu full rc=$?"
