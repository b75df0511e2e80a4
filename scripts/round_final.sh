#!/bin/bash
# End-of-round measurement on one B200: bench lines for every config, ncu
# launch lists (time + DRAM bytes per launch) for P128 / R4M / P64, and one
# `ncu --set full` capture of P128's longest kernels. Each ncu command runs
# only after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
for c in p128 v256 r4m p64 p2d; do
  python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"
done
for c in ${LAUNCH_CFGS:-p128 r4m p64 v256}; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks"
  $CMD > $OUT/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k_stream|k_band" --csv --log-file $OUT/launches_$c.csv $CMD > $OUT/ncu_l_$c.log 2>&1
  echo "launches $c rc=$?"
done
CMD="python bench.py --config p128 --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks"
for k in ${FULL_KERNELS:-"GvK1<\(bool\)1>" "HsK2<\(bool\)1>"}; do
  n=$(echo $k | cut -c1-4 | tr 'A-Z' 'a-z')
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"k_stream<cgvk::$k" -s 2 -c 1 -o $OUT/full_p128_$n $CMD > $OUT/ncu_f_$n.log 2>&1
  echo "full $n rc=$?"
done
