# ncu --set full of one kernel for each build_ab/*.so (A/B evidence)
# usage: BENCH_CONFIG=r4m bash scripts/ab_ncu.sh 'regex' tag
CFG=${BENCH_CONFIG:-r4m}
for lib in build_ab/*.so; do
  n=$(basename $lib .so)
  CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks"
  CGVK_LIB=$PWD/$lib $CMD > gpurun_out/plain_$n.log 2>&1 && \
  CGVK_LIB=$PWD/$lib ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$1" -s 2 -c 1 -o gpurun_out/${2}_$n $CMD > gpurun_out/ncu_$n.log 2>&1
  echo "$n rc=$?"
done
