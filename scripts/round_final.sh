#!/bin/bash
# End-of-round measurement on one B200: the driver's bench line (P128 with the
# V256 / R4M per_config lines), bench lines of P64 / P2D, ncu launch lists
# (time + DRAM bytes per launch) for P128 / R4M / P64 / V256, and `ncu --set
# full` captures of the top kernels. Each ncu command runs only after the same
# command exited 0 without ncu.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_driver.json 2> $OUT/bench_driver.err; echo "bench driver rc=$?"
for c in p64 p2d; do
  python bench.py --config $c --per-config "" > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"
done
for c in ${LAUNCH_CFGS:-p128 r4m p64 v256 p2d}; do
  CMD=(python bench.py --config $c --per-config "" --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks)
  "${CMD[@]}" > $OUT/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k 'regex:k_stream|k_band' --csv --log-file $OUT/launches_$c.csv "${CMD[@]}" > $OUT/ncu_l_$c.log 2>&1
  echo "launches $c rc=$?"
done
full() {  # config, kernel regex, name   (ONLY_FULL=name: just that capture)
  [ -n "${ONLY_FULL:-}" ] && [ "${ONLY_FULL}" != "$3" ] && return
  local CMD=(python bench.py --config $1 --per-config "" --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks)
  "${CMD[@]}" > $OUT/plain_full_$3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$2" -s 2 -c 1 -o $OUT/full_$3 "${CMD[@]}" > $OUT/ncu_f_$3.log 2>&1
  echo "full $3 rc=$?"
  # the report itself is too large to bring back: its raw and source pages
  ncu -i $OUT/full_$3.ncu-rep --page raw --csv > $OUT/full_$3.raw.csv 2>/dev/null
  ncu -i $OUT/full_$3.ncu-rep --page source --csv --print-source sass > $OUT/full_$3.sass.csv 2>/dev/null
  python scripts/ncu_summary.py $OUT/full_$3.ncu-rep 30 > $OUT/full_$3.summary.txt 2>&1
  gzip -f $OUT/full_$3.sass.csv
  rm -f $OUT/full_$3.ncu-rep
}
full p128 'k_stream<cgvk::GvK1<\(bool\)1>' p128_gvk1
full r4m 'k_band(_nr)?<cgvk::HsK2<\(bool\)1>' r4m_band_hsk2
full r4m 'k_band(_nr)?<cgvk::PrK2<\(bool\)1>' r4m_band_prk2
full p64 'k_stream<cgvk::PrF<\(bool\)1>' p64_prf
