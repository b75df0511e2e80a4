#!/bin/bash
# One-call health check on one B200: the GPU test suite, smoke(), the bench
# line at the driver's settings, and the ncu launch list of a short P128 run
# (after the same command exits 0). SKIP_TESTS=1 skips the test suite.
set -u
OUT=gpurun_out/check
mkdir -p $OUT
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?"
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_k20.json 2> $OUT/bench_k20.err; echo "bench k20 rc=$?"
if [ -z "${SKIP_LAUNCHES:-}" ]; then
  CMD=(python bench.py --config p128 --per-config "" --steps 3 --warmup 3 --no-e2e --no-cpu --no-clocks)
  timeout 300 "${CMD[@]}" > $OUT/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k 'regex:k_stream|k_band' --csv --log-file $OUT/launches_p128.csv "${CMD[@]}" > $OUT/ncu_l.log 2>&1
  echo "launches rc=$?"
fi
