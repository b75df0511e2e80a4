#!/bin/bash
# One-kernel PR / M iteration (PrF) against the two-kernel schedule on the
# L2-resident configs. LIBS = A/B builds under build_ab/ ("" = the in-tree
# library); each is first checked bit-exact on a quick test subset (hard
# timeouts everywhere: a wrong barrier hangs the GPU).
set -u
OUT=gpurun_out/fuse
mkdir -p $OUT
run() {  # name, env...
  local name=$1; shift
  for c in ${CFGS:-p64 p2d}; do
    env "$@" timeout 120 python bench.py --config $c --per-config "" --no-e2e --no-cpu --no-clocks --steps ${AB_STEPS:-200} > $OUT/b_${c}_$name.json 2> $OUT/b_${c}_$name.err || tail -3 $OUT/b_${c}_$name.err
    echo "== $c $name: $(python scripts/show_bench.py $OUT/b_${c}_$name.json | grep -E '^(m|pr) ' | tr '\n' ' ')"
  done
}
run unfused CGVK_FUSE=0
run fused CGVK_FUSE=1
for l in ${LIBS:-}; do
  L=build_ab/libcgvk_$l.so
  CGVK_LIB=$L timeout 300 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -m gpu -x -q > $OUT/t_$l.log 2>&1
  echo "tests $l rc=$? $(tail -1 $OUT/t_$l.log)"
  if tail -1 $OUT/t_$l.log | grep -q passed; then run $l CGVK_LIB=$L; fi
done
if [ -n "${FULL_TESTS:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$? $(tail -1 $OUT/gpu_tests.log)"
fi
