# A/B: in-tree build vs build_ab/*.so on several configs
# usage: bash scripts/ab_cfgs.sh "p128 p64" [lib ...]
cfgs=${1:-p128}; shift
run() { echo "=== $*"; env "$@" timeout 300 python bench.py --per-config "" --no-e2e --no-cpu --no-clocks --steps ${AB_STEPS:-100} > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err; python scripts/show_bench.py gpurun_out/ab.json 2>/dev/null | sed -n '1p;3,20p'; }
for c in $cfgs; do
  run BENCH_CONFIG=$c
  for lib in "$@"; do run CGVK_LIB=$PWD/build_ab/libcgvk_$lib.so BENCH_CONFIG=$c; done
done
