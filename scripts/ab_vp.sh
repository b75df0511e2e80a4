# virtual-CTA count A/B (CSR engine configs)
run() { echo "=== $*"; env "$@" timeout 300 python bench.py --no-e2e --no-cpu --no-clocks --steps 100 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err; python scripts/show_bench.py gpurun_out/ab.json 2>/dev/null | sed -n '1p;3,8p'; }
L=$PWD/build_ab/libcgvk_k1m3.so
for c in ${CFGS:-p128 v256 p64 p2d}; do
  run BENCH_CONFIG=$c
  run BENCH_CONFIG=$c CGVK_LIB=$L CGVK_VPERSM=3 CGVK_SMEM_CTAS=3
  run BENCH_CONFIG=$c CGVK_LIB=$L CGVK_VPERSM=6 CGVK_SMEM_CTAS=3
  run BENCH_CONFIG=$c CGVK_VPERSM=3 CGVK_SMEM_CTAS=3
done
