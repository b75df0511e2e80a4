# band-engine A/B on R4M: every build_ab/*.so (scripts/build_ab.sh), then env knobs
AB_STEPS=100 bash scripts/ab.sh r4m
run() { echo "=== $*"; env "$@" timeout 300 python bench.py --no-e2e --no-cpu --no-clocks --steps 100 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err; python scripts/show_bench.py gpurun_out/ab.json 2>/dev/null | sed -n '1p;3,8p'; }
run BENCH_CONFIG=r4m CGVK_BAND_NSTAGE=3
run BENCH_CONFIG=r4m CGVK_BAND_PF=1
