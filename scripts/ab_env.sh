# A/B of env knobs on the in-tree build: bash scripts/ab_env.sh "p128 p64" "" "VAR=a" "VAR=b OTHER=c" ...
cfgs=$1; shift
run() { echo "=== $*"; env "$@" timeout 300 python bench.py --per-config "" --no-e2e --no-cpu --no-clocks --steps ${AB_STEPS:-100} > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err; python scripts/show_bench.py gpurun_out/ab.json 2>/dev/null | sed -n '1p;3,8p;9,20p'; }
for c in $cfgs; do for kv in "$@"; do run BENCH_CONFIG=$c $kv; done; done
