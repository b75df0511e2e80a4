set -u
OUT=gpurun_out/e2e; mkdir -p $OUT
for o in concurrent chained; do
 for r in 1 2; do
  timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --per-config "" --no-cpu --e2e-order $o --e2e-reps 3 > $OUT/e2e_${o}_$r.json 2>$OUT/e2e_${o}_$r.err; echo "$o $r rc=$?"
 done
done
