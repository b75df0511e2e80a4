set -u
OUT=gpurun_out/p2p
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_p2p.py -x -q > $OUT/p2p_tests.log 2>&1; echo "p2p tests rc=$?"
timeout 600 python -m pytest tests/test_gpu_group.py tests/test_gpu_variants.py -x -q > $OUT/group_tests.log 2>&1; echo "group tests rc=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py --config p128 --per-config "" --steps 200 --no-e2e --no-cpu > $OUT/bench_p128.json 2>$OUT/bench_p128.err; echo "bench p128 rc=$?"
for P in 2 4 8; do
  timeout 300 python bench.py --config p64 --per-config "" --emulate-ranks $P --steps 200 --no-e2e --no-cpu --no-clocks > $OUT/p64_copy_$P.json 2>$OUT/p64_copy_$P.err; echo "p64 copy $P rc=$?"
  timeout 300 python bench.py --config p64 --per-config "" --emulate-ranks $P --p2p --steps 200 --no-e2e --no-cpu --no-clocks > $OUT/p64_p2p_$P.json 2>$OUT/p64_p2p_$P.err; echo "p64 p2p $P rc=$?"
done
timeout 300 python bench.py --config p64 --per-config "" --steps 200 --no-e2e --no-cpu --no-clocks > $OUT/p64_1.json 2>$OUT/p64_1.err; echo "p64 1 rc=$?"
