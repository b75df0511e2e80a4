#!/bin/bash
# Peer-memory transport on one GPU: correctness, then emulated P64 ranks for
# the copy / peer transports and the gpu-scope A/B build.
set -u
OUT=gpurun_out/p2p
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_p2p.py -x -q > $OUT/p2p_tests.log 2>&1; echo "p2p tests rc=$?"
b() { timeout 300 python bench.py --config ${CFG:-p64} --per-config "" --steps 200 --no-e2e --no-cpu --no-clocks "$@"; }
for P in ${RANKS:-2 8}; do
  b --emulate-ranks $P > $OUT/copy_$P.json 2>$OUT/copy_$P.err; echo "copy $P rc=$?"
  b --emulate-ranks $P --p2p > $OUT/p2p_$P.json 2>$OUT/p2p_$P.err; echo "p2p $P rc=$?"
  CGVK_LIB=$PWD/build_ab/libcgvk_gpuscope.so b --emulate-ranks $P --p2p > $OUT/p2pgpu_$P.json 2>$OUT/p2pgpu_$P.err; echo "p2p gpu-scope $P rc=$?"
done
