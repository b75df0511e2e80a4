#!/bin/bash
# Peer-memory transport on one GPU: correctness, then emulated ranks (P64 /
# P128 z-slabs) for the copy and peer transports (bench's auto ladder).
set -u
OUT=gpurun_out/p2p
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_p2p.py -x -q > $OUT/p2p_tests.log 2>&1; echo "p2p tests rc=$?"
b() { timeout 300 python bench.py --per-config "" --steps 200 --no-e2e --no-cpu --no-clocks "$@"; }
for C in ${CFGS:-p64}; do
for P in ${RANKS:-2 8}; do
  b --config $C --emulate-ranks $P --transport copy > $OUT/${C}_copy_$P.json 2>$OUT/${C}_copy_$P.err; echo "$C copy $P rc=$?"
  b --config $C --emulate-ranks $P > $OUT/${C}_auto_$P.json 2>$OUT/${C}_auto_$P.err; echo "$C auto $P rc=$?"
done
done
