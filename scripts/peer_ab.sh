#!/bin/bash
# One-kernel PR / M iteration on peer-memory ranks: the p2p / group GPU tests,
# then emulated ranks (in-process, one GPU) with CGVK_FUSE_PEER=0 / 1.
set -u
OUT=gpurun_out/peer
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_group.py -m gpu -x -q > $OUT/tests.log 2>&1; echo "p2p tests rc=$? $(tail -1 $OUT/tests.log)"
for c in ${CFGS:-p64}; do for P in ${RANKS:-8 2}; do for f in 0 1; do
  CGVK_FUSE_PEER=$f timeout 200 python bench.py --config $c --emulate-ranks $P --per-config "" --no-e2e --no-cpu --no-clocks --steps ${AB_STEPS:-100} > $OUT/b_${c}_${P}_$f.json 2> $OUT/b_${c}_${P}_$f.err || tail -3 $OUT/b_${c}_${P}_$f.err
  python - <<PY
import json
d=json.loads(open("$OUT/b_${c}_${P}_$f.json").read().strip().splitlines()[-1])
print("== $c ranks=$P fuse_peer=$f transport", d["config"].get("transport"), "| us per rank-iteration:", {v: round(p["us_per_iter"]/$P,1) for v,p in d["per_variant"].items()})
PY
done; done; done
