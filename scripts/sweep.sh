#!/bin/bash
for cfg in "CGVK_PDL=1" "CGVK_PDL=1"; do
  echo "=== $cfg"
  env $cfg python bench.py --no-e2e --no-cpu --no-clocks --steps 200 > gpurun_out/sweep.json 2>gpurun_out/sweep.err || tail -3 gpurun_out/sweep.err
  python scripts/show_bench.py gpurun_out/sweep.json 2>/dev/null | head -20
done
