#!/bin/bash
# one bench line per tuning configuration (run on the GPU box)
for cfg in "CGVK_PDL=1" "CGVK_PDL=0" "CGVK_PDL=1 CGVK_NSTAGE_SPMV=2" "CGVK_PDL=1 CGVK_SMEM_CTAS=1"; do
  echo "=== $cfg"
  env $cfg python bench.py --no-e2e --no-cpu --no-clocks --steps 100 > gpurun_out/sweep.json 2>gpurun_out/sweep.err || tail -3 gpurun_out/sweep.err
  python scripts/show_bench.py gpurun_out/sweep.json | head -8
done
