#!/bin/bash
# one bench line per tuning configuration (run on the GPU box)
for cfg in "CGVK_SPMV_ENGINE=staged" "CGVK_SPMV_ENGINE=staged CGVK_NSTAGE_SPMV=2" "CGVK_SPMV_ENGINE=staged CGVK_NSTAGE_SPMV=2 CGVK_SMEM_CTAS=3" "CGVK_SPMV_ENGINE=staged CGVK_NSTAGE_SPMV=3 CGVK_SMEM_CTAS=1" "CGVK_SPMV_ENGINE=sell"; do
  echo "=== $cfg"
  env $cfg python bench.py --no-e2e --no-cpu --no-clocks --steps 100 > gpurun_out/sweep.json 2>gpurun_out/sweep.err || tail -3 gpurun_out/sweep.err
  python scripts/show_bench.py gpurun_out/sweep.json
done
