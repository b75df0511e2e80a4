#!/bin/bash
run() { echo "=== $*"; env "$@" python bench.py --no-e2e --no-cpu --no-clocks --steps 200 > gpurun_out/sweep.json 2>gpurun_out/sweep.err || tail -3 gpurun_out/sweep.err; python scripts/show_bench.py gpurun_out/sweep.json 2>/dev/null | sed -n '1p;3,8p;10,11p'; }
run CGVK_PDL=1
run CGVK_PDL=0
run CGVK_SMEM_CTAS_SPMV=2
run CGVK_SMEM_CTAS_SPMV=2 CGVK_PDL=0
