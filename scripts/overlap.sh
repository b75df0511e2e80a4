#!/bin/bash
# Reduction/SpMV overlap of the row-partitioned path, measured on one GPU
# through a one-rank NCCL communicator (real NCCL AllGather + finalize per
# reduction): CGVK_GROUP_OVERLAP=1 (GV / pipe-PR exchange their reduction
# beside K2) vs 0 (serialised), next to the plain single-GPU solve.
for cfg in p64 p128; do
  for mode in plain nccl_overlap nccl_serial; do
    case $mode in
      plain) python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ov_${cfg}_plain.json 2>/dev/null ;;
      nccl_overlap) CGVK_GROUP_OVERLAP=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --nccl --config $cfg --steps 200 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ov_${cfg}_$mode.json 2>/dev/null ;;
      nccl_serial) CGVK_GROUP_OVERLAP=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 1 --nccl --config $cfg --steps 200 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ov_${cfg}_$mode.json 2>/dev/null ;;
    esac
    python - "$cfg" "$mode" <<'PY'
import json, sys
cfg, mode = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/ov_{cfg}_{mode}.json").read().strip().splitlines()[-1])
print(cfg, mode, " ".join(f"{v}:{x['us_per_iter']:.1f}" for v, x in d["per_variant"].items()))
PY
  done
done
# the partitioned data path with P in-process ranks on one GPU (halo copies,
# rank-ordered finalize; no NCCL): per-iteration cost of partitioning
for cfg in p64 p128; do
  for P in 2 4 8; do
    python bench.py --config $cfg --emulate-ranks $P --steps 100 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ov_${cfg}_emu$P.json 2>/dev/null
    python - "$cfg" "$P" <<'PY'
import json, sys
cfg, P = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/ov_{cfg}_emu{P}.json").read().strip().splitlines()[-1])
print(cfg, f"emulated_{P}_ranks", " ".join(f"{v}:{x['us_per_iter']:.1f}" for v, x in d["per_variant"].items()))
PY
  done
done
