#!/bin/bash
# Copy a round_final.sh result (gpurun_out/final) into profiles/<round>/ under
# the names profiles/README.md lists, and refresh profiles/traffic.json.
set -eu
R=${1:-r02}
F=gpurun_out/final
D=profiles/$R
mkdir -p $D
cp $F/bench_driver.json $D/bench_p128_k20.json
for c in p64 p2d; do cp $F/bench_$c.json $D/bench_$c.json; done
for c in p128 r4m p64 v256 p2d; do
  [ -f $F/launches_$c.csv ] || continue
  cp $F/launches_$c.csv $D/launches_$c.csv
  python scripts/summarize_launches.py $F/launches_$c.csv profiles/traffic.json $c > $D/launches_$c.md
done
for k in p128_gvk1 r4m_band_hsk2 r4m_band_prk2 p64_prf; do
  [ -f $F/full_$k.summary.txt ] || continue
  cp $F/full_$k.summary.txt $D/ncu_full_$k.txt
  cp $F/full_$k.sass.csv.gz $D/ncu_full_$k.sass.csv.gz
done
echo "published into $D"
