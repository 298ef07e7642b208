#!/bin/bash
# ncu --set full of the AUTO kernel at config 4 for every p; summaries into gpurun_out/ncu_allp.txt
set -u
mkdir -p gpurun_out
: > gpurun_out/ncu_allp.txt
for P in 1 2 3 4 5 6 7 8; do
  K="regex:apply_"
  timeout 600 ncu --set full --clock-control none --import-source on -k "$K" -s 2 -c 1 -o gpurun_out/ncu_allp_$P -f \
      python tools/run_variant.py $P 0 3 > /dev/null 2>&1
  echo "== p=$P rc=$?" >> gpurun_out/ncu_allp.txt
done
