#!/bin/bash
# One ncu --set full capture of the fused apply kernel at config 4, degree $1 (AUTO variant),
# written to gpurun_out/ncu_p$1.ncu-rep (+ a raw csv page).  Usage: bash tools/ncu_capture.sh P [KREGEX]
set -u
mkdir -p gpurun_out
P=$1
K=${2:-regex:apply_}
ARGS="--config 4 --p $P --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --e2e-steps 1"
timeout 300 python bench.py $ARGS > gpurun_out/plain_p$P.json 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 3 -c 1 -o gpurun_out/ncu_p$P -f \
    python bench.py $ARGS > gpurun_out/ncu_p$P.log 2>&1
echo "ncu p=$P rc=$?"
ncu -i gpurun_out/ncu_p$P.ncu-rep --page raw --csv > gpurun_out/ncu_p$P.raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_p$P.ncu-rep --page source --csv > gpurun_out/ncu_p$P.src.csv 2>/dev/null
