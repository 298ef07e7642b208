#!/bin/bash
# Profile the bench workload: plain run, ncu launch list, one full capture of the dominant kernel.
set -u
mkdir -p gpurun_out
ARGS="${BENCH_PROF_ARGS:---steps 3 --warmup 3 --no-sweep --no-cpu-baseline --e2e-steps 1}"
KREGEX="${KREGEX:-regex:apply_}"
python bench.py $ARGS > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "$KREGEX" -s 3 -c 1 -o gpurun_out/prof_bench \
    python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
tail -2 gpurun_out/ncu_full.log
