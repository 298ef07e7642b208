#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, the default bench line, the ncu launch
# list of the bench workload and one full capture of the dominant kernel (config 5).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
ARGS="--steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-solver --e2e-steps 1"
timeout 900 python bench.py $ARGS > gpurun_out/ncu_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:apply_ -s 3 -c 1 -o gpurun_out/ncu_cfg5_eo -f \
    python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; head -c 400 gpurun_out/bench.json; tail -1 gpurun_out/ncu_full.log
