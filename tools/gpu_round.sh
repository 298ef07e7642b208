#!/bin/bash
# One gpurun call: full GPU tests, the bench line, the ncu launch list and one full capture.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
if [ "${PYTEST:-1}" = "1" ]; then
  python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
  NARGS="--config 4 --p ${NCU_P:-6} --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --e2e-steps 1"
  python bench.py $NARGS > gpurun_out/ncu_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py $NARGS > gpurun_out/ncu_launch.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:apply_kernel -s 3 -c 1 \
      -o gpurun_out/prof_apply python bench.py $NARGS > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
