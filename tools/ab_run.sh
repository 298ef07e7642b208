mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined or config5 or config4 or launches or apply_host or dirichlet" > gpurun_out/pz_tests.log 2>&1; tail -3 gpurun_out/pz_tests.log
bash tools/ab_libs.sh 0 2 4 6 > gpurun_out/ab_ic.txt 2>&1
for L in libelas.so libt_ic1.so libt_ic16.so libelas.so libt_ic1.so; do ELAS_LIBNAME=$L timeout 300 python tools/ab_cfg5.py 4 2>&1 | tail -1; done >> gpurun_out/ab_ic.txt
cat gpurun_out/ab_ic.txt
