mkdir -p gpurun_out
for L in libt_p1s3.so libt_p1s4.so; do ELAS_LIBNAME=$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "p1_variants or config4_full_size and 1 or single_element or all_degrees or pipelined" 2>&1 | tail -1; done
bash tools/ab_libs.sh 0 1 2>&1
