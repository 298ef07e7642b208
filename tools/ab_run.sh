mkdir -p gpurun_out
bash tools/ab_libs.sh 0,5,6 3 4 5 2>&1
ELAS_LIBNAME=libt_r3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "folded_variant or all_degrees or folded_f32_vs or otf_vs" 2>&1 | tail -1
