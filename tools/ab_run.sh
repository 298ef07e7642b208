mkdir -p gpurun_out
bash tools/ab_libs.sh 0,5,6 2 3 4 5 6 7 8 > gpurun_out/ab_ldc.txt 2>&1
for L in libelas.so libt_m31.so libt_m29.so libt_m26.so; do ELAS_LIBNAME=$L timeout 300 python tools/ab_cfg5.py 4 2>&1 | tail -1; done >> gpurun_out/ab_ldc.txt
cat gpurun_out/ab_ldc.txt
