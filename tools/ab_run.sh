mkdir -p gpurun_out
bash tools/ab_libs.sh 0,5,6 3 4 5 6 7 8 > gpurun_out/ab_ctab4.txt 2>&1
for L in libelas.so libt_ct8.so libt_ct9.so; do ELAS_LIBNAME=$L timeout 300 python tools/ab_cfg5.py 4 2>&1 | tail -1; done
cat gpurun_out/ab_ctab4.txt
