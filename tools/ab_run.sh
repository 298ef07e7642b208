mkdir -p gpurun_out
bash tools/ab_libs.sh 0,5,6 6 > gpurun_out/ab_nt64.txt 2>&1
for L in libelas.so libt_p6nt64.so; do ELAS_LIBNAME=$L timeout 300 python tools/ab_cfg5.py 4 2>&1 | tail -1; done >> gpurun_out/ab_nt64.txt
cat gpurun_out/ab_nt64.txt
