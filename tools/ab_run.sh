mkdir -p gpurun_out
for L in libelas.so libt_ch32.so libt_ch128.so libelas.so; do ELAS_LIBNAME=$L timeout 300 python tools/e2e_probe.py 2>&1 | tail -1; done
