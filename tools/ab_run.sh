mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ctab.log 2>&1; tail -2 gpurun_out/pytest_ctab.log
for L in libelas.so libt_noct.so; do ELAS_LIBNAME=$L timeout 300 python tools/ab_aniso.py 2 3 4 2>&1 | tail -1; done
