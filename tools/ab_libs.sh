#!/bin/bash
# Run tools/ab_variants.py (variants $1, degrees $2...) against every lib/libt_*.so and libelas.so.
V=$1; shift
for L in libelas.so $(cd paper_2601_08374_b200/lib && ls libt_*.so); do
  ELAS_LIBNAME=$L timeout 300 python tools/ab_variants.py $V "$@" 2>&1 | tail -1
done
