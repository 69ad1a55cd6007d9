#!/bin/bash
# ncu --set full of one apply-phase launch of each hot kernel (tools/prof_precond.py, NVTX range
# "measure"), one report per kernel under gpurun_out/.  Usage: tools/ncu_full.sh TAG [kernel-regex...]
tag=$1; shift
ks=${@:-"k_plane_fast k_column_fast_db k_column_fast k_faces k_ozaki k_corr k_spmv"}
for k in $ks; do
  timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "measure/" \
    -k regex:"^${k}\$|${k}<" -c 1 -o gpurun_out/${tag}_${k} -f python tools/prof_precond.py > gpurun_out/${tag}_${k}.log 2>&1
done
