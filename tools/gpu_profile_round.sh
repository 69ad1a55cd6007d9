#!/bin/bash
# One round's profile set (run under gpurun from the repo root): launch lists of one step / one
# apply / the bench command, and ncu --set full of one launch of each hot kernel.  TAG names files.
tag=${1:-vXX}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "measure/" --csv \
  --log-file gpurun_out/launch_step_$tag.csv python tools/prof_step.py > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "measure/" --csv \
  --log-file gpurun_out/launch_prec_$tag.csv python tools/prof_precond.py > /dev/null 2>&1
bash tools/ncu_full.sh $tag k_plane_fast k_faces k_ozaki k_corr k_spmv_bulk k_ozaki_slice_rows
for s in 0 1; do
  timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "measure/" \
    -k regex:k_column_fast_db --launch-skip $s -c 1 -o gpurun_out/${tag}_col$s -f python tools/prof_precond.py > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "measure/" \
  -k regex:k_plane_fast --launch-skip 1 -c 1 -o gpurun_out/${tag}_plane_inv -f python tools/prof_precond.py > /dev/null 2>&1
ls gpurun_out | grep $tag
