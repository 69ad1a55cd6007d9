python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "measure/" --csv --log-file gpurun_out/launch_step_v24.csv python tools/prof_step.py > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "measure/" --csv --log-file gpurun_out/launch_prec_v24.csv python tools/prof_precond.py > /dev/null 2>&1
bash tools/ncu_full.sh v24 k_plane_fast k_faces k_ozaki k_corr k_spmv_bulk k_ozaki_slice_rows
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "measure/" -k regex:k_plane_fast --launch-skip 1 -c 1 -o gpurun_out/v24_plane_inv -f python tools/prof_precond.py > /dev/null 2>&1
ls gpurun_out | grep v24
