timeout 300 python -m pytest tests/test_precond_gpu.py -x -q -k fused > gpurun_out/s8_fused.log 2>&1; echo "fused rc=$?" >> gpurun_out/s8_fused.log
timeout 300 python tools/time_fused.py > gpurun_out/s8_time.txt 2>&1
FMP_NO_PDL_VEC=1 timeout 300 python tools/time_fused.py > gpurun_out/s8_time_nopdlvec.txt 2>&1
bash tools/ab_bench.sh FMP_NO_FUSED_LINCOMB "1 0 1 0" 10 > gpurun_out/s8_ab.txt 2>&1
bash tools/ab_bench.sh FMP_NO_PDL_VEC "1 0" 10 > gpurun_out/s8_ab_vec.txt 2>&1
