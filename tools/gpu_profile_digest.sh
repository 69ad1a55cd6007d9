#!/bin/bash
# tools/gpu_profile_round.sh TAG plus the digests, run on the GPU box (the .ncu-rep files are too
# large to bring back): launch-list summaries, ncu --set full digest, DRAM traffic and hot SASS
# under gpurun_out/, the reports themselves deleted.  Usage: tools/gpu_profile_digest.sh TAG
tag=$1
bash tools/gpu_profile_round.sh $tag > gpurun_out/${tag}_prof.log 2>&1
python tools/ncu_summary.py gpurun_out/launch_step_$tag.csv > gpurun_out/${tag}_launches_step_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/launch_prec_$tag.csv > gpurun_out/${tag}_launches_prec_summary.txt 2>&1
python tools/ncu_digest.py gpurun_out/${tag}_*.ncu-rep > gpurun_out/${tag}_ncu_full_digest.txt 2>&1
python tools/ncu_traffic.py gpurun_out/${tag}_ncu_traffic.json gpurun_out/${tag}_*.ncu-rep > /dev/null 2>&1
for k in k_ozaki col1 k_faces k_plane_fast; do
  [ -f gpurun_out/${tag}_$k.ncu-rep ] && python tools/ncu_hot.py gpurun_out/${tag}_$k.ncu-rep 30 > gpurun_out/${tag}_${k}_hot_sass.txt 2>&1
done
rm -f gpurun_out/${tag}_*.ncu-rep
# launch list of the bench command itself (set-up, warm-up, timed steps, stage timing)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_bench_$tag.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/${tag}_ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/launch_bench_$tag.csv > gpurun_out/${tag}_launches_bench_summary.txt 2>&1
