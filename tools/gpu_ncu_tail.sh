#!/bin/bash
# The ncu part of gpu_final3.sh alone (launch list, --set full of one c4 pair's
# kernels, DRAM traffic of K3 and K2 per workload).  Usage: bash tools/gpu_ncu_tail.sh <tag>
T=${1:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 1 --warmup 1 --profile-only --pairs 4 > gpurun_out/${T}_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c4.csv \
    python bench.py --steps 1 --warmup 1 --profile-only --pairs 4 > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python tools/profile_pipeline.py c4 1 > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cost_wta|k_mask|k_descriptor4|k_vote_refine_fold|k_lr_check_keys" -c 5 \
    -o gpurun_out/${T}_c4_full python tools/profile_pipeline.py c4 1 > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/summarize_ncu.py gpurun_out/${T}_c4_full.ncu-rep > gpurun_out/${T}_ncu_kernels_c4.txt 2>&1
for wl in c1 c2 c3 c4 c5; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_cost_wta|k_mask" -c 3 --csv \
      --log-file gpurun_out/${T}_traffic_$wl.csv python tools/profile_pipeline.py $wl 1 > /dev/null 2>&1; echo "traffic $wl rc=$?"
done
echo done
