#!/bin/bash
# ncu captures of the pipeline's kernels (one launch each) + launch list.
# Usage (under gpurun): bash tools/gpu_prof.sh <tag> [workload]
TAG=${1:-p}
WL=${2:-c2}
mkdir -p gpurun_out
timeout 300 python tools/profile_pipeline.py $WL 1 > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/${TAG}_plain.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python tools/profile_pipeline.py $WL 2 > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for K in k_cost_wta k_mask4 k_descriptor4 k_vote_refine_fold k_lr_check_keys; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
      -o gpurun_out/${TAG}_${K} python tools/profile_pipeline.py $WL 1 > gpurun_out/${TAG}_${K}.log 2>&1; echo "ncu $K rc=$?"
done
