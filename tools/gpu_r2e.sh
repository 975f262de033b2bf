#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2e}
timeout 900 python tools/k3_ab.py c1 c2 c3 c4 c5 -- 0 2 4 6 > gpurun_out/${T}_k3_ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/${T}_k3_ab.txt
for wl in c2 c4; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_cost_wta -c 1 --csv \
      --log-file gpurun_out/${T}_traffic_$wl.csv python tools/profile_pipeline.py $wl 1 > gpurun_out/${T}_traffic_$wl.log 2>&1; echo "traffic $wl rc=$?"
  grep -o '"dram__bytes_[a-z]*.sum","[a-z]*","[0-9.]*"' gpurun_out/${T}_traffic_$wl.csv
done
