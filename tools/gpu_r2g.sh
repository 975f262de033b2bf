#!/bin/bash
mkdir -p gpurun_out
T=${1:-r2g}
timeout 900 python tools/k3_ab.py c1 c2 c3 c4 c5 -- 0 4 8 > gpurun_out/${T}_k3_ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/${T}_k3_ab.txt
for v in 0 4; do for wl in c2 c4; do
  BSM_K3_VARIANT=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_cost_wta -c 1 --csv \
      --log-file gpurun_out/${T}_traffic_${wl}_v$v.csv python tools/profile_pipeline.py $wl 1 > gpurun_out/${T}_traffic_$wl.log 2>&1; echo "traffic $wl v$v rc=$?"
  grep -o '"dram__bytes_read.sum","[a-z]*","[0-9.]*"' gpurun_out/${T}_traffic_${wl}_v$v.csv
done; done
