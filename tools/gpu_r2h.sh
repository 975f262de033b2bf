#!/bin/bash
mkdir -p gpurun_out
for g in 32 148 592 1184 3000; do
  echo "group $g"; BSM_K3_GROUP=$g timeout 900 python tools/k3_ab.py c2 c4 -- 0 2>&1 | grep variant
done
for g in 592 1184 3000; do for wl in c2 c4; do
  BSM_K3_GROUP=$g timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_cost_wta -c 1 --csv \
      --log-file gpurun_out/r2h_traffic_${wl}_g$g.csv python tools/profile_pipeline.py $wl 1 > /dev/null 2>&1; echo "traffic $wl g$g"
  grep -o '"dram__bytes_read.sum","[a-z]*","[0-9.]*"' gpurun_out/r2h_traffic_${wl}_g$g.csv
done; done
