#!/bin/bash
# Bench every workload at N=1 (+ torchrun launch of the default), JSON lines to gpurun_out/<tag>_bench_<wl>.json
TAG=${1:-b}
mkdir -p gpurun_out
for WL in c2 c1 c3 c5 c4 c2rgb; do
  timeout 600 python bench.py --workload $WL --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_${WL}.json 2> gpurun_out/${TAG}_bench_${WL}.err
  echo "$WL rc=$?"; cut -c1-400 gpurun_out/${TAG}_bench_${WL}.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_torchrun.json 2> gpurun_out/${TAG}_bench_torchrun.err
echo "torchrun rc=$?"; cut -c1-300 gpurun_out/${TAG}_bench_torchrun.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
echo "reference rc=$?"; cat gpurun_out/${TAG}_bench_reference.json
timeout 900 python bench.py --impl reference --workload c2rgb --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference_c2rgb.json 2> gpurun_out/${TAG}_bench_reference_c2rgb.err
echo "reference c2rgb rc=$?"; cut -c1-300 gpurun_out/${TAG}_bench_reference_c2rgb.json
