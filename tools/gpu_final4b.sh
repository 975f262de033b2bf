#!/bin/bash
# Round-2 closing evidence, part B (guard suite, the other workloads, A/B tables).  Usage (under gpurun): bash tools/gpu_final4b.sh <tag>
T=${1:-r02}
mkdir -p gpurun_out
BSM_GUARD=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu_guard.log 2>&1; echo "guard pytest rc=$?"; tail -2 gpurun_out/${T}_pytest_gpu_guard.log
for wl in c1 c2 c3 c5 c2rgb; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/${T}_bench_$wl.json 2> gpurun_out/${T}_bench_$wl.err; echo "bench $wl rc=$?"
done
timeout 900 python bench.py --impl reference --workload c2 --steps 10 --warmup 3 > gpurun_out/${T}_bench_reference_c2.json 2>&1; echo "bench reference c2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_torchrun.json 2> gpurun_out/${T}_bench_torchrun.err; echo "torchrun rc=$?"
timeout 900 python tools/k3_ab.py c1 c2 c3 c4 c5 -- 0 32 16 > gpurun_out/${T}_k3_ab.txt 2>&1; echo "k3 ab rc=$?"
for wl in c1 c2 c3 c5; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_cost_wta|k_mask" -c 3 --csv \
      --log-file gpurun_out/${T}_traffic_$wl.csv python tools/profile_pipeline.py $wl 1 > /dev/null 2>&1; echo "traffic $wl rc=$?"
done
timeout 300 python tools/profile_colour.py > gpurun_out/${T}_colour_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mask_f32|k_descriptor_f32|k_rgb_planes" -c 4 \
      -o gpurun_out/${T}_colour python tools/profile_colour.py > gpurun_out/${T}_colour_ncu.log 2>&1; echo "ncu colour rc=$?"
python tools/summarize_ncu.py gpurun_out/${T}_colour.ncu-rep > gpurun_out/${T}_ncu_kernels_c2rgb.txt 2>&1
echo done
