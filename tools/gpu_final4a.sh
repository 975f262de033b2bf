#!/bin/bash
# Round-2 closing evidence, part A (the essentials first).  Usage (under gpurun): bash tools/gpu_final4a.sh <tag>
T=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${T}_smi.txt
lscpu > gpurun_out/${T}_lscpu.txt 2>&1; nproc >> gpurun_out/${T}_lscpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo "bench reference rc=$?"
timeout 600 python bench.py --steps 1 --warmup 1 --profile-only --pairs 4 > gpurun_out/${T}_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c4.csv \
    python bench.py --steps 1 --warmup 1 --profile-only --pairs 4 > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python tools/profile_pipeline.py c4 1 > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cost_wta|k_mask|k_descriptor4|k_vote_refine_fold|k_lr_check_keys" -c 5 \
    -o gpurun_out/${T}_c4_full python tools/profile_pipeline.py c4 1 > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/summarize_ncu.py gpurun_out/${T}_c4_full.ncu-rep > gpurun_out/${T}_ncu_kernels_c4.txt 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_cost_wta|k_mask" -c 3 --csv \
    --log-file gpurun_out/${T}_traffic_c4.csv python tools/profile_pipeline.py c4 1 > /dev/null 2>&1; echo "traffic c4 rc=$?"
echo done
