#!/bin/bash
# One GPU call: tests, bench, launch list and an ncu capture of the top kernels.
# Usage (under gpurun): bash tools/gpu_round.sh <tag> [skip_tests] [ncu_kernels_regex]
TAG=${1:-r}
SKIP_TESTS=${2:-0}
KREGEX=${3:-"k_mask4|k_cost_wta"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt
if [ "$SKIP_TESTS" = "0" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json
timeout 300 python tools/profile_pipeline.py c2 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python tools/profile_pipeline.py c2 2 > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python tools/profile_pipeline.py c2 1 > gpurun_out/${TAG}_plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -c 3 \
    -o gpurun_out/${TAG}_prof python tools/profile_pipeline.py c2 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/${TAG}_ncu_full.log
