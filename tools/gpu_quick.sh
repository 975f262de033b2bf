#!/bin/bash
# Quick GPU check: gpu tests + bench.  Usage: bash tools/gpu_quick.sh <tag> [pytest -k expr]
TAG=${1:-q}
K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -15 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
