#!/bin/bash
# Round-2: multi-process tests + compute-sanitizer evidence.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist.py tests/test_gpu_batch.py -x -q -m gpu > gpurun_out/r2b_dist.log 2>&1; echo "dist tests rc=$?"
tail -8 gpurun_out/r2b_dist.log
timeout 300 python tools/sanitize_run.py > gpurun_out/r2b_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/r2b_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2b_san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2b_san_$tool.log
done
