#!/bin/bash
# Round-2 check: batch tests + default (c4 batch) bench + c2 bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/r2a_batch.log 2>&1; echo "batch tests rc=$?"
tail -5 gpurun_out/r2a_batch.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a_bench_c4.json 2> gpurun_out/r2a_bench_c4.err; echo "bench c4 rc=$?"
cat gpurun_out/r2a_bench_c4.json; tail -5 gpurun_out/r2a_bench_c4.err
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_c2.json 2> gpurun_out/r2a_bench_c2.err; echo "bench c2 rc=$?"
cat gpurun_out/r2a_bench_c2.json; tail -5 gpurun_out/r2a_bench_c2.err
