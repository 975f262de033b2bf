#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2j_pytest_gpu.log
BSM_GUARD=1 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_pytest_gpu_guard.log 2>&1; echo "guard pytest rc=$?"; tail -2 gpurun_out/r2j_pytest_gpu_guard.log
bash tools/gpu_stage.sh c2 c4 c1 c5
