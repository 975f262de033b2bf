#!/bin/bash
# Build the tensor-core cost-kernel probe (tools/microbench/tc_probe) for sm_100a.
set -e
D=/root/repo/tools/microbench
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo "$@" -I$D/../../paper_1402_2020_b200/csrc \
     -o $D/tc_probe $D/tc_probe.cu -lcuda
