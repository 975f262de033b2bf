#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/csa_mixes tools/microbench/csa_mixes.cu && timeout 300 /tmp/csa_mixes > gpurun_out/r2d_csa_mixes.txt 2>&1; echo "mixes rc=$?"; cat gpurun_out/r2d_csa_mixes.txt
timeout 900 python tools/k3_ab.py c1 c2 c4 c5 -- 0 1 2 3 > gpurun_out/r2d_k3_ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/r2d_k3_ab.txt
