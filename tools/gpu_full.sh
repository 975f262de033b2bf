#!/bin/bash
# Round evidence in one GPU call: smoke, pytest -m gpu, bench of every workload
# (+ torchrun launch, reference arm), launch list and ncu --set full captures
# of the pipeline kernels.  Usage (under gpurun): bash tools/gpu_full.sh <tag>
TAG=${1:-f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest_gpu.log
bash tools/gpu_bench_all.sh ${TAG}
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
echo "default bench rc=$?"; cut -c1-300 gpurun_out/${TAG}_bench_default.json
bash tools/gpu_prof.sh ${TAG} c2
for K in k_cost_wta k_mask4 k_descriptor4 k_vote_refine_fold k_lr_check_keys; do
  python tools/summarize_ncu.py gpurun_out/${TAG}_${K}.ncu-rep >> gpurun_out/${TAG}_ncu_kernels_c2.txt 2>&1
done
# colour path: the three colour kernels of one c2-size RGB pipeline in one report
timeout 300 python tools/profile_colour.py > gpurun_out/${TAG}_colour_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mask_f32|k_descriptor_f32|k_rgb_planes" -c 4 \
      -o gpurun_out/${TAG}_colour python tools/profile_colour.py > gpurun_out/${TAG}_colour_ncu.log 2>&1; echo "ncu colour rc=$?"
python tools/summarize_ncu.py gpurun_out/${TAG}_colour.ncu-rep > gpurun_out/${TAG}_ncu_kernels_c2rgb.txt 2>&1
echo done
