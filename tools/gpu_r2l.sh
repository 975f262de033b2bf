#!/bin/bash
echo "single-warp"; BSM_MASK_VARIANT=2 bash tools/gpu_stage.sh c2 c4
for mb in 4 6 8; do echo "k_mask4w minb $mb"; BSM_MASK_MINB=$mb bash tools/gpu_stage.sh c2 c4; done
for mb in 4 6 8; do BSM_MASK_MINB=$mb timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or compute_field or random" 2>&1 | tail -1; done
