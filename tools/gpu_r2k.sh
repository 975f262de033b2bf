#!/bin/bash
for v in 0 1; do echo "mask variant $v"; BSM_MASK_VARIANT=$v bash tools/gpu_stage.sh c2 c4; done
BSM_MASK_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or compute_field or random" 2>&1 | tail -2
