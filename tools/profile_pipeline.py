"""Short device-resident pipeline run for ncu (one workload, few steps).

    python tools/profile_pipeline.py [workload] [steps]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1402_2020_b200 as bsm  # noqa: E402
from paper_1402_2020_b200._lib import bsm_params, check, lib  # noqa: E402
from paper_1402_2020_b200.synth import WORKLOADS, workload_pair  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = WORKLOADS[key]
    import torch
    ctx = bsm.Context(0)
    ctx.set_pattern(bsm.generate_pattern())
    if len(sys.argv) > 3:
        ctx.set_refine_mode(int(sys.argv[3]))
    left, right = workload_pair(key)
    dl = torch.from_numpy(left).cuda()
    dr = torch.from_numpy(right).cuda()
    p = bsm_params(w.d_max, 9.0, 16.0, 1.0, 20)
    for _ in range(steps):
        check(lib().bsm_pipeline_u8_device(ctx.handle, C.c_void_p(dl.data_ptr()), C.c_void_p(dr.data_ptr()),
                                           w.width, w.height, C.byref(p), 0))
    torch.cuda.synchronize()
    print(f"{key}: {steps} pipelines, {ctx.last_launch_count()} launches per pipeline")


if __name__ == "__main__":
    main()
