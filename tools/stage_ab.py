"""A/B of per-stage device times across refine modes on one workload.

    python tools/stage_ab.py [workload] [modes...]
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
    modes = [int(m) for m in sys.argv[2:]] or [-1]
    w = WORKLOADS[key]
    import torch
    left, right = workload_pair(key)
    dl = torch.from_numpy(left).cuda()
    dr = torch.from_numpy(right).cuda()
    p = bsm_params(w.d_max, 9.0, 16.0, 1.0, 20)
    ref = None
    for mode in modes:
        ctx = bsm.Context(0)
        ctx.set_pattern(bsm.generate_pattern())
        ctx.set_refine_mode(mode)
        ctx.set_profiling(True)
        acc = {}
        for it in range(8):
            check(lib().bsm_pipeline_u8_device(ctx.handle, C.c_void_p(dl.data_ptr()), C.c_void_p(dr.data_ptr()),
                                               w.width, w.height, C.byref(p), 0))
            torch.cuda.synchronize()
            if it >= 3:
                for k, v in ctx.last_timings().items():
                    acc.setdefault(k, []).append(v)
        d = np.empty((w.height, w.width), np.float32)
        v = np.empty((w.height, w.width), np.uint8)
        from paper_1402_2020_b200._lib import bsm_maps
        maps = bsm_maps(d.ctypes.data, v.ctypes.data, None, None, None, None, None)
        check(lib().bsm_fetch_maps(ctx.handle, C.byref(maps)))
        same = None
        if ref is None:
            ref = (d.copy(), v.copy())
        else:
            same = bool(np.array_equal(ref[0], d) and np.array_equal(ref[1], v))
        print(key, "mode", mode, {k: round(float(np.median(x)), 3) for k, x in acc.items()}, "same_as_first", same)


if __name__ == "__main__":
    main()
