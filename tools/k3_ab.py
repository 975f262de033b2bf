"""A/B of the cost kernel variants (BSM_K3_VARIANT bits: 16 = the integer-pipe
kernel K3p instead of the tensor-core K3, 32 = K3 with A in shared memory; for
K3p: 1 = thread-0
refill with empty barriers instead of last-warp refill, 2 = one launch per
direction) on device-resident workloads; every variant's refined map must
equal the first one's.

    python tools/k3_ab.py c2 c4 -- 0 1 2 3
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1402_2020_b200 as bsm  # noqa: E402
from paper_1402_2020_b200._lib import bsm_maps, bsm_params, check, lib  # noqa: E402
from paper_1402_2020_b200.synth import WORKLOADS, workload_pair  # noqa: E402


def main():
    args = sys.argv[1:]
    sep = args.index("--") if "--" in args else len(args)
    keys, variants = args[:sep] or ["c2"], [int(v) for v in args[sep + 1:]] or [0]
    import torch
    for key in keys:
        w = WORKLOADS[key]
        left, right = workload_pair(key)
        dl, dr = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
        p = bsm_params(w.d_max, 9.0, 16.0, 1.0, 20)
        first = None
        for v in variants:
            os.environ["BSM_K3_VARIANT"] = str(v)
            ctx = bsm.Context(0)
            ctx.set_pattern(bsm.generate_pattern())
            ctx.set_profiling(True)
            t = []
            for it in range(12):
                check(lib().bsm_pipeline_u8_device(ctx.handle, C.c_void_p(dl.data_ptr()), C.c_void_p(dr.data_ptr()),
                                                   w.width, w.height, C.byref(p), 0))
                if it >= 2:
                    t.append(ctx.last_timings()["wta"])
            d = np.empty((w.height, w.width), np.float32)
            vv = np.empty((w.height, w.width), np.uint8)
            check(lib().bsm_fetch_maps(ctx.handle, C.byref(bsm_maps(d.ctypes.data, vv.ctypes.data, None, None, None,
                                                                     None, None))))
            same = None if first is None else bool(np.array_equal(first[0], d) and np.array_equal(first[1], vv))
            if first is None:
                first = (d.copy(), vv.copy())
            print(f"{key} variant {v}: wta median {np.median(t):.3f} ms  min {min(t):.3f}  same_as_first {same}",
                  flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
