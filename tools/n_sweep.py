"""Stage times vs descriptor length n (the length-sweep axis, eval.hpp:108-139).

    python tools/n_sweep.py [workload] [n ...]
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
    ns = [int(v) for v in sys.argv[2:]] or [512, 1024, 2048, 4096, 8192]
    w = WORKLOADS[key]
    import torch
    left, right = workload_pair(key)
    dl = torch.from_numpy(left).cuda()
    dr = torch.from_numpy(right).cuda()
    p = bsm_params(w.d_max, 9.0, 16.0, 1.0, 20)
    for n in ns:
        ctx = bsm.Context(0)
        ctx.set_pattern(bsm.generate_pattern(n=n))
        ctx.set_profiling(True)
        acc = {}
        for it in range(6):
            check(lib().bsm_pipeline_u8_device(ctx.handle, C.c_void_p(dl.data_ptr()), C.c_void_p(dr.data_ptr()),
                                               w.width, w.height, C.byref(p), 0))
            torch.cuda.synchronize()
            if it >= 2:
                for k, t in ctx.last_timings().items():
                    acc.setdefault(k, []).append(t)
        st = {k: round(float(np.median(x)), 3) for k, x in acc.items() if np.median(x) > 0}
        print(key, "n", n, st, "total", round(sum(st.values()), 2), flush=True)


if __name__ == "__main__":
    main()
