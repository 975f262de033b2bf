"""Throughput of back-to-back pairs: one context vs two contexts (two streams) alternating.

    python tools/overlap_test.py [workload] [pairs]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1402_2020_b200 as bsm  # noqa: E402
from paper_1402_2020_b200._lib import bsm_params, check, lib  # noqa: E402
from paper_1402_2020_b200.synth import WORKLOADS, workload_pair  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c4"
    npairs = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    w = WORKLOADS[key]
    import torch
    views = []
    for i in range(2):
        L, R = workload_pair(key, index=i)
        views.append((torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()))
    p = bsm_params(w.d_max, 9.0, 16.0, 1.0, 20)
    pat = bsm.generate_pattern()
    for nctx in (1, 2, 3):
        ctxs = [bsm.Context(0) for _ in range(nctx)]
        for c in ctxs:
            c.set_pattern(pat)
        def run(i):
            c = ctxs[i % nctx]
            dl, dr = views[i % 2]
            check(lib().bsm_pipeline_u8_device(c.handle, C.c_void_p(dl.data_ptr()), C.c_void_p(dr.data_ptr()),
                                               w.width, w.height, C.byref(p), 0))
        for i in range(2 * nctx):
            run(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(npairs):
            run(i)
        for c in ctxs:
            torch.cuda.ExternalStream(c.stream_ptr()).synchronize()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{key} contexts={nctx}: {ms / npairs:.2f} ms/pair", flush=True)


if __name__ == "__main__":
    main()
