"""Band pipeline vs full frame, every map, fresh contexts (run with BSM_GUARD=1
to expose reads of never-written device memory).

    BSM_GUARD=1 python tools/band_diag.py c5 2
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1402_2020_b200 as bsm  # noqa: E402
from paper_1402_2020_b200._lib import bsm_maps, bsm_params, check, lib  # noqa: E402
from paper_1402_2020_b200.dist import band_rows  # noqa: E402
from paper_1402_2020_b200.synth import WORKLOADS, workload_pair  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c5"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = WORKLOADS[key]
    left, right = workload_pair(key)
    H, W = left.shape
    cfg = bsm.BsmConfig(d_max=w.d_max)
    full = bsm.run_pipeline(left, right, cfg, ctx=bsm.Context(0))
    for r in range(world):
        y0, y1 = band_rows(H, world, r)
        ctx = bsm.Context(0)
        ctx.set_pattern(bsm.generate_pattern(cfg=cfg))
        p = bsm_params(w.d_max, 9.0, 16.0, 1.0, 20)
        rd = np.empty((y1 - y0, W), np.float32)
        rv = np.empty((y1 - y0), np.uint8) if False else np.empty((y1 - y0, W), np.uint8)
        check(lib().bsm_pipeline_band_u8(ctx.handle, left.ctypes.data, right.ctypes.data, W, H, y0, y1, C.byref(p),
                                         rd.ctypes.data, rv.ctypes.data))
        r0, r1 = max(0, y0 - 20), min(H, y1 + 20)
        mk = lambda dt: np.empty((r1 - r0, W), dt)
        ld, rwd, cd, cv = mk(np.float32), mk(np.float32), mk(np.float32), mk(np.uint8)
        m = bsm_maps(None, None, ld.ctypes.data, rwd.ctypes.data, cd.ctypes.data, cv.ctypes.data, None)
        check(lib().bsm_fetch_maps(ctx.handle, C.byref(m)))
        for name, got, want in (("left_d", ld, full.left_wta.disparity[r0:r1]),
                                ("right_d", rwd, full.right_wta.disparity[r0:r1]),
                                ("checked_d", cd, full.checked.disparity[r0:r1]),
                                ("checked_v", cv, full.checked.valid[r0:r1]),
                                ("refined_d", rd, full.refined.disparity[y0:y1]),
                                ("refined_v", rv, full.refined.valid[y0:y1])):
            bad = np.argwhere(got != want)
            if len(bad):
                print(f"rank {r} rows [{y0},{y1}) {name}: {len(bad)} differ; rows {bad[:, 0].min()}..{bad[:, 0].max()}"
                      f" cols {bad[:, 1].min()}..{bad[:, 1].max()}; first {bad[:3].tolist()}", flush=True)
            else:
                print(f"rank {r} {name}: equal", flush=True)
        print("guards", ctx.debug_check_guards(), flush=True)


if __name__ == "__main__":
    main()
