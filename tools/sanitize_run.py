"""Small invocations of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): a c1 crop through the fused pipeline
(gray and colour, masked + unmasked WTA), every refine mode, the per-stage
entry points, a 3-pair batch and two row bands.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1402_2020_b200 as bsm  # noqa: E402
from paper_1402_2020_b200.synth import colour_pair, workload_pair  # noqa: E402


def main():
    ctx = bsm.Context(0)
    left, right = workload_pair("c1")
    L, R = np.ascontiguousarray(left[100:164, 60:250]), np.ascontiguousarray(right[100:164, 60:250])
    cfg = bsm.BsmConfig(d_max=60)
    pat = bsm.generate_pattern(cfg=cfg)
    res = bsm.run_pipeline(L, R, cfg, pat, want_unmasked=True, ctx=ctx)
    for mode in (2, 3, 4):
        ctx.set_refine_mode(mode)
        r2 = bsm.run_pipeline(L, R, cfg, pat, ctx=ctx)
        assert r2.refined == res.refined, mode
    ctx.set_refine_mode(-1)
    cl, cr = colour_pair(48, 150, seed=3)
    bsm.run_pipeline(cl, cr, bsm.BsmConfig(d_max=40), pat, ctx=ctx)
    d, m = bsm.compute_field(L[:20, :70], pat, ctx=ctx)
    bsm.wta(d, m, d, 30, "left", ctx=ctx)
    bsm.wta(d, m, d, 30, "right", use_mask=False, ctx=ctx)
    chk = bsm.lr_check(res.left_wta, res.right_wta, 1.0, ctx=ctx)
    bsm.vote_refine(chk, L, ctx=ctx)
    pairs = [(np.ascontiguousarray(left[y:y + 40, 0:200]), np.ascontiguousarray(right[y:y + 40, 0:200]))
             for y in (0, 100, 300)]
    bsm.run_pipeline_batch(pairs, cfg, pat, ctx=ctx)
    for y0, y1 in ((0, 30), (30, 64)):
        bsm.run_pipeline_band(L, R, cfg, y0, y1, pattern=pat, ctx=ctx)
    small = bsm.generate_pattern(n=1000, window=12, seed=5)
    bsm.run_pipeline(L[:30, :90], R[:30, :90], bsm.BsmConfig(n=1000, window=12, seed=5, d_max=20), small, ctx=ctx)
    print("sanitize_run ok")
    return ctx


if __name__ == "__main__":
    main()
