"""Envelope edges: large vote radii (the exact weight table would exceed its
256 MiB cap, so the device exp takes over), images taller than the launch
grid allows, unaligned device inputs, and a failed pattern upload."""
import ctypes as C

import numpy as np
import pytest

import paper_1402_2020_b200 as bsm
from paper_1402_2020_b200.synth import synth_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("radius", [60, 180])
def test_large_vote_radius_matches_reference(ctx, ref, radius):
    """refine.hpp:62-111 at radii whose exact gray weight table would take
    0.4-3 GB: auto mode evaluates the weights with the device exp instead
    (bit-identical), without building the table."""
    left, right = synth_pair(0, 77, 150, 40)
    pairs = ref.generate_pattern(512, 16, 4.0, 3)
    want = ref.pipeline(left, right, pairs, 16, 30, radius=radius, threads=8)
    cfg = bsm.BsmConfig(n=512, window=16, seed=3, d_max=30, vote_radius=radius)
    res = bsm.run_pipeline(left, right, cfg, bsm.SamplingPattern(512, 16, 4.0, 3, pairs), ctx=ctx)
    assert np.array_equal(res.refined.disparity, want["refined_d"])
    assert np.array_equal(res.refined.valid, want["refined_v"])


def test_rows_beyond_grid_limit_rejected(ctx):
    img = np.zeros((70000, 1), np.uint8)
    with pytest.raises(bsm.Unsupported, match="65535 rows"):
        bsm.run_pipeline(img, img, bsm.BsmConfig(d_max=1), ctx=ctx)


def test_unaligned_device_views(ctx):
    """Device entry points accept views at any byte address (the mask
    kernel's word-wide tile loads fall back to bytes)."""
    import torch
    from paper_1402_2020_b200._lib import bsm_maps, bsm_params, check, lib
    left, right = synth_pair(0, 5, 124, 36)
    want = bsm.run_pipeline(left, right, bsm.BsmConfig(d_max=40), ctx=ctx)
    buf_l = torch.zeros(124 * 36 + 1, dtype=torch.uint8, device="cuda")
    buf_r = torch.zeros(124 * 36 + 1, dtype=torch.uint8, device="cuda")
    buf_l[1:] = torch.from_numpy(left.reshape(-1)).cuda()
    buf_r[1:] = torch.from_numpy(right.reshape(-1)).cuda()
    torch.cuda.synchronize()
    p = bsm_params(40, 9.0, 16.0, 1.0, 20)
    check(lib().bsm_pipeline_u8_device(ctx.handle, C.c_void_p(buf_l.data_ptr() + 1), C.c_void_p(buf_r.data_ptr() + 1),
                                       124, 36, C.byref(p), 0))
    d, v = np.zeros((36, 124), np.float32), np.zeros((36, 124), np.uint8)
    check(lib().bsm_fetch_maps(ctx.handle, C.byref(bsm_maps(d.ctypes.data, v.ctypes.data, None, None, None, None,
                                                             None))))
    assert np.array_equal(d, want.refined.disparity) and np.array_equal(v, want.refined.valid)


def test_rejected_pattern_keeps_context_consistent(ctx):
    """A pattern the device cannot take raises and leaves the context usable
    with the next valid pattern (no half-updated tables)."""
    good = bsm.generate_pattern(n=256, window=10, seed=9)
    bad = bsm.SamplingPattern(9000, 26, 4.0, 1, np.zeros((9000, 4), np.int16))
    with pytest.raises(bsm.Unsupported):
        ctx.set_pattern(bad)
    left, right = synth_pair(0, 6, 60, 20)
    a = bsm.run_pipeline(left, right, bsm.BsmConfig(n=256, window=10, seed=9, d_max=10), good, ctx=ctx)
    b = bsm.run_pipeline(left, right, bsm.BsmConfig(n=256, window=10, seed=9, d_max=10), good, ctx=bsm.Context(0))
    assert a.refined == b.refined


def test_vote_refine_rejects_out_of_range_valid_disparities(ctx):
    """The per-stage vote_refine's device pre-pass (invalid list, max_bin)
    rejects valid disparities that cannot name a bin (refine.hpp:68-72):
    negative beyond -0.5, NaN, or beyond the envelope."""
    g = synth_pair(0, 3, 40, 12)[0]
    d = np.full((12, 40), 5.0, np.float32)
    v = np.ones((12, 40), np.uint8)
    v[3, 4] = 0
    ok = bsm.vote_refine(bsm.DisparityMap(d, v), g, ctx=ctx)
    assert ok.valid[3, 4] == 1 and ok.disparity[3, 4] == 5.0  # the only invalid pixel takes its voters' bin
    for bad in (-0.75, np.nan, 2e6):
        d2 = d.copy()
        d2[0, 0] = bad
        with pytest.raises(bsm.InvalidArgument, match="out of range"):
            bsm.vote_refine(bsm.DisparityMap(d2, v), g, ctx=ctx)
    # an invalid pixel may hold anything (it is never read as a voter)
    d3 = d.copy()
    d3[3, 4] = np.nan
    assert bsm.vote_refine(bsm.DisparityMap(d3, v), g, ctx=ctx) == ok
