"""One colour pipeline (for ncu): python tools/profile_colour.py [W] [H] [d_max]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1402_2020_b200 as bsm  # noqa: E402
from paper_1402_2020_b200._lib import bsm_maps, bsm_params, check, lib  # noqa: E402
from paper_1402_2020_b200.synth import colour_pair  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 1392
H = int(sys.argv[2]) if len(sys.argv) > 2 else 1104
D = int(sys.argv[3]) if len(sys.argv) > 3 else 240
L, R = colour_pair(H, W, seed=2)
ctx = bsm.Context(0)
ctx.set_pattern(bsm.generate_pattern())
p = bsm_params(D, 9.0, 16.0, 1.0, 20)
d = np.empty((H, W), np.float32)
v = np.empty((H, W), np.uint8)
maps = bsm_maps(d.ctypes.data, v.ctypes.data, None, None, None, None, None)
check(lib().bsm_pipeline_rgb(ctx.handle, C.c_void_p(L.ctypes.data), C.c_void_p(R.ctypes.data), W, H, C.byref(p), 0,
                             C.byref(maps)))
print("ok")
