"""BASELINE.json synthetic stereo pairs (bench / test input; csrc/synth.cpp).

configs[0..4] of BASELINE.json with the builder choices pinned in SURVEY.md
section 8(d): shapes, disparity ranges, seeds (c1..c5 -> 1..5, c4 pair i ->
4000 + i).  These stand in for the paper's Middlebury data, which is not
available here.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._lib import SYNTH_PATH


@dataclass(frozen=True)
class Workload:
    name: str
    config: int  # index into BASELINE.json configs
    width: int
    height: int
    d_max: int
    seed: int
    pairs: int = 1


WORKLOADS = {
    "c1": Workload("c1_450x375_d60", 0, 450, 375, 60, 1),
    "c2": Workload("c2_1392x1104_d240", 1, 1392, 1104, 240, 2),
    "c3": Workload("c3_640x480_d64_radiometric", 2, 640, 480, 64, 3),
    "c4": Workload("c4_64x1920x1080_d192", 3, 1920, 1080, 192, 4000, pairs=64),
    "c5": Workload("c5_4096x2160_d256", 4, 4096, 2160, 256, 5),
    # colour input at the configs[1] size: colour_pair views
    "c2rgb": Workload("c2rgb_1392x1104_d240_colour", 1, 1392, 1104, 240, 2),
}

_synth = None


def _lib():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise RuntimeError(f"{SYNTH_PATH} missing: run __graft_entry__.build()")
        _synth = C.CDLL(SYNTH_PATH)
        _synth.bsm_synth_pair.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
        _synth.bsm_synth_pair.restype = C.c_int
    return _synth


def synth_pair(config: int, seed: int, width: int, height: int, with_gt: bool = False):
    """(left, right[, gt_disparity]) uint8 views of one synthetic pair."""
    left = np.empty((height, width), np.uint8)
    right = np.empty((height, width), np.uint8)
    gt = np.empty((height, width), np.int32) if with_gt else None
    rc = _lib().bsm_synth_pair(int(config), C.c_uint64(int(seed)), int(width), int(height),
                               left.ctypes.data, right.ctypes.data, gt.ctypes.data if with_gt else None)
    if rc != 0:
        raise ValueError("synth_pair: bad arguments")
    return (left, right, gt) if with_gt else (left, right)


def workload_pair(key: str, index: int = 0, with_gt: bool = False):
    w = WORKLOADS[key]
    if key.endswith("rgb"):
        if with_gt:
            raise ValueError("colour workloads carry no ground truth")
        return colour_pair(w.height, w.width, seed=w.seed + index)
    return synth_pair(w.config, w.seed + index, w.width, w.height, with_gt)


def colour_pair(height: int, width: int, seed: int = 1, gen=None):
    """(left, right) (H, W, 3) uint8 RGB views of a synthetic colour pair.

    The scene geometry is synth_pair's (configs[0] builder, disparities
    below 60); each view's gray
    level is mapped through three different tone curves and perturbed by
    independent per-channel noise, so r, g and b differ everywhere and the
    colour conversion is exercised on genuinely colour input.  `gen` replaces
    synth_pair (same signature) -- the reference arm passes the generator
    compiled into oracle/_ref.
    """
    left, right = (gen or synth_pair)(0, seed, width, height)
    return colour_views(left, right, seed)


def colour_views(left, right, seed: int):
    """Colour views of a gray pair: three tone curves + per-channel noise."""
    v = np.arange(256, dtype=np.float64)
    luts = np.stack([v, 255.0 * np.sqrt(v / 255.0), 255.0 - 0.8 * v]).round().astype(np.int32)
    rng = np.random.default_rng(seed)
    out = []
    for img in (left, right):
        c = np.stack([luts[k][img] for k in range(3)], axis=-1) + rng.integers(-6, 7, size=img.shape + (3,))
        out.append(np.clip(c, 0, 255).astype(np.uint8))
    return out[0], out[1]


def workload_pair_with(gen, key: str, index: int = 0):
    """workload_pair through another generator with synth_pair's signature."""
    w = WORKLOADS[key]
    if key.endswith("rgb"):
        return colour_pair(w.height, w.width, seed=w.seed + index, gen=gen)
    return gen(w.config, w.seed + index, w.width, w.height)
