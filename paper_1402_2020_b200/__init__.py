"""B200-native Binary Stereo Matching (arXiv 1402.2020) hot path.

Python host mirror of the reference library's public API
(/root/reference/proj/include/bsm): same function names, argument meaning and
error behaviour, over the sm_100a kernels in ``libbsm_cuda.so`` (C ABI:
include/bsm_cuda.h).  Images are grayscale ``uint8`` views (a gray PGM loads as
r = g = b, image_io.hpp:257-259); disparity maps are ``DisparityMap`` objects
(float32 disparity + uint8 valid, image.hpp:243-263).

There is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from ._lib import (
    BsmError,
    CudaError,
    DimensionMismatch,
    InvalidArgument,
    Unsupported,
    bsm_maps,
    bsm_params,
    check,
    lib,
)

__all__ = [
    "BsmConfig", "SamplingPattern", "DisparityMap", "PipelineResult", "Context",
    "generate_pattern", "gray_lab_lut", "to_gray_lab", "compute_field", "wta", "lr_check",
    "vote_refine", "run_pipeline", "run_pipeline_band", "run_pipeline_batch", "default_context",
    "BsmError", "InvalidArgument", "DimensionMismatch", "CudaError", "Unsupported",
    "GENERATOR_NAME",
]

GENERATOR_NAME = "mt19937_64-boxmuller-v1"  # pattern.hpp:16


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# Value types
@dataclass
class BsmConfig:
    """BsmConfig (config.hpp:16-47).  d_max has no default (config.hpp:14-15)."""

    n: int = 4096
    window: int = 26
    spread: float = 4.0
    seed: int = 42
    d_max: int = 0
    lambda_c: float = 9.0
    lambda_e: float = 16.0
    lr_tolerance: float = 1.0
    vote_radius: int = 20
    gt_scale: float = 16.0
    threads: int = 1  # accepted and ignored for device work (output is thread-count independent)
    generator: str = GENERATOR_NAME

    def validate(self) -> None:  # config.hpp:30-44
        if self.n < 1: raise InvalidArgument("config: n must be >= 1")
        if self.window < 2: raise InvalidArgument("config: S must be >= 2")
        if not self.spread > 0: raise InvalidArgument("config: spread must be > 0")
        if self.d_max < 1: raise InvalidArgument("config: d_max must be set (>= 1)")
        if not self.lambda_c > 0: raise InvalidArgument("config: lambda_c must be > 0")
        if not self.lambda_e > 0: raise InvalidArgument("config: lambda_e must be > 0")
        if self.lr_tolerance < 0: raise InvalidArgument("config: lr_tolerance must be >= 0")
        if self.vote_radius < 1: raise InvalidArgument("config: vote_radius must be >= 1")
        if not self.gt_scale > 0: raise InvalidArgument("config: gt_scale must be > 0")
        if self.threads < 1: raise InvalidArgument("config: threads must be >= 1")
        if self.generator != GENERATOR_NAME:
            raise InvalidArgument(
                f"config: unknown generator '{self.generator}', this build provides {GENERATOR_NAME}")


@dataclass
class SamplingPattern:
    """SamplingPattern (pattern.hpp:62-72); pairs is (n, 4) int16 {px, py, qx, qy}."""

    n: int
    window: int
    spread: float
    seed: int
    pairs: np.ndarray

    def half_window(self) -> int:
        return self.window // 2


@dataclass
class DisparityMap:
    """DisparityMap (image.hpp:243-263)."""

    disparity: np.ndarray  # (H, W) float32
    valid: np.ndarray      # (H, W) uint8

    @property
    def width(self) -> int:
        return int(self.disparity.shape[1])

    @property
    def height(self) -> int:
        return int(self.disparity.shape[0])

    def __eq__(self, other) -> bool:
        return (isinstance(other, DisparityMap)
                and np.array_equal(self.disparity.view(np.uint32), other.disparity.view(np.uint32))
                and np.array_equal(self.valid, other.valid))


@dataclass
class PipelineResult:
    """PipelineResult (pipeline.hpp:14-20)."""

    refined: DisparityMap
    left_wta: DisparityMap
    right_wta: DisparityMap
    checked: DisparityMap
    unmasked: Optional[DisparityMap] = None


# ---------------------------------------------------------------------------
# Context
class Context:
    """A device context: one CUDA device, one stream, the uploaded pattern."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().bsm_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = int(device)
        self._pattern_key = None

    def close(self) -> None:
        for comm in list(self.__dict__.get("_comms", {}).values()):  # NCCL communicators first
            comm.close()
        if getattr(self, "_h", None):
            lib().bsm_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        if not self._h:
            raise BsmError("bsm: context is closed")
        return self._h

    def set_pattern(self, pattern: SamplingPattern) -> None:
        pairs = np.ascontiguousarray(pattern.pairs, dtype=np.int16).reshape(-1, 4)
        key = (pattern.window, pairs.tobytes())
        if key == self._pattern_key:
            return
        self._pattern_key = None  # a failed upload leaves the context without a pattern
        check(lib().bsm_set_pattern(self.handle, _ptr(pairs), int(pairs.shape[0]), int(pattern.window)))
        self._pattern_key = key

    def stream_ptr(self) -> int:
        s = C.c_void_p()
        check(lib().bsm_stream(self.handle, C.byref(s)))
        return int(s.value or 0)

    def set_profiling(self, enable: bool) -> None:
        check(lib().bsm_set_profiling(self.handle, 1 if enable else 0))

    def last_timings(self) -> dict:
        names = lib().bsm_timing_names().decode().split(",")
        ms = np.zeros(len(names), np.float32)
        cnt = C.c_int()
        check(lib().bsm_last_timings(self.handle, _ptr(ms), len(names), C.byref(cnt)))
        return {n: float(v) for n, v in zip(names, ms[: cnt.value])}

    def last_launch_count(self) -> int:
        cnt = C.c_int()
        check(lib().bsm_last_launch_count(self.handle, C.byref(cnt)))
        return int(cnt.value)

    def measure_popc_peak(self) -> float:
        v = C.c_double()
        check(lib().bsm_measure_popc_peak(self.handle, C.byref(v)))
        return float(v.value)

    def debug_check_guards(self) -> tuple:
        """(damaged guard bytes, guard mode on) -- see bsm_debug_check_guards."""
        n, on = C.c_longlong(), C.c_int()
        check(lib().bsm_debug_check_guards(self.handle, C.byref(n), C.byref(on)))
        return int(n.value), bool(on.value)

    def set_refine_mode(self, mode: int) -> None:
        """-1 auto, 2 warp per pixel + host weight table, 3 ordered fold + table, 4 fold + device exp."""
        check(lib().bsm_set_refine_mode(self.handle, int(mode)))

    def device_exp(self, x) -> np.ndarray:
        """The device restatement of libm's exp (refine weights) on `x`."""
        xs = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(xs)
        check(lib().bsm_device_exp(self.handle, _ptr(xs), int(xs.size), _ptr(out)))
        return out

    def measure_word_peaks(self) -> tuple:
        """(direct POPC mix, carry-save mix) word-op rates of this GPU, words/s."""
        a, b = C.c_double(), C.c_double()
        check(lib().bsm_measure_word_peaks(self.handle, C.byref(a), C.byref(b)))
        return float(a.value), float(b.value)

    def measure_mma_peak(self) -> float:
        """Dense FP4 tensor rate (kind::mxf4 MMAs back to back) of this GPU, flop/s."""
        v = C.c_double()
        check(lib().bsm_measure_mma_peak(self.handle, C.byref(v)))
        return float(v.value)


_tls = threading.local()


def default_context() -> Context:
    """Per-thread context on LOCAL_RANK's device (0 by default)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(int(os.environ.get("LOCAL_RANK", "0")))
        _tls.ctx = ctx
    return ctx


# ---------------------------------------------------------------------------
# Host-side helpers (pattern.hpp, image.hpp)
def generate_pattern(n: int = 4096, window: int = 26, spread: float = 4.0, seed: int = 42,
                     cfg: Optional[BsmConfig] = None) -> SamplingPattern:
    """generate_pattern (pattern.hpp:74-103; config overload config.hpp:104-108)."""
    if cfg is not None:
        if cfg.generator != GENERATOR_NAME:
            raise InvalidArgument(f"config: unknown generator '{cfg.generator}'")
        n, window, spread, seed = cfg.n, cfg.window, cfg.spread, cfg.seed
    out = np.zeros((max(int(n), 1), 4), np.int16)
    check(lib().bsm_generate_pattern(int(n), int(window), float(spread), C.c_uint64(int(seed)), _ptr(out)))
    return SamplingPattern(int(n), int(window), float(spread), int(seed), out)


def gray_lab_lut():
    """to_gray / to_lab of (v, v, v) for v = 0..255 (image.hpp:90-140)."""
    g = np.zeros(256, np.float32)
    l = np.zeros((256, 3), np.float32)
    check(lib().bsm_gray_lab_lut(_ptr(g), _ptr(l)))
    return g, l


def to_gray_lab(rgb):
    """to_gray / to_lab (image.hpp:90-140) of an (H, W, 3) uint8 image, host-side."""
    a = np.ascontiguousarray(rgb, dtype=np.uint8)
    if a.ndim != 3 or a.shape[2] != 3:
        raise InvalidArgument("bsm: to_gray_lab expects an (H, W, 3) uint8 image")
    H, W = a.shape[:2]
    g = np.zeros((H, W), np.float32)
    l = np.zeros((H, W, 3), np.float32)
    check(lib().bsm_to_gray_lab(_ptr(a), W, H, _ptr(g), _ptr(l)))
    return g, l


def _rgb(img, name="image") -> np.ndarray:
    a = np.ascontiguousarray(img)
    if a.dtype != np.uint8 or a.ndim != 3 or a.shape[2] != 3:
        raise InvalidArgument(f"bsm: {name} must be a 2-D uint8 grayscale or (H, W, 3) uint8 RGB array")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise InvalidArgument("bsm: image dimensions must be >= 1")
    return a


def _view(img, name="image") -> np.ndarray:
    """A grayscale (H, W) or RGB (H, W, 3) uint8 view."""
    a = np.asarray(img)
    return _rgb(a, name) if a.ndim == 3 else _u8(a, name)


def _is_gray(rgb: np.ndarray) -> bool:
    return bool(np.array_equal(rgb[:, :, 0], rgb[:, :, 1]) and np.array_equal(rgb[:, :, 1], rgb[:, :, 2]))


def rgb24_tables():
    """to_gray / to_lab of every 24-bit colour, index (r << 16) | (g << 8) | b."""
    g = np.zeros(1 << 24, np.float32)
    l = np.zeros((1 << 24, 3), np.float32)
    check(lib().bsm_rgb24_tables(_ptr(g), _ptr(l)))
    return g, l


def _u8(img, name="image") -> np.ndarray:
    a = np.ascontiguousarray(img)
    if a.dtype != np.uint8 or a.ndim != 2:
        raise InvalidArgument(f"bsm: {name} must be a 2-D uint8 (grayscale) array")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise InvalidArgument("bsm: image dimensions must be >= 1")
    return a


# ---------------------------------------------------------------------------
# Hot path
def compute_field(img, pattern: SamplingPattern, threads: int = 1, ctx: Optional[Context] = None):
    """compute_field (descriptor.hpp:200-239).

    `img` is a grayscale uint8 view, an (H, W, 3) uint8 RGB view, or the
    reference's own argument pair (gray (H, W) float32, lab (H, W, 3) float32).
    Returns (descriptors, masks), each (H, W, words64) uint64 in the
    reference's AoS layout (descriptor.hpp:48-50).
    """
    ctx = ctx or default_context()
    ctx.set_pattern(pattern)
    words = (pattern.n + 63) // 64
    if isinstance(img, tuple):
        if len(img) != 2:
            raise InvalidArgument("bsm: compute_field expects (gray, lab) planes")
        g = np.ascontiguousarray(img[0], dtype=np.float32)
        lab = np.ascontiguousarray(img[1], dtype=np.float32)
        if g.ndim != 2 or lab.ndim != 3 or lab.shape[2] != 3:
            raise InvalidArgument("bsm: planes must be gray (H, W) and lab (H, W, 3)")
        if lab.shape[:2] != g.shape:
            raise DimensionMismatch("compute_field: gray/lab dimensions differ")
    else:
        a = _view(img)
        if a.ndim == 2:
            H, W = a.shape
            desc = np.zeros((H, W, words), np.uint64)
            mask = np.zeros((H, W, words), np.uint64)
            check(lib().bsm_compute_field_u8(ctx.handle, _ptr(a), W, H, _ptr(desc), _ptr(mask)))
            return desc, mask
        g, lab = to_gray_lab(a)
    H, W = g.shape
    desc = np.zeros((H, W, words), np.uint64)
    mask = np.zeros((H, W, words), np.uint64)
    check(lib().bsm_compute_field_f32(ctx.handle, _ptr(g), _ptr(lab), W, H, _ptr(desc), _ptr(mask)))
    return desc, mask


def wta(desc_ref, mask_ref, desc_other, d_max: int, direction: str = "left", threads: int = 1,
        use_mask: bool = True, n: Optional[int] = None, ctx: Optional[Context] = None) -> DisparityMap:
    """wta (matcher.hpp:80-113).  direction 'left' = RefView::left (x - d)."""
    dr = np.ascontiguousarray(desc_ref, dtype=np.uint64)
    do = np.ascontiguousarray(desc_other, dtype=np.uint64)
    mr = np.ascontiguousarray(mask_ref, dtype=np.uint64) if mask_ref is not None else None
    if dr.shape != do.shape or (mr is not None and mr.shape != dr.shape):
        raise DimensionMismatch("wta: descriptor fields do not agree in size")
    if dr.ndim != 3:
        raise InvalidArgument("bsm: fields must be (H, W, words64) arrays")
    H, W, words = dr.shape
    n = int(n) if n is not None else 64 * words
    if (n + 63) // 64 != words:
        raise DimensionMismatch("wta: descriptor fields do not agree in size")
    if direction not in ("left", "right"):
        raise InvalidArgument("wta: direction must be 'left' or 'right'")
    ctx = ctx or default_context()
    out = np.zeros((H, W), np.float32)
    check(lib().bsm_wta(ctx.handle, _ptr(dr), _ptr(mr), _ptr(do), W, H, n, int(d_max),
                        1 if direction == "right" else 0, 1 if use_mask else 0, _ptr(out)))
    return DisparityMap(out, np.ones((H, W), np.uint8))


def lr_check(left: DisparityMap, right: DisparityMap, tol: float, ctx: Optional[Context] = None) -> DisparityMap:
    """lr_check (refine.hpp:39-54)."""
    if left.disparity.shape != right.disparity.shape:
        raise DimensionMismatch("lr_check: map dimensions differ")
    ctx = ctx or default_context()
    dl = np.ascontiguousarray(left.disparity, dtype=np.float32)
    dr = np.ascontiguousarray(right.disparity, dtype=np.float32)
    H, W = dl.shape
    od = np.zeros((H, W), np.float32)
    ov = np.zeros((H, W), np.uint8)
    check(lib().bsm_lr_check(ctx.handle, _ptr(dl), _ptr(dr), W, H, float(tol), _ptr(od), _ptr(ov)))
    return DisparityMap(od, ov)


def vote_refine(m: DisparityMap, image, lambda_c: float = 9.0, lambda_e: float = 16.0,
                vote_radius: int = 20, threads: int = 1, ctx: Optional[Context] = None) -> DisparityMap:
    """vote_refine (refine.hpp:62-111).

    `image` is the grayscale uint8 view (its Lab is the conversion of (v,v,v))
    or an (H, W, 3) float32 Lab plane (e.g. from to_gray_lab of a colour view).
    """
    lab = None
    a = np.asarray(image)
    if a.ndim == 3:
        lab = np.ascontiguousarray(a, dtype=np.float32)
        if lab.shape[2] != 3:
            raise InvalidArgument("bsm: Lab planes must be (H, W, 3)")
        shape = lab.shape[:2]
    else:
        g = _u8(a)
        shape = g.shape
    if shape != m.disparity.shape:
        raise DimensionMismatch("vote_refine: map/image dimensions differ")
    if not lambda_c > 0: raise InvalidArgument("refine: lambda_c must be > 0")
    if not lambda_e > 0: raise InvalidArgument("refine: lambda_e must be > 0")
    if vote_radius < 1: raise InvalidArgument("refine: vote_radius must be >= 1")
    ctx = ctx or default_context()
    d = np.ascontiguousarray(m.disparity, dtype=np.float32)
    v = np.ascontiguousarray(m.valid, dtype=np.uint8)
    H, W = d.shape
    od = np.zeros((H, W), np.float32)
    ov = np.zeros((H, W), np.uint8)
    if lab is not None:
        check(lib().bsm_vote_refine_lab(ctx.handle, _ptr(d), _ptr(v), _ptr(lab), W, H, float(lambda_c),
                                        float(lambda_e), int(vote_radius), _ptr(od), _ptr(ov)))
    else:
        check(lib().bsm_vote_refine_u8(ctx.handle, _ptr(d), _ptr(v), _ptr(g), W, H, float(lambda_c),
                                       float(lambda_e), int(vote_radius), _ptr(od), _ptr(ov)))
    return DisparityMap(od, ov)


def _params(cfg: BsmConfig) -> bsm_params:
    return bsm_params(int(cfg.d_max), float(cfg.lambda_c), float(cfg.lambda_e),
                      float(cfg.lr_tolerance), int(cfg.vote_radius))


def run_pipeline(left, right, cfg: BsmConfig, pattern: Optional[SamplingPattern] = None,
                 want_unmasked: bool = False, ctx: Optional[Context] = None,
                 outputs: str = "all") -> PipelineResult:
    """run_pipeline (pipeline.hpp:25-56, and the config overload :58-61).

    Views are grayscale (H, W) uint8 or colour (H, W, 3) uint8 RGB.
    outputs='refined' downloads only the refined map (the others are None-filled
    with empty arrays) -- the end-to-end serving path.
    """
    L = _view(left, "left")
    R = _view(right, "right")
    if L.shape != R.shape:
        raise DimensionMismatch("pipeline: left/right dimensions differ")
    cfg.validate()
    if L.ndim == 3 and _is_gray(L) and _is_gray(R):  # r = g = b views take the uint8 path
        L, R = np.ascontiguousarray(L[:, :, 0]), np.ascontiguousarray(R[:, :, 0])
    if pattern is None:
        pattern = generate_pattern(cfg=cfg)
    ctx = ctx or default_context()
    ctx.set_pattern(pattern)
    H, W = L.shape[:2]
    full = outputs == "all"
    mk = lambda dt: np.empty((H, W), dt)
    rd, rv = mk(np.float32), mk(np.uint8)
    ld = mk(np.float32) if full else None
    rwd = mk(np.float32) if full else None
    cd = mk(np.float32) if full else None
    cv = mk(np.uint8) if full else None
    ud = mk(np.float32) if (full and want_unmasked) else None
    maps = bsm_maps(rd.ctypes.data, rv.ctypes.data, ld.ctypes.data if ld is not None else None,
                    rwd.ctypes.data if rwd is not None else None, cd.ctypes.data if cd is not None else None,
                    cv.ctypes.data if cv is not None else None, ud.ctypes.data if ud is not None else None)
    p = _params(cfg)
    fn = lib().bsm_pipeline_rgb if L.ndim == 3 else lib().bsm_pipeline_u8
    check(fn(ctx.handle, _ptr(L), _ptr(R), W, H, C.byref(p), 1 if want_unmasked else 0, C.byref(maps)))
    ones = np.ones((H, W), np.uint8)
    res = PipelineResult(
        refined=DisparityMap(rd, rv),
        left_wta=DisparityMap(ld, ones) if full else None,
        right_wta=DisparityMap(rwd, ones) if full else None,
        checked=DisparityMap(cd, cv) if full else None,
    )
    if ud is not None:
        res.unmasked = DisparityMap(ud, ones)
    return res


def run_pipeline_band(left, right, cfg: BsmConfig, y0: int, y1: int,
                      pattern: Optional[SamplingPattern] = None, ctx: Optional[Context] = None) -> DisparityMap:
    """Rows [y0, y1) of run_pipeline(...).refined, computed with a local
    vote-radius halo (the row-band unit of the multi-GPU frame partition)."""
    L = _u8(left, "left")
    R = _u8(right, "right")
    if L.shape != R.shape:
        raise DimensionMismatch("pipeline: left/right dimensions differ")
    cfg.validate()
    if pattern is None:
        pattern = generate_pattern(cfg=cfg)
    ctx = ctx or default_context()
    ctx.set_pattern(pattern)
    H, W = L.shape
    rd = np.empty((y1 - y0, W), np.float32)
    rv = np.empty((y1 - y0, W), np.uint8)
    p = _params(cfg)
    check(lib().bsm_pipeline_band_u8(ctx.handle, _ptr(L), _ptr(R), W, H, int(y0), int(y1), C.byref(p),
                                     _ptr(rd), _ptr(rv)))
    return DisparityMap(rd, rv)


def _ptr_array(arrays):
    return (C.c_void_p * max(len(arrays), 1))(*[a.ctypes.data for a in arrays])


def run_pipeline_batch(pairs, cfg: BsmConfig, pattern: Optional[SamplingPattern] = None,
                       ctx: Optional[Context] = None) -> list:
    """run_pipeline(...).refined of every (left, right) grayscale pair of a batch
    (BASELINE configs[3]; pipeline.hpp:25-56 per pair).  One C-ABI call
    (bsm_pipeline_batch_u8) overlaps each pair's upload and download with its
    neighbours' compute.  All pairs share one shape."""
    views = [(_u8(l, "left"), _u8(r, "right")) for l, r in pairs]
    if not views:
        return []
    H, W = views[0][0].shape
    for L, R in views:
        if L.shape != R.shape or L.shape != (H, W):
            raise DimensionMismatch("pipeline: left/right dimensions differ")
    cfg.validate()
    if pattern is None:
        pattern = generate_pattern(cfg=cfg)
    ctx = ctx or default_context()
    ctx.set_pattern(pattern)
    outs = [(np.empty((H, W), np.float32), np.empty((H, W), np.uint8)) for _ in views]
    p = _params(cfg)
    check(lib().bsm_pipeline_batch_u8(ctx.handle, len(views), _ptr_array([v[0] for v in views]),
                                      _ptr_array([v[1] for v in views]), W, H, C.byref(p),
                                      _ptr_array([o[0] for o in outs]), _ptr_array([o[1] for o in outs])))
    return [DisparityMap(d, v) for d, v in outs]
