"""Evaluation driven by the GPU pipeline (eval.hpp).

``bad_pixel_rate`` (eval.hpp:31-59), the 3x3 ``radiometric_protocol``
(:63-92), the descriptor ``length_sweep`` (:94-139), ``time_pipeline``
(:144-159), ``linear_fit_r2`` (:163-187) and the CSV writers (:189-211).  The
scoring, the fit and the CSV files are the C++ layer's (include/bsm/eval.hpp
through libbsm_io.so, the reference's arithmetic order and messages); the
protocols here drive ``run_pipeline`` on the device.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import BsmConfig, DisparityMap, SamplingPattern, generate_pattern, run_pipeline
from ._lib import DimensionMismatch, InvalidArgument
from .io import EmptyRegion, IoError, check, lib  # noqa: F401  (EmptyRegion: errors.hpp:30-33)


@dataclass
class ErrorReport:
    """ErrorReport (eval.hpp:21-27)."""

    bad_pixel_rate: float = 0.0
    region: str = "all"
    threshold: float = 1.0
    counted: int = 0
    bad: int = 0


def bad_pixel_rate(result: DisparityMap, gt: DisparityMap, region: Optional[np.ndarray] = None,
                   threshold: float = 1.0) -> ErrorReport:
    """Percentage of region pixels (region >= 128) with ground truth whose error
    exceeds `threshold`; invalid estimates count as wrong (eval.hpp:31-59)."""
    if result.disparity.shape != gt.disparity.shape:
        raise DimensionMismatch("bad_pixel_rate: result and ground truth differ in size")
    if region is not None and np.asarray(region).shape != gt.disparity.shape:
        raise DimensionMismatch("bad_pixel_rate: region mask size mismatch")
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    u8 = lambda a: np.ascontiguousarray(a, dtype=np.uint8)
    d, v, gd, gv = f32(result.disparity), u8(result.valid), f32(gt.disparity), u8(gt.valid)
    reg = f32(region) if region is not None else None
    rate, counted, bad = C.c_double(), C.c_long(), C.c_long()
    H, W = d.shape
    check(lib().bsmio_bad_pixel_rate(d.ctypes.data, v.ctypes.data, gd.ctypes.data, gv.ctypes.data,
                                     reg.ctypes.data if reg is not None else None, W, H, float(threshold),
                                     C.byref(rate), C.byref(counted), C.byref(bad)))
    return ErrorReport(rate.value, "all", float(threshold), counted.value, bad.value)


@dataclass
class RadiometricMatrix:
    """RadiometricMatrix (eval.hpp:63-77): rate[i][j] = left condition i vs right j."""

    rate: List[List[float]] = field(default_factory=lambda: [[0.0] * 3 for _ in range(3)])

    def diagonal_mean(self) -> float:
        return (self.rate[0][0] + self.rate[1][1] + self.rate[2][2]) / 3.0

    def off_diagonal_mean(self) -> float:
        s = 0.0
        for i in range(3):
            for j in range(3):
                if i != j:
                    s += self.rate[i][j]
        return s / 6.0


def radiometric_protocol(lefts: Sequence, rights: Sequence, gt: DisparityMap, region: Optional[np.ndarray],
                         pattern: SamplingPattern, cfg: BsmConfig, threshold: float = 1.0,
                         ctx=None) -> RadiometricMatrix:
    """radiometric_protocol (eval.hpp:79-92): all 3x3 exposure combinations."""
    m = RadiometricMatrix()
    for i in range(3):
        for j in range(3):
            res = run_pipeline(lefts[i], rights[j], cfg, pattern, ctx=ctx, outputs="refined")
            m.rate[i][j] = bad_pixel_rate(res.refined, gt, region, threshold).bad_pixel_rate
    return m


@dataclass
class SweepPoint:
    """SweepPoint (eval.hpp:94-98)."""

    n: int = 0
    avg_error: float = 0.0
    wall_time: float = 0.0


@dataclass
class SweepScene:
    """SweepScene (eval.hpp:100-106)."""

    left: np.ndarray
    right: np.ndarray
    gt: DisparityMap
    region: Optional[np.ndarray] = None
    d_max: int = 0


def length_sweep(scenes: Sequence[SweepScene], n_values: Sequence[int], base: BsmConfig,
                 threshold: float = 1.0, ctx=None) -> List[SweepPoint]:
    """length_sweep (eval.hpp:108-139): accuracy and pipeline wall time per
    descriptor length (pattern generation excluded from the time)."""
    if not scenes:
        raise InvalidArgument("length_sweep: no scenes")
    for n in n_values:
        if n < 64:
            raise InvalidArgument("length_sweep: descriptor lengths below 64 are not supported")
    points = []
    for n in n_values:
        cfg = BsmConfig(**{**base.__dict__, "n": int(n)})
        pattern = generate_pattern(cfg=cfg)
        err_sum, secs = 0.0, 0.0
        for sc in scenes:
            cfg.d_max = sc.d_max
            t0 = time.perf_counter()
            res = run_pipeline(sc.left, sc.right, cfg, pattern, ctx=ctx, outputs="refined")
            secs += time.perf_counter() - t0
            err_sum += bad_pixel_rate(res.refined, sc.gt, sc.region, threshold).bad_pixel_rate
        points.append(SweepPoint(int(n), err_sum / float(len(scenes)), secs))
    return points


def time_pipeline(left, right, pattern: SamplingPattern, cfg: BsmConfig, runs: int = 3, ctx=None) -> float:
    """time_pipeline (eval.hpp:144-159): median wall seconds of the full pipeline
    (host views in, all maps out)."""
    if runs < 1:
        raise InvalidArgument("time_pipeline: runs must be >= 1")
    secs = []
    for _ in range(runs):
        t0 = time.perf_counter()
        run_pipeline(left, right, cfg, pattern, ctx=ctx)
        secs.append(time.perf_counter() - t0)
    secs.sort()
    return secs[len(secs) // 2]


def linear_fit_r2(xs: Sequence[float], ys: Sequence[float]) -> float:
    """linear_fit_r2 (eval.hpp:163-187)."""
    x = np.ascontiguousarray(xs, dtype=np.float64)
    y = np.ascontiguousarray(ys, dtype=np.float64)
    if x.shape != y.shape:
        raise InvalidArgument("linear_fit_r2: need two or more points")
    out = C.c_double()
    check(lib().bsmio_linear_fit_r2(x.ctypes.data, y.ctypes.data, int(x.size), C.byref(out)))
    return out.value


def write_sweep_csv(path: str, points: Sequence[SweepPoint]) -> None:
    """write_sweep_csv (eval.hpp:189-198)."""
    n = np.ascontiguousarray([p.n for p in points], dtype=np.int32)
    e = np.ascontiguousarray([p.avg_error for p in points], dtype=np.float64)
    t = np.ascontiguousarray([p.wall_time for p in points], dtype=np.float64)
    check(lib().bsmio_write_sweep_csv(os.fsencode(path), n.ctypes.data, e.ctypes.data, t.ctypes.data, len(points)))


def write_radiometric_csv(path: str, m: RadiometricMatrix) -> None:
    """write_radiometric_csv (eval.hpp:200-211)."""
    r = np.ascontiguousarray(m.rate, dtype=np.float64).reshape(9)
    diag, off = C.c_double(), C.c_double()
    check(lib().bsmio_write_radiometric_csv(os.fsencode(path), r.ctypes.data, C.byref(diag), C.byref(off)))
