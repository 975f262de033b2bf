"""Data formats either side of the matching path.

Python binding of the file layer implemented once, in C++ (include/bsm/
image_io.hpp, config.hpp, pattern.hpp; C ABI include/bsm_io.h in
``libbsm_io.so``) -- the same behaviour and messages as the reference:

* image_io.hpp -- ``load_image`` (PGM P2/P5, PPM P3/P6 at 8/16 bits, PNG),
  ``load_gt_disparity`` (16-bit PGM / PFM / 8-bit gray PNG), ``save_disparity``
  (16-bit PGM of round(d * scale)), ``save_disparity_pfm`` (bottom-up float,
  +inf = invalid), ``save_gray_pgm``, ``save_ppm``;
* JSON sidecars -- ``save_config`` / ``load_config`` (config.hpp:48-110) and
  ``save_pattern`` / ``load_pattern`` (pattern.hpp:104-160), byte-identical to
  the reference's nlohmann ``dump(1, '\\t')``;
* dataset.hpp -- ``load_stereo_dataset``, ``discover_middlebury``,
  ``load_radiometric_set`` (stock Middlebury file names), composed here from
  the readers.

PNG: 8-bit gray, RGB and palette, non-interlaced (zlib); other variants
(16-bit, alpha, interlaced, colour-to-gray) raise FormatError.  Images are
returned as (H, W, 3) uint8 RGB like the reference's RgbImage; ``run_pipeline``
takes grayscale (r = g = b) views on the uint8 path automatically.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import BsmConfig, DisparityMap, SamplingPattern
from ._lib import BsmError, DimensionMismatch, InvalidArgument


class IoError(BsmError):
    """bsm::IoError (errors.hpp:12-15): file missing, unreadable or unwritable."""


class FormatError(BsmError):
    """bsm::FormatError (errors.hpp:17-20): corrupt header or truncated payload."""


class EmptyRegion(BsmError):
    """bsm::EmptyRegion (eval.hpp): no pixel of the evaluation region has ground truth."""


IO_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbsm_io.so")
_P, _I, _D = C.c_void_p, C.c_int, C.c_double
_SIGS = {
    "bsmio_load_image": [C.c_char_p, C.POINTER(_I), C.POINTER(_I), _P],
    "bsmio_load_gt": [C.c_char_p, _D, C.POINTER(_I), C.POINTER(_I), _P, _P],
    "bsmio_save_disparity": [C.c_char_p, _P, _P, _I, _I, _D, _I],
    "bsmio_save_gray_pgm": [C.c_char_p, _P, _I, _I],
    "bsmio_save_ppm": [C.c_char_p, _P, _I, _I],
    "bsmio_save_config": [C.c_char_p, _P, _P, C.c_char_p],
    "bsmio_load_config": [C.c_char_p, _P, _P, C.c_char_p, _I],
    "bsmio_save_pattern": [C.c_char_p, _P, _I, _I, _D, C.c_uint64],
    "bsmio_load_pattern": [C.c_char_p, C.POINTER(_I), C.POINTER(_I), C.POINTER(_D), C.POINTER(C.c_uint64), _P, _I],
    "bsmio_bad_pixel_rate": [_P, _P, _P, _P, _P, _I, _I, _D, C.POINTER(_D), C.POINTER(C.c_long),
                             C.POINTER(C.c_long)],
    "bsmio_linear_fit_r2": [_P, _P, _I, C.POINTER(_D)],
    "bsmio_write_sweep_csv": [C.c_char_p, _P, _P, _P, _I],
    "bsmio_write_radiometric_csv": [C.c_char_p, _P, C.POINTER(_D), C.POINTER(_D)],
}
_io = None


def lib() -> C.CDLL:
    """Load libbsm_io.so (built with the product by __graft_entry__.build())."""
    global _io
    if _io is None:
        if not os.path.exists(IO_PATH):
            raise BsmError(f"{IO_PATH} is missing: run __graft_entry__.build()")
        L = C.CDLL(IO_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.bsmio_last_error.argtypes = []
        L.bsmio_last_error.restype = C.c_char_p
        _io = L
    return _io


_EXC = {1: InvalidArgument, 2: DimensionMismatch, 10: IoError, 11: FormatError, 12: EmptyRegion}


def check(rc: int) -> None:
    if rc:
        raise _EXC.get(rc, BsmError)(lib().bsmio_last_error().decode(errors="replace"))


def _b(path: str) -> bytes:
    return os.fsencode(path)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# image_io.hpp
def load_image(path: str) -> np.ndarray:
    """load_image (image_io.hpp:240-263): (H, W, 3) uint8 RGB; gray sources
    expand to r = g = b, 16-bit samples rescale to 8 bits."""
    w, h = C.c_int(), C.c_int()
    check(lib().bsmio_load_image(_b(path), C.byref(w), C.byref(h), None))
    out = np.empty((h.value, w.value, 3), np.uint8)
    check(lib().bsmio_load_image(_b(path), C.byref(w), C.byref(h), _ptr(out)))
    return out


def load_gt_disparity(path: str, scale: float) -> DisparityMap:
    """load_gt_disparity (image_io.hpp:268-314): stored value / scale; PGM 0 and
    non-finite PFM values are unknown."""
    w, h = C.c_int(), C.c_int()
    check(lib().bsmio_load_gt(_b(path), float(scale), C.byref(w), C.byref(h), None, None))
    d = np.empty((h.value, w.value), np.float32)
    v = np.empty((h.value, w.value), np.uint8)
    check(lib().bsmio_load_gt(_b(path), float(scale), C.byref(w), C.byref(h), _ptr(d), _ptr(v)))
    return DisparityMap(d, v)


def _map(m: DisparityMap):
    return (np.ascontiguousarray(m.disparity, dtype=np.float32), np.ascontiguousarray(m.valid, dtype=np.uint8))


def save_disparity(m: DisparityMap, path: str, scale: float) -> None:
    """save_disparity (image_io.hpp:317-337): 16-bit PGM of round(d * scale), 0 = invalid."""
    d, v = _map(m)
    check(lib().bsmio_save_disparity(_b(path), _ptr(d), _ptr(v), d.shape[1], d.shape[0], float(scale), 0))


def save_disparity_pfm(m: DisparityMap, path: str) -> None:
    """save_disparity_pfm (image_io.hpp:340-355): bottom-up float, +inf = invalid."""
    d, v = _map(m)
    check(lib().bsmio_save_disparity(_b(path), _ptr(d), _ptr(v), d.shape[1], d.shape[0], 1.0, 1))


def save_gray_pgm(gray: np.ndarray, path: str) -> None:
    """save_gray_pgm (image_io.hpp:358-371)."""
    g = np.ascontiguousarray(gray, dtype=np.float32)
    check(lib().bsmio_save_gray_pgm(_b(path), _ptr(g), g.shape[1], g.shape[0]))


def save_ppm(rgb: np.ndarray, path: str) -> None:
    """save_ppm (image_io.hpp:373-382)."""
    a = np.ascontiguousarray(rgb, dtype=np.uint8)
    if a.ndim != 3 or a.shape[2] != 3:
        raise InvalidArgument("save_ppm: expected an (H, W, 3) uint8 image")
    check(lib().bsmio_save_ppm(_b(path), _ptr(a), a.shape[1], a.shape[0]))


# ---------------------------------------------------------------------------
# JSON sidecars (config.hpp, pattern.hpp)
def save_config(cfg: BsmConfig, path: str) -> None:
    """save_config (config.hpp:81-86)."""
    iv = np.array([cfg.n, cfg.window, cfg.seed, cfg.d_max, cfg.vote_radius, cfg.threads], np.int64)
    dv = np.array([cfg.spread, cfg.lambda_c, cfg.lambda_e, cfg.lr_tolerance, cfg.gt_scale], np.float64)
    check(lib().bsmio_save_config(_b(path), _ptr(iv), _ptr(dv), str(cfg.generator).encode()))


def load_config(path: str) -> BsmConfig:
    """load_config (config.hpp:88-101); missing keys keep their defaults."""
    iv = np.zeros(6, np.int64)
    dv = np.zeros(5, np.float64)
    gen = C.create_string_buffer(4096)
    check(lib().bsmio_load_config(_b(path), _ptr(iv), _ptr(dv), gen, 4096))
    return BsmConfig(n=int(iv[0]), window=int(iv[1]), seed=int(iv[2]), d_max=int(iv[3]), vote_radius=int(iv[4]),
                     threads=int(iv[5]), spread=float(dv[0]), lambda_c=float(dv[1]), lambda_e=float(dv[2]),
                     lr_tolerance=float(dv[3]), gt_scale=float(dv[4]), generator=gen.value.decode())


def save_pattern(p: SamplingPattern, path: str) -> None:
    """save_pattern (pattern.hpp:106-121): generator, parameters and the offset list."""
    pairs = np.ascontiguousarray(np.asarray(p.pairs, dtype=np.int16).reshape(-1, 4)[: p.n])
    check(lib().bsmio_save_pattern(_b(path), _ptr(pairs), int(p.n), int(p.window), float(p.spread),
                                   C.c_uint64(int(p.seed))))


def load_pattern(path: str) -> SamplingPattern:
    """load_pattern (pattern.hpp:123-158)."""
    n, w, sp, sd = C.c_int(), C.c_int(), C.c_double(), C.c_uint64()
    check(lib().bsmio_load_pattern(_b(path), C.byref(n), C.byref(w), C.byref(sp), C.byref(sd), None, 0))
    arr = np.zeros((max(n.value, 1), 4), np.int16)
    check(lib().bsmio_load_pattern(_b(path), C.byref(n), C.byref(w), C.byref(sp), C.byref(sd), _ptr(arr),
                                   n.value))
    return SamplingPattern(n.value, w.value, sp.value, sd.value, arr)


# ---------------------------------------------------------------------------
# dataset.hpp
@dataclass
class StereoDataset:
    """StereoDataset (dataset.hpp:15-27)."""

    name: str
    left: np.ndarray
    right: np.ndarray
    gt: DisparityMap
    mask_nonocc: Optional[np.ndarray]
    mask_all: Optional[np.ndarray]
    mask_disc: Optional[np.ndarray]
    d_max: int
    gt_scale: float


# name, d_max, gt_scale (dataset.hpp:35-41)
MIDDLEBURY_SCENES = (("tsukuba", 16, 16.0), ("venus", 20, 8.0), ("teddy", 60, 4.0), ("cones", 60, 4.0))


def _find(root: str, names: Sequence[str]) -> Optional[str]:
    for nm in names:
        p = os.path.join(root, nm)
        if os.path.exists(p):
            return p
    return None


def _mask(root: str, names: Sequence[str]) -> Optional[np.ndarray]:
    p = _find(root, names)
    if p is None:
        return None
    from . import to_gray_lab
    g, _ = to_gray_lab(load_image(p))  # to_gray(load_image(...)), dataset.hpp:57-63
    return g


def load_stereo_dataset(root: str, name: str, d_max: int, gt_scale: float) -> StereoDataset:
    """load_stereo_dataset (dataset.hpp:67-90)."""
    left = _find(root, ["im2.png", "im2.ppm", "im2.pgm", "left.png", "left.ppm", "left.pgm"])
    right = _find(root, ["im6.png", "im6.ppm", "im6.pgm", "right.png", "right.ppm", "right.pgm"])
    gt = _find(root, ["disp2.pgm", "disp2.png", "disp2.pfm", "gt.pgm", "gt.png", "gt.pfm"])
    if not (left and right and gt):
        raise IoError(f"dataset {root}: need left (im2.*), right (im6.*) and ground truth (disp2.*)")
    return StereoDataset(name, load_image(left), load_image(right), load_gt_disparity(gt, gt_scale),
                         _mask(root, ["nonocc.png", "nonocc.pgm"]), _mask(root, ["all.png", "all.pgm"]),
                         _mask(root, ["disc.png", "disc.pgm"]), int(d_max), float(gt_scale))


def discover_middlebury(root: str) -> List[StereoDataset]:
    """discover_middlebury (dataset.hpp:93-103)."""
    out = []
    for name, d_max, scale in MIDDLEBURY_SCENES:
        d = os.path.join(root, name)
        if os.path.isdir(d):
            out.append(load_stereo_dataset(d, name, d_max, scale))
    return out


@dataclass
class RadiometricSet:
    """RadiometricSet (dataset.hpp:107-117)."""

    lefts: List[np.ndarray]
    rights: List[np.ndarray]
    gt: DisparityMap
    mask_nonocc: Optional[np.ndarray]
    mask_all: Optional[np.ndarray]
    mask_disc: Optional[np.ndarray]
    d_max: int
    gt_scale: float


def load_radiometric_set(root: str, d_max: int, gt_scale: float) -> RadiometricSet:
    """load_radiometric_set (dataset.hpp:120-141): left_c0..2, right_c0..2, gt."""
    lefts, rights = [], []
    for c in range(3):
        ln, rn = f"left_c{c}", f"right_c{c}"
        lp = _find(root, [ln + ".png", ln + ".ppm", ln + ".pgm"])
        rp = _find(root, [rn + ".png", rn + ".ppm", rn + ".pgm"])
        if not lp:
            raise IoError(f"radiometric set {root}: missing {ln}.{{png,ppm,pgm}}")
        if not rp:
            raise IoError(f"radiometric set {root}: missing {rn}.{{png,ppm,pgm}}")
        lefts.append(load_image(lp))
        rights.append(load_image(rp))
    gt = _find(root, ["gt.pgm", "gt.pfm", "gt.png", "disp2.pgm"])
    if not gt:
        raise IoError(f"radiometric set {root}: missing gt.{{pgm,pfm,png}}")
    return RadiometricSet(lefts, rights, load_gt_disparity(gt, gt_scale),
                          _mask(root, ["nonocc.png", "nonocc.pgm"]), _mask(root, ["all.png", "all.pgm"]),
                          _mask(root, ["disc.png", "disc.pgm"]), int(d_max), float(gt_scale))
