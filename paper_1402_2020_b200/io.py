"""Data formats either side of the matching path.

Host-side mirror of the reference's file layer, same behaviour and messages:

* image_io.hpp -- ``load_image`` (PGM P2/P5, PPM P3/P6 at 8/16 bits, PNG),
  ``load_gt_disparity`` (16-bit PGM / PFM / 8-bit gray PNG), ``save_disparity``
  (16-bit PGM of round(d * scale)), ``save_disparity_pfm`` (bottom-up float,
  +inf = invalid), ``save_gray_pgm``, ``save_ppm``;
* JSON sidecars -- ``save_config`` / ``load_config`` (config.hpp:48-110) and
  ``save_pattern`` / ``load_pattern`` (pattern.hpp:104-160), byte-identical to
  nlohmann's ``dump(1, '\\t')`` (sorted keys, tab indent);
* dataset.hpp -- ``load_stereo_dataset``, ``discover_middlebury``,
  ``load_radiometric_set`` (stock Middlebury file names).

PNG: libpng's simplified read API is restated for the variants a stereo
dataset uses (8-bit gray, RGB and palette, non-interlaced); other variants
(16-bit, alpha, interlaced, colour-to-gray) raise FormatError.  Images are
returned as (H, W, 3) uint8 RGB like the reference's RgbImage; ``run_pipeline``
takes grayscale (r = g = b) views on the uint8 path automatically.
"""
from __future__ import annotations

import json
import math
import os
import struct
import sys
import zlib
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import GENERATOR_NAME, BsmConfig, DisparityMap, SamplingPattern
from ._lib import BsmError, InvalidArgument


class IoError(BsmError):
    """bsm::IoError (errors.hpp:12-15): file missing, unreadable or unwritable."""


class FormatError(BsmError):
    """bsm::FormatError (errors.hpp:17-20): corrupt header or truncated payload."""


_SPACE = b" \t\n\v\f\r"


def _read_file(path: str) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError:
        raise IoError(f"cannot open {path}") from None


class _Cursor:
    """PnmCursor (image_io.hpp:33-78): whitespace tokens, '#' comments."""

    def __init__(self, data: bytes):
        self.data = data
        self.pos = 0

    def skip(self):
        d, n = self.data, len(self.data)
        while self.pos < n:
            c = d[self.pos]
            if c == 0x23:  # '#'
                while self.pos < n and d[self.pos] != 0x0A:
                    self.pos += 1
            elif c in _SPACE:
                self.pos += 1
            else:
                break

    def token(self, what: str) -> str:
        self.skip()
        d, n = self.data, len(self.data)
        start = self.pos
        while self.pos < n and d[self.pos] not in _SPACE and d[self.pos] != 0x23:
            self.pos += 1
        if self.pos == start:
            raise FormatError(f"missing {what} in PNM header")
        return d[start:self.pos].decode("latin-1")

    def int_token(self, what: str) -> int:
        t = self.token(what)
        s = t[1:] if t[:1] in "+-" else t
        if not s or not s.isdigit() or not s.isascii():
            if s[:1].isdigit():  # std::stol parsed a prefix: "bad <what> in PNM header"
                raise FormatError(f"bad {what} in PNM header")
            raise FormatError(f"bad {what} '{t}' in PNM header")
        return int(t)

    def expect_single_space(self):
        if self.pos >= len(self.data) or self.data[self.pos] not in _SPACE:
            raise FormatError("missing separator before PNM payload")
        self.pos += 1


def _pnm_header(cur: _Cursor):
    magic = cur.token("magic")
    if len(magic) != 2 or magic[0] != "P" or magic[1] not in "2356":
        raise FormatError(f"unsupported PNM magic '{magic}'")
    w = cur.int_token("width")
    h = cur.int_token("height")
    maxval = cur.int_token("maxval")
    if w < 1 or h < 1 or w > (1 << 20) or h > (1 << 20):
        raise FormatError("bad PNM dimensions")
    if maxval < 1 or maxval > 65535:
        raise FormatError("bad PNM maxval")
    return magic[1], w, h, maxval


def _pnm_samples(cur: _Cursor, magic: str, w: int, h: int, maxval: int, channels: int) -> np.ndarray:
    count = w * h * channels
    if magic in "23":
        out = np.empty(count, np.uint16)
        for i in range(count):
            v = cur.int_token("sample")
            if v < 0 or v > maxval:
                raise FormatError("PNM sample out of range")
            out[i] = v
        return out
    cur.expect_single_space()
    nbytes = 2 if maxval > 255 else 1
    if len(cur.data) - cur.pos < count * nbytes:
        raise FormatError("truncated PNM payload")
    raw = np.frombuffer(cur.data, np.uint8, count * nbytes, cur.pos)
    cur.pos += count * nbytes
    if nbytes == 1:
        return raw.astype(np.uint16)
    return raw.view(">u2").astype(np.uint16)  # big-endian samples


def _to_8bit(v: np.ndarray, maxval: int) -> np.ndarray:
    if maxval == 255:
        return v.astype(np.uint8)
    return ((v.astype(np.int64) * 255 + maxval // 2) // maxval).astype(np.uint8)


# ---------------------------------------------------------------------------
# PNG (restated subset of libpng's simplified read API)
_PNG_SIG = b"\x89PNG\r\n\x1a\n"


def _png_decode(data: bytes, path: str, want_rgb: bool) -> np.ndarray:
    def bad(msg):
        return FormatError(f"bad PNG {path}: {msg}")

    pos = 8
    ihdr = None
    plte = None
    idat = []
    while pos + 8 <= len(data):
        ln, typ = struct.unpack(">I4s", data[pos:pos + 8])
        body = data[pos + 8:pos + 8 + ln]
        if len(body) != ln or pos + 12 + ln > len(data):
            raise bad("truncated chunk")
        crc = struct.unpack(">I", data[pos + 8 + ln:pos + 12 + ln])[0]
        if zlib.crc32(typ + body) & 0xFFFFFFFF != crc:
            raise bad("CRC error")
        if typ == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", body)
        elif typ == b"PLTE":
            plte = np.frombuffer(body, np.uint8).reshape(-1, 3)
        elif typ == b"IDAT":
            idat.append(body)
        elif typ == b"IEND":
            break
        pos += 12 + ln
    if ihdr is None or not idat:
        raise bad("missing IHDR/IDAT")
    w, h, depth, ctype, comp, filt, interlace = ihdr
    if w < 1 or h < 1 or comp != 0 or filt != 0:
        raise bad("invalid IHDR")
    if depth != 8 or ctype not in (0, 2, 3) or interlace != 0:
        raise bad("unsupported PNG variant (this build reads 8-bit gray/RGB/palette, non-interlaced)")
    if ctype == 3 and plte is None:
        raise bad("palette image without PLTE")
    bpp = {0: 1, 2: 3, 3: 1}[ctype]
    try:
        raw = zlib.decompress(b"".join(idat))
    except zlib.error as e:
        raise bad(str(e)) from None
    stride = w * bpp
    if len(raw) < h * (stride + 1):
        raise bad("truncated image data")
    img = np.zeros((h, stride), np.uint8)
    prev = np.zeros(stride, np.int32)
    for y in range(h):
        ft = raw[y * (stride + 1)]
        line = np.frombuffer(raw, np.uint8, stride, y * (stride + 1) + 1).astype(np.int32)
        if ft == 0:
            cur = line
        elif ft == 2:
            cur = (line + prev) & 255
        elif ft == 1:
            cur = (np.cumsum(line.reshape(w, bpp), axis=0) & 255).reshape(-1)
        elif ft in (3, 4):
            cur = np.zeros(stride, np.int32)
            for x in range(stride):
                a = cur[x - bpp] if x >= bpp else 0
                b = prev[x]
                if ft == 3:
                    p = (a + b) >> 1
                else:
                    c = prev[x - bpp] if x >= bpp else 0
                    pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                    p = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
                cur[x] = (line[x] + p) & 255
        else:
            raise bad("bad filter type")
        img[y] = cur
        prev = cur
    if ctype == 3:
        idx = img.reshape(h, w)
        if idx.max(initial=0) >= len(plte):
            raise bad("palette index out of range")
        rgb = plte[idx]
        if not want_rgb:
            raise bad("colour-to-gray conversion is not supported by this build")
        return rgb
    if ctype == 2:
        if not want_rgb:
            raise bad("colour-to-gray conversion is not supported by this build")
        return img.reshape(h, w, 3)
    g = img.reshape(h, w)
    return np.repeat(g[:, :, None], 3, axis=2) if want_rgb else g


# ---------------------------------------------------------------------------
# image_io.hpp
def load_image(path: str) -> np.ndarray:
    """load_image (image_io.hpp:240-263): (H, W, 3) uint8 RGB; gray sources give r = g = b."""
    data = _read_file(path)
    if not data:
        raise FormatError(f"empty file {path}")
    if data[:8] == _PNG_SIG:
        return _png_decode(data, path, want_rgb=True)
    cur = _Cursor(data)
    magic, w, h, maxval = _pnm_header(cur)
    color = magic in "36"
    s = _to_8bit(_pnm_samples(cur, magic, w, h, maxval, 3 if color else 1), maxval)
    if color:
        return s.reshape(h, w, 3)
    g = s.reshape(h, w)
    return np.repeat(g[:, :, None], 3, axis=2)


def _parse_pfm(data: bytes, path: str):
    cur = _Cursor(data)
    magic = cur.token("magic")
    if magic not in ("Pf", "PF"):
        raise FormatError(f"bad PFM magic in {path}")
    ch = 3 if magic == "PF" else 1
    w = cur.int_token("width")
    h = cur.int_token("height")
    if w < 1 or h < 1 or w > (1 << 20) or h > (1 << 20):
        raise FormatError(f"bad PFM dimensions in {path}")
    tok = cur.token("scale")
    try:
        scale = float(tok)
    except ValueError:
        raise FormatError(f"bad PFM scale in {path}") from None
    if scale == 0:
        raise FormatError(f"bad PFM scale in {path}")
    cur.expect_single_space()
    count = w * h * ch
    if len(data) - cur.pos < count * 4:
        raise FormatError(f"truncated PFM payload in {path}")
    vals = np.frombuffer(data, ">f4" if scale > 0 else "<f4", count, cur.pos).astype(np.float32)
    return w, h, ch, vals.reshape(h, w * ch)[::-1].reshape(-1)  # rows are stored bottom-up


def load_gt_disparity(path: str, scale: float) -> DisparityMap:
    """load_gt_disparity (image_io.hpp:268-314): stored value / scale; PGM 0 and
    non-finite PFM values are unknown."""
    if not scale > 0:
        raise InvalidArgument("disparity scale must be > 0")
    data = _read_file(path)
    if not data:
        raise FormatError(f"empty file {path}")
    if len(data) >= 2 and data[0] == 0x50 and data[1] in (0x66, 0x46):
        w, h, ch, vals = _parse_pfm(data, path)
        if ch != 1:
            raise FormatError(f"disparity PFM must be grayscale: {path}")
        fin = np.isfinite(vals)
        d = np.where(fin, (vals.astype(np.float64) / scale).astype(np.float32), np.float32(0)).astype(np.float32)
        return DisparityMap(d.reshape(h, w), fin.astype(np.uint8).reshape(h, w))
    if data[:8] == _PNG_SIG:
        stored = _png_decode(data, path, want_rgb=False).astype(np.uint16)
        h, w = stored.shape
        stored = stored.reshape(-1)
    else:
        cur = _Cursor(data)
        magic, w, h, maxval = _pnm_header(cur)
        if magic in "36":
            raise FormatError(f"disparity PGM must be grayscale: {path}")
        stored = _pnm_samples(cur, magic, w, h, maxval, 1)
    ok = stored != 0
    d = np.where(ok, (stored.astype(np.float64) / scale).astype(np.float32), np.float32(0)).astype(np.float32)
    return DisparityMap(d.reshape(h, w), ok.astype(np.uint8).reshape(h, w))


def _write(path: str, payload: bytes) -> None:
    try:
        with open(path, "wb") as f:
            f.write(payload)
    except OSError:
        raise IoError(f"cannot open {path} for writing") from None


def _round_half_away(x: np.ndarray) -> np.ndarray:
    """std::round / std::lround: nearest, halves away from zero (exact: trunc + fraction test)."""
    t = np.trunc(x)
    return t + np.sign(x) * (np.abs(x - t) >= 0.5)


def save_disparity(m: DisparityMap, path: str, scale: float) -> None:
    """save_disparity (image_io.hpp:317-337): 16-bit PGM of lround(d * scale), invalid = 0."""
    if scale <= 0:
        raise InvalidArgument("disparity scale must be > 0")
    v = _round_half_away(m.disparity.astype(np.float64) * float(scale))
    v = np.clip(v, 0, 65535)
    v = np.where(m.valid != 0, v, 0).astype(">u2")
    _write(path, f"P5\n{m.width} {m.height}\n65535\n".encode() + v.tobytes())


def save_disparity_pfm(m: DisparityMap, path: str) -> None:
    """save_disparity_pfm (image_io.hpp:340-355): grayscale PFM, bottom-up, +inf invalid."""
    big = sys.byteorder == "big"
    d = np.where(m.valid != 0, m.disparity, np.float32(np.inf)).astype(np.float32)
    hdr = f"Pf\n{m.width} {m.height}\n{'1.0' if big else '-1.0'}\n".encode()
    _write(path, hdr + np.ascontiguousarray(d[::-1]).astype("=f4").tobytes())


def save_gray_pgm(gray: np.ndarray, path: str) -> None:
    """save_gray_pgm (image_io.hpp:358-371): 8-bit PGM of round(v) clamped to [0, 255]."""
    g = np.asarray(gray, np.float32)
    h, w = g.shape
    r = np.clip(_round_half_away(g), 0, 255).astype(np.uint8)
    _write(path, f"P5\n{w} {h}\n255\n".encode() + r.tobytes())


def save_ppm(rgb: np.ndarray, path: str) -> None:
    """save_ppm (image_io.hpp:373-382)."""
    a = np.ascontiguousarray(rgb, np.uint8)
    h, w = a.shape[:2]
    _write(path, f"P6\n{w} {h}\n255\n".encode() + a.tobytes())


# ---------------------------------------------------------------------------
# JSON sidecars (nlohmann dump(1, '\t'): keys sorted, one tab per level)
def _dump(obj) -> bytes:
    return (json.dumps(obj, indent="\t", sort_keys=True, ensure_ascii=False) + "\n").encode()


def save_config(cfg: BsmConfig, path: str) -> None:
    """save_config (config.hpp:81-86)."""
    obj = {"n": int(cfg.n), "S": int(cfg.window), "spread": float(cfg.spread), "seed": int(cfg.seed),
           "d_max": int(cfg.d_max), "lambda_c": float(cfg.lambda_c), "lambda_e": float(cfg.lambda_e),
           "lr_tolerance": float(cfg.lr_tolerance), "vote_radius": int(cfg.vote_radius),
           "gt_scale": float(cfg.gt_scale), "threads": int(cfg.threads), "generator": str(cfg.generator)}
    _write(path, _dump(obj))


def _load_json(path: str, what: str):
    data = _read_file(path)
    try:
        return json.loads(data.decode("utf-8"))
    except (ValueError, UnicodeDecodeError) as e:
        raise FormatError(f"bad {what} file {path}: {e}") from None


def load_config(path: str) -> BsmConfig:
    """load_config (config.hpp:88-101); missing keys keep their defaults."""
    j = _load_json(path, "config")
    if not isinstance(j, dict):
        raise FormatError(f"bad config file {path}: not an object")
    c = BsmConfig()
    spec = [("n", "n", int), ("S", "window", int), ("spread", "spread", float), ("seed", "seed", int),
            ("d_max", "d_max", int), ("lambda_c", "lambda_c", float), ("lambda_e", "lambda_e", float),
            ("lr_tolerance", "lr_tolerance", float), ("vote_radius", "vote_radius", int),
            ("gt_scale", "gt_scale", float), ("threads", "threads", int), ("generator", "generator", str)]
    for key, attr, typ in spec:
        if key not in j:
            continue
        v = j[key]
        if typ is str:
            if not isinstance(v, str):
                raise FormatError(f"bad config file {path}: '{key}' must be a string")
        elif isinstance(v, bool) or not isinstance(v, (int, float)):
            raise FormatError(f"bad config file {path}: '{key}' must be a number")
        elif typ is int:
            v = int(v)
        else:
            v = float(v)
        setattr(c, attr, v)
    return c


def save_pattern(p: SamplingPattern, path: str) -> None:
    """save_pattern (pattern.hpp:106-121): generator, parameters and the offset list."""
    # the sidecar writer prints each offset quadruple on one line ("[px,py,qx,qy]")
    rows = ",\n".join("\t\t[" + ",".join(str(int(v)) for v in row) + "]" for row in np.asarray(p.pairs)[: p.n])
    obj = {"generator": GENERATOR_NAME, "n": int(p.n), "S": int(p.window), "spread": float(p.spread),
           "seed": int(p.seed), "pairs": "@PAIRS@"}
    text = _dump(obj).decode().replace('"@PAIRS@"', "[\n" + rows + "\n\t]")
    _write(path, text.encode())


def load_pattern(path: str) -> SamplingPattern:
    """load_pattern (pattern.hpp:123-158)."""
    j = _load_json(path, "pattern")
    try:
        gen = j["generator"]
        if gen != GENERATOR_NAME:
            raise FormatError(f"pattern file {path} uses unknown generator '{gen}'")
        n, window, spread, seed = int(j["n"]), int(j["S"]), float(j["spread"]), int(j["seed"])
        pairs = j["pairs"]
        if len(pairs) != n:
            raise FormatError(f"pattern file {path}: pair count does not match n")
        half = window // 2
        arr = np.zeros((max(n, 1), 4), np.int16)
        for i, e in enumerate(pairs):
            q = [int(e[k]) for k in range(4)]
            if any(v < -half or v > half for v in q):
                raise FormatError(f"pattern file {path}: offset outside window")
            arr[i] = q
    except (KeyError, IndexError, TypeError, ValueError) as e:
        raise FormatError(f"bad pattern file {path}: {e}") from None
    return SamplingPattern(n, window, spread, seed, arr)


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
