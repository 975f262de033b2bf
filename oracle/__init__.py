"""TEST INFRASTRUCTURE ONLY -- the checkers the CUDA path is compared against.

Two CPU implementations of the hot path, loaded with ctypes:

* ``Restatement`` -- oracle/bsm_oracle.c, an independent C restatement of the
  reference algorithm (built to oracle/_build/libbsm_oracle.so);
* ``Reference`` -- the UNMODIFIED reference headers compiled in place by
  oracle/Makefile (oracle/_ref/libbsm_ref_native.so, or the portable
  _v3 build when the host lacks the native build's ISA extensions).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package; the product (paper_1402_2020_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_PATH = os.path.join(HERE, "_build", "libbsm_oracle.so")
REF_NATIVE_PATH = os.path.join(HERE, "_ref", "libbsm_ref_native.so")
REF_V3_PATH = os.path.join(HERE, "_ref", "libbsm_ref_v3.so")

_P = C.c_void_p
_I = C.c_int
_D = C.c_double


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _host_isa() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def ref_path() -> str:
    """Native build when every ISA extension it was built with is present."""
    isa_file = os.path.join(HERE, "_ref", "native_isa.txt")
    if os.path.exists(REF_NATIVE_PATH) and os.path.exists(isa_file):
        need = set(open(isa_file).read().split())
        have = _host_isa()
        # /proc/cpuinfo spells some flags differently (avx512_vpopcntdq vs avx512vpopcntdq)
        norm = lambda s: {x.replace("_", "") for x in s}
        if norm(need) <= norm(have):
            return REF_NATIVE_PATH
    return REF_V3_PATH


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.path = path
        self.L = C.CDLL(path)
        self.prefix = prefix

    def f(self, name, argtypes, restype=C.c_int):
        fn = getattr(self.L, self.prefix + name)
        fn.argtypes = argtypes
        fn.restype = restype
        return fn


class Restatement(_Lib):
    """oracle/bsm_oracle.c"""

    def __init__(self):
        super().__init__(RESTATEMENT_PATH, "oracle_")

    def generate_pattern(self, n, window, spread, seed):
        out = np.zeros((n, 4), np.int16)
        rc = self.f("generate_pattern", [_I, _I, _D, C.c_uint64, _P])(n, window, spread, seed, _p(out))
        assert rc == 0
        return out

    def gray_lab_lut(self):
        g = np.zeros(256, np.float32)
        l = np.zeros((256, 3), np.float32)
        self.f("gray_lab_lut", [_P, _P], None)(_p(g), _p(l))
        return g, l

    def to_gray_lab(self, rgb):
        rgb = np.ascontiguousarray(rgb, np.uint8)
        H, W = rgb.shape[:2]
        g = np.zeros((H, W), np.float32)
        l = np.zeros((H, W, 3), np.float32)
        self.f("to_gray_lab", [_P, _I, _I, _P, _P], None)(_p(rgb), W, H, _p(g), _p(l))
        return g, l

    def compute_field_u8(self, img, pairs, window):
        img = np.ascontiguousarray(img, np.uint8)
        H, W = img.shape
        n = pairs.shape[0]
        words = (n + 63) // 64
        d = np.zeros((H, W, words), np.uint64)
        m = np.zeros((H, W, words), np.uint64)
        rc = self.f("compute_field_u8", [_P, _I, _I, _P, _I, _I, _P, _P])(
            _p(img), W, H, _p(np.ascontiguousarray(pairs, np.int16)), n, window, _p(d), _p(m))
        assert rc == 0
        return d, m

    def quarter_threshold(self, w):
        w = np.ascontiguousarray(w, np.float32)
        return self.f("quarter_threshold", [_P, _I], C.c_float)(_p(w), len(w))

    def masked_hamming_words(self, a, b, m):
        a, b, m = (np.ascontiguousarray(x, np.uint64) for x in (a, b, m))
        return self.f("masked_hamming_words", [_P, _P, _P, _I])(_p(a), _p(b), _p(m), len(a))

    def wta(self, dref, mref, doth, n, d_max, right_ref, use_mask=True):
        H, W, _ = dref.shape
        out = np.zeros((H, W), np.float32)
        rc = self.f("wta", [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P])(
            _p(dref), _p(mref), _p(doth), W, H, n, d_max, int(right_ref), int(use_mask), _p(out))
        assert rc == 0
        return out

    def lr_check(self, dl, dr, tol):
        H, W = dl.shape
        od = np.zeros((H, W), np.float32)
        ov = np.zeros((H, W), np.uint8)
        self.f("lr_check", [_P, _P, _I, _I, _D, _P, _P])(
            _p(np.ascontiguousarray(dl, np.float32)), _p(np.ascontiguousarray(dr, np.float32)), W, H, tol,
            _p(od), _p(ov))
        return od, ov

    def vote_refine(self, d, v, lab, lc, le, radius):
        H, W = d.shape
        od = np.zeros((H, W), np.float32)
        ov = np.zeros((H, W), np.uint8)
        self.f("vote_refine", [_P, _P, _P, _I, _I, _D, _D, _I, _P, _P])(
            _p(np.ascontiguousarray(d, np.float32)), _p(np.ascontiguousarray(v, np.uint8)),
            _p(np.ascontiguousarray(lab, np.float32)), W, H, lc, le, radius, _p(od), _p(ov))
        return od, ov

    def vote_weight(self, lx, lp, dx, dy, lc, le):
        lx = np.ascontiguousarray(lx, np.float32)
        lp = np.ascontiguousarray(lp, np.float32)
        return self.f("vote_weight", [_P, _P, _I, _I, _D, _D], C.c_double)(_p(lx), _p(lp), dx, dy, lc, le)

    def pipeline_u8(self, left, right, pairs, window, d_max, lc=9.0, le=16.0, tol=1.0, radius=20):
        H, W = left.shape
        out = {k: np.zeros((H, W), np.float32) for k in ("refined_d", "left_d", "right_d", "checked_d")}
        out.update({k: np.zeros((H, W), np.uint8) for k in ("refined_v", "checked_v")})
        rc = self.f("pipeline_u8", [_P, _P, _I, _I, _P, _I, _I, _I, _D, _D, _D, _I] + [_P] * 6)(
            _p(np.ascontiguousarray(left, np.uint8)), _p(np.ascontiguousarray(right, np.uint8)), W, H,
            _p(np.ascontiguousarray(pairs, np.int16)), pairs.shape[0], window, d_max, lc, le, tol, radius,
            _p(out["refined_d"]), _p(out["refined_v"]), _p(out["left_d"]), _p(out["right_d"]),
            _p(out["checked_d"]), _p(out["checked_v"]))
        assert rc == 0
        return out


class Reference(_Lib):
    """The reference library compiled in place (oracle/_ref)."""

    def __init__(self, path: str | None = None):
        super().__init__(path or ref_path(), "ref_")

    def err(self):
        return self.f("last_error", [], C.c_char_p)().decode()

    def generate_pattern(self, n, window, spread, seed):
        out = np.zeros((n, 4), np.int16)
        rc = self.f("generate_pattern", [_I, _I, _D, C.c_uint64, _P])(n, window, spread, seed, _p(out))
        if rc:
            raise ValueError(self.err())
        return out

    def gray_lab_lut(self):
        g = np.zeros(256, np.float32)
        l = np.zeros((256, 3), np.float32)
        self.f("gray_lab_lut", [_P, _P], None)(_p(g), _p(l))
        return g, l

    def to_gray_lab(self, rgb):
        rgb = np.ascontiguousarray(rgb, np.uint8)
        H, W = rgb.shape[:2]
        g = np.zeros((H, W), np.float32)
        l = np.zeros((H, W, 3), np.float32)
        self.f("to_gray_lab", [_P, _I, _I, _P, _P], None)(_p(rgb), W, H, _p(g), _p(l))
        return g, l

    def compute_field_u8(self, img, pairs, window, threads=1):
        img = np.ascontiguousarray(img, np.uint8)
        H, W = img.shape
        n = pairs.shape[0]
        words = (n + 63) // 64
        d = np.zeros((H, W, words), np.uint64)
        m = np.zeros((H, W, words), np.uint64)
        rc = self.f("compute_field_u8", [_P, _I, _I, _P, _I, _I, _I, _P, _P])(
            _p(img), W, H, _p(np.ascontiguousarray(pairs, np.int16)), n, window, threads, _p(d), _p(m))
        if rc:
            raise ValueError(self.err())
        return d, m

    def compute_field(self, gray, lab, pairs, window, threads=1):
        """compute_field (descriptor.hpp:200) of float gray / Lab planes."""
        gray = np.ascontiguousarray(gray, np.float32)
        lab = np.ascontiguousarray(lab, np.float32)
        H, W = gray.shape
        n = pairs.shape[0]
        words = (n + 63) // 64
        d = np.zeros((H, W, words), np.uint64)
        m = np.zeros((H, W, words), np.uint64)
        rc = self.f("compute_field", [_P, _P, _I, _I, _P, _I, _I, _I, _P, _P])(
            _p(gray), _p(lab), W, H, _p(np.ascontiguousarray(pairs, np.int16)), n, window, threads, _p(d), _p(m))
        if rc:
            raise ValueError(self.err())
        return d, m

    def quarter_threshold(self, w):
        w = np.ascontiguousarray(w, np.float32)
        return self.f("quarter_threshold", [_P, _I], C.c_float)(_p(w), len(w))

    def masked_hamming_words(self, a, b, m):
        a, b, m = (np.ascontiguousarray(x, np.uint64) for x in (a, b, m))
        return self.f("masked_hamming_words", [_P, _P, _P, _I])(_p(a), _p(b), _p(m), len(a))

    def wta(self, dref, mref, doth, n, d_max, right_ref, use_mask=True, threads=1):
        H, W, _ = dref.shape
        out = np.zeros((H, W), np.float32)
        rc = self.f("wta", [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P])(
            _p(dref), _p(mref), _p(doth), W, H, n, d_max, int(right_ref), int(use_mask), threads, _p(out))
        if rc:
            raise ValueError(self.err())
        return out

    def lr_check(self, dl, dr, tol):
        H, W = dl.shape
        od = np.zeros((H, W), np.float32)
        ov = np.zeros((H, W), np.uint8)
        ones = np.ones((H, W), np.uint8)
        rc = self.f("lr_check", [_P, _P, _P, _P, _I, _I, _D, _P, _P])(
            _p(np.ascontiguousarray(dl, np.float32)), _p(ones), _p(np.ascontiguousarray(dr, np.float32)),
            _p(ones), W, H, tol, _p(od), _p(ov))
        if rc:
            raise ValueError(self.err())
        return od, ov

    def vote_refine(self, d, v, lab, lc, le, radius, threads=1):
        H, W = d.shape
        od = np.zeros((H, W), np.float32)
        ov = np.zeros((H, W), np.uint8)
        rc = self.f("vote_refine", [_P, _P, _P, _I, _I, _D, _D, _D, _I, _I, _P, _P])(
            _p(np.ascontiguousarray(d, np.float32)), _p(np.ascontiguousarray(v, np.uint8)),
            _p(np.ascontiguousarray(lab, np.float32)), W, H, lc, le, 1.0, radius, threads, _p(od), _p(ov))
        if rc:
            raise ValueError(self.err())
        return od, ov

    def vote_weight(self, lx, lp, dx, dy, lc, le):
        lx = np.ascontiguousarray(lx, np.float32)
        lp = np.ascontiguousarray(lp, np.float32)
        return self.f("vote_weight", [_P, _P, _I, _I, _D, _D], C.c_double)(_p(lx), _p(lp), dx, dy, lc, le)

    def synth_pair(self, config, seed, width, height):
        """(left, right) uint8 views of a BASELINE synthetic pair (the generator
        compiled into this library, so callers load no product library)."""
        left = np.empty((height, width), np.uint8)
        right = np.empty((height, width), np.uint8)
        rc = self.f("synth_pair", [_I, C.c_uint64, _I, _I, _P, _P, _P])(
            int(config), int(seed), int(width), int(height), _p(left), _p(right), None)
        if rc:
            raise ValueError("synth_pair: bad arguments")
        return left, right

    def pipeline(self, left, right, pairs, window, d_max, lc=9.0, le=16.0, tol=1.0, radius=20, threads=1,
                 want_unmasked=False, channels=1):
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        H, W = left.shape[:2]
        out = {k: np.zeros((H, W), np.float32) for k in ("refined_d", "left_d", "right_d", "checked_d",
                                                           "unmasked_d")}
        out.update({k: np.zeros((H, W), np.uint8) for k in ("refined_v", "checked_v")})
        secs = C.c_double()
        rc = self.f("pipeline", [_P, _P, _I, _I, _I, _P, _I, _I, _I, _D, _D, _D, _I, _I, _I] + [_P] * 8)(
            _p(left), _p(right), channels, W, H, _p(np.ascontiguousarray(pairs, np.int16)), pairs.shape[0],
            window, d_max, lc, le, tol, radius, threads, int(want_unmasked), _p(out["refined_d"]),
            _p(out["refined_v"]), _p(out["left_d"]), _p(out["right_d"]), _p(out["checked_d"]),
            _p(out["checked_v"]), _p(out["unmasked_d"]), C.byref(secs))
        if rc:
            raise ValueError(self.err())
        out["seconds"] = secs.value
        return out


REF_IO_PATH = os.path.join(HERE, "_ref", "libbsm_ref_io.so")


class RefIO(_Lib):
    """image_io.hpp / eval.hpp / JSON sidecars of the reference (oracle/ref_io_driver.cpp)."""

    ERR = {10: "IoError", 11: "FormatError", 1: "InvalidArgument", 2: "DimensionMismatch", 12: "EmptyRegion",
           9: "Error"}

    def __init__(self, path: str | None = None, prefix: str = "refio_"):
        super().__init__(path or REF_IO_PATH, prefix)

    def _raise(self, rc):
        msg = self.f("last_error", [], C.c_char_p)().decode()
        raise RefIOError(self.ERR.get(rc, "Error"), msg)

    def load_image(self, path):
        w, h = C.c_int(), C.c_int()
        fn = self.f("load_image", [C.c_char_p, _P, _P, _P])
        rc = fn(path.encode(), C.byref(w), C.byref(h), None)
        if rc:
            self._raise(rc)
        out = np.zeros((h.value, w.value, 3), np.uint8)
        fn(path.encode(), C.byref(w), C.byref(h), _p(out))
        return out

    def load_gt(self, path, scale):
        w, h = C.c_int(), C.c_int()
        fn = self.f("load_gt", [C.c_char_p, _D, _P, _P, _P, _P])
        rc = fn(path.encode(), scale, C.byref(w), C.byref(h), None, None)
        if rc:
            self._raise(rc)
        d = np.zeros((h.value, w.value), np.float32)
        v = np.zeros((h.value, w.value), np.uint8)
        fn(path.encode(), scale, C.byref(w), C.byref(h), _p(d), _p(v))
        return d, v

    def save_disparity(self, path, d, v, scale, pfm=False):
        d = np.ascontiguousarray(d, np.float32)
        v = np.ascontiguousarray(v, np.uint8)
        rc = self.f("save_disparity", [C.c_char_p, _P, _P, _I, _I, _D, _I])(
            path.encode(), _p(d), _p(v), d.shape[1], d.shape[0], scale, int(pfm))
        if rc:
            self._raise(rc)

    def save_gray_pgm(self, path, g):
        g = np.ascontiguousarray(g, np.float32)
        rc = self.f("save_gray_pgm", [C.c_char_p, _P, _I, _I])(path.encode(), _p(g), g.shape[1], g.shape[0])
        if rc:
            self._raise(rc)

    def save_ppm(self, path, rgb):
        rgb = np.ascontiguousarray(rgb, np.uint8)
        rc = self.f("save_ppm", [C.c_char_p, _P, _I, _I])(path.encode(), _p(rgb), rgb.shape[1], rgb.shape[0])
        if rc:
            self._raise(rc)

    def save_config(self, path, n, S, seed, d_max, radius, threads, spread, lc, le, tol, gt_scale, generator):
        iv = np.array([n, S, seed, d_max, radius, threads], np.int64)
        dv = np.array([spread, lc, le, tol, gt_scale], np.float64)
        rc = self.f("save_config", [C.c_char_p, _P, _P, C.c_char_p])(path.encode(), _p(iv), _p(dv),
                                                                       generator.encode())
        if rc:
            self._raise(rc)

    def load_config(self, path):
        iv = np.zeros(6, np.int64)
        dv = np.zeros(5, np.float64)
        gen = C.create_string_buffer(256)
        rc = self.f("load_config", [C.c_char_p, _P, _P, C.c_char_p, _I])(path.encode(), _p(iv), _p(dv), gen, 256)
        if rc:
            self._raise(rc)
        keys = ["n", "window", "seed", "d_max", "vote_radius", "threads"]
        out = {k: int(v) for k, v in zip(keys, iv)}
        out.update({k: float(v) for k, v in zip(["spread", "lambda_c", "lambda_e", "lr_tolerance", "gt_scale"], dv)})
        out["generator"] = gen.value.decode()
        return out

    def save_pattern(self, path, pairs, n, window, spread, seed):
        pairs = np.ascontiguousarray(pairs, np.int16)
        rc = self.f("save_pattern", [C.c_char_p, _P, _I, _I, _D, C.c_uint64])(
            path.encode(), _p(pairs), n, window, spread, seed)
        if rc:
            self._raise(rc)

    def load_pattern(self, path, cap=16384):
        n, w, sp, sd = C.c_int(), C.c_int(), C.c_double(), C.c_uint64()
        pairs = np.zeros((cap, 4), np.int16)
        rc = self.f("load_pattern", [C.c_char_p, _P, _P, _P, _P, _P, _I])(
            path.encode(), C.byref(n), C.byref(w), C.byref(sp), C.byref(sd), _p(pairs), cap)
        if rc:
            self._raise(rc)
        return n.value, w.value, sp.value, sd.value, pairs[: n.value].copy()

    def bad_pixel_rate(self, d, v, gd, gv, region, threshold):
        H, W = d.shape
        rate, cnt, bad = C.c_double(), C.c_long(), C.c_long()
        args = [np.ascontiguousarray(x, t) for x, t in ((d, np.float32), (v, np.uint8), (gd, np.float32),
                                                         (gv, np.uint8))]
        reg = None if region is None else np.ascontiguousarray(region, np.float32)
        rc = self.f("bad_pixel_rate", [_P, _P, _P, _P, _P, _I, _I, _D, _P, _P, _P])(
            *[_p(a) for a in args], _p(reg), W, H, threshold, C.byref(rate), C.byref(cnt), C.byref(bad))
        if rc:
            self._raise(rc)
        return rate.value, cnt.value, bad.value

    def linear_fit_r2(self, xs, ys):
        xs = np.ascontiguousarray(xs, np.float64)
        ys = np.ascontiguousarray(ys, np.float64)
        out = C.c_double()
        rc = self.f("linear_fit_r2", [_P, _P, _I, _P])(_p(xs), _p(ys), len(xs), C.byref(out))
        if rc:
            self._raise(rc)
        return out.value

    def write_sweep_csv(self, path, n, err, secs):
        n = np.ascontiguousarray(n, np.int32)
        err = np.ascontiguousarray(err, np.float64)
        secs = np.ascontiguousarray(secs, np.float64)
        rc = self.f("write_sweep_csv", [C.c_char_p, _P, _P, _P, _I])(path.encode(), _p(n), _p(err), _p(secs), len(n))
        if rc:
            self._raise(rc)

    def radiometric(self, path, rate9):
        r = np.ascontiguousarray(rate9, np.float64).reshape(9)
        dg, od = C.c_double(), C.c_double()
        rc = self.f("write_radiometric_csv", [C.c_char_p, _P, _P, _P])(
            path.encode() if path else None, _p(r), C.byref(dg), C.byref(od))
        if rc:
            self._raise(rc)
        return dg.value, od.value


class RefIOError(Exception):
    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.msg = msg
