"""Data formats and evaluation either side of the matching path (SURVEY.md
8(f) rows 2-4) against the reference's own image_io.hpp / eval.hpp / JSON
sidecar code compiled in place (oracle/_ref/libbsm_ref_io.so): same pixels,
same error kinds and messages, byte-identical files.  Host only."""
import os
import struct
import subprocess
import sys
import zlib

import numpy as np
import pytest

import paper_1402_2020_b200 as bsm
from paper_1402_2020_b200 import evaluation as ev
from paper_1402_2020_b200 import io as bio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rio():
    from oracle import RefIO
    try:
        return RefIO()
    except FileNotFoundError as e:
        pytest.skip(str(e))


def _kind(exc):
    return {bio.IoError: "IoError", bio.FormatError: "FormatError", bsm.InvalidArgument: "InvalidArgument",
            bsm.DimensionMismatch: "DimensionMismatch", ev.EmptyRegion: "EmptyRegion"}.get(type(exc), "Error")


def _same_outcome(tmp_path, name, payload, ours, theirs):
    """Both loaders succeed with equal results, or both fail with the same kind and message."""
    p = str(tmp_path / name)
    with open(p, "wb") as f:
        f.write(payload)
    from oracle import RefIOError
    try:
        want = theirs(p)
    except RefIOError as e:
        with pytest.raises(bsm.BsmError) as got:
            ours(p)
        assert _kind(got.value) == e.kind, (name, str(got.value), e.msg)
        assert str(got.value) == e.msg, (name, str(got.value), e.msg)
        return None
    got = ours(p)
    return got, want


# ---------------------------------------------------------------------------
# load_image (image_io.hpp:240-263)
PNM_CASES = [
    ("a.pgm", b"P2\n2 2\n255\n0 64\n128 255\n"),
    ("b.ppm", b"P6\n1 1\n255\n\x0a\x14\x1e"),
    ("c.ppm", b"P3 # comment\n# another\n1 2\n255\n1 2 3\n250 251 252\n"),
    ("d16.pgm", b"P5\n2 1\n65535\n" + struct.pack(">HH", 0, 65535)),
    ("d12.pgm", b"P2\n3 1\n4095\n0 2048 4095\n"),
    ("e16.ppm", b"P6\n1 1\n1023\n" + struct.pack(">HHH", 1, 512, 1023)),
    ("bad_magic.pgm", b"P7\n1 1\n255\n\x00"),
    ("bad_dims.pgm", b"P5\n0 1\n255\n"),
    ("bad_maxval.pgm", b"P5\n1 1\n70000\n\x00"),
    ("range.pgm", b"P2\n1 1\n10\n11\n"),
    ("trunc.pgm", b"P5\n4 4\n255\n\x00\x01"),
    ("nosep.pgm", b"P5\n1 1\n255"),
    ("badtok.pgm", b"P5\nx 1\n255\n\x00"),
    ("badtok2.pgm", b"P5\n1x 1\n255\n\x00"),
    ("missing.pgm", b"P5\n1"),
    ("empty.pgm", b""),
]


@pytest.mark.parametrize("name,payload", PNM_CASES)
def test_load_image_matches_reference(tmp_path, rio, name, payload):
    r = _same_outcome(tmp_path, name, payload, bio.load_image, rio.load_image)
    if r is not None:
        got, want = r
        assert np.array_equal(got, want)


def test_load_image_missing_file(tmp_path, rio):
    with pytest.raises(bio.IoError, match="cannot open"):
        bio.load_image(str(tmp_path / "nope.pgm"))


def test_load_image_random_binary_pnm(tmp_path, rio):
    rng = np.random.default_rng(3)
    for maxval, ch, magic in ((255, 1, b"P5"), (255, 3, b"P6"), (4000, 1, b"P5"), (65535, 3, b"P6")):
        h, w = 5, 7
        s = rng.integers(0, maxval + 1, size=(h, w, ch))
        body = s.astype(">u2" if maxval > 255 else np.uint8).tobytes()
        r = _same_outcome(tmp_path, "r.pnm", magic + b"\n%d %d\n%d\n" % (w, h, maxval) + body, bio.load_image,
                          rio.load_image)
        assert np.array_equal(*r)


# ---------------------------------------------------------------------------
# load_gt_disparity (image_io.hpp:268-314)
def _pfm(vals, big=False, magic=b"Pf"):
    h, w = vals.shape[:2]
    body = np.ascontiguousarray(vals[::-1]).astype(">f4" if big else "<f4").tobytes()
    return magic + b"\n%d %d\n%s\n" % (w, h, b"1.0" if big else b"-1.0") + body


@pytest.mark.parametrize("scale", [1.0, 4.0, 16.0, 3.0])
def test_load_gt_matches_reference(tmp_path, rio, scale):
    rng = np.random.default_rng(int(scale))
    v16 = rng.integers(0, 4000, size=(6, 9)).astype(np.uint16)
    v16[0, :3] = 0
    pf = rng.normal(30, 10, size=(4, 5)).astype(np.float32)
    pf[1, 1], pf[2, 3] = np.inf, np.nan
    cases = [
        ("g.pgm", b"P5\n9 6\n65535\n" + v16.astype(">u2").tobytes()),
        ("g8.pgm", b"P5\n9 6\n255\n" + (v16 % 256).astype(np.uint8).tobytes()),
        ("le.pfm", _pfm(pf)), ("be.pfm", _pfm(pf, big=True)),
        ("col.pfm", _pfm(np.repeat(pf[:, :, None], 3, 2).reshape(4, 15), magic=b"PF")),
        ("col.ppm", b"P6\n1 1\n255\n\x01\x02\x03"),
        ("badscale.pfm", b"Pf\n1 1\nabc\n\x00\x00\x00\x00"), ("zeroscale.pfm", b"Pf\n1 1\n0\n\x00\x00\x00\x00"),
        ("trunc.pfm", b"Pf\n2 2\n-1.0\n\x00\x00"),
    ]
    for name, payload in cases:
        r = _same_outcome(tmp_path, name, payload, lambda p: bio.load_gt_disparity(p, scale),
                          lambda p: rio.load_gt(p, scale))
        if r is not None:
            got, (d, v) = r
            assert np.array_equal(got.disparity.view(np.uint32), d.view(np.uint32)), name
            assert np.array_equal(got.valid, v), name


def test_load_gt_rejects_bad_scale(tmp_path):
    p = tmp_path / "g.pgm"
    p.write_bytes(b"P5\n1 1\n255\n\x05")
    with pytest.raises(bsm.InvalidArgument, match="disparity scale must be > 0"):
        bio.load_gt_disparity(str(p), 0.0)


# ---------------------------------------------------------------------------
# writers: byte-identical files
def _map(rng, h=7, w=11):
    d = (rng.random((h, w)) * 80).astype(np.float32)
    d[0, :4] = [0.5 / 16, 1.5 / 16, 2.5 / 16, 1e6]  # rounding halves, clamp above 65535
    d[1, 0] = -3.0                                # clamp below 0
    v = (rng.random((h, w)) < 0.8).astype(np.uint8)
    return bsm.DisparityMap(d, v)


@pytest.mark.parametrize("scale", [16.0, 4.0, 1.5, 1.0])
def test_save_disparity_byte_identical(tmp_path, rio, scale):
    m = _map(np.random.default_rng(7))
    a, b = str(tmp_path / "a.pgm"), str(tmp_path / "b.pgm")
    bio.save_disparity(m, a, scale)
    rio.save_disparity(b, m.disparity, m.valid, scale)
    assert open(a, "rb").read() == open(b, "rb").read()


def test_save_pfm_and_roundtrip(tmp_path, rio):
    m = _map(np.random.default_rng(8))
    a, b = str(tmp_path / "a.pfm"), str(tmp_path / "b.pfm")
    bio.save_disparity_pfm(m, a)
    rio.save_disparity(b, m.disparity, m.valid, 1.0, pfm=True)
    assert open(a, "rb").read() == open(b, "rb").read()
    back = bio.load_gt_disparity(a, 1.0)
    assert np.array_equal(back.valid, m.valid)
    assert np.array_equal(back.disparity[m.valid == 1], m.disparity[m.valid == 1])


def test_save_gray_pgm_and_ppm_byte_identical(tmp_path, rio):
    rng = np.random.default_rng(9)
    g = (rng.random((5, 8)) * 300 - 20).astype(np.float32)
    g[0, :4] = [0.49999997, 0.5, 254.5, 1.5]
    bio.save_gray_pgm(g, str(tmp_path / "a.pgm"))
    rio.save_gray_pgm(str(tmp_path / "b.pgm"), g)
    assert (tmp_path / "a.pgm").read_bytes() == (tmp_path / "b.pgm").read_bytes()
    rgb = rng.integers(0, 256, size=(4, 6, 3), dtype=np.uint8)
    bio.save_ppm(rgb, str(tmp_path / "a.ppm"))
    rio.save_ppm(str(tmp_path / "b.ppm"), rgb)
    assert (tmp_path / "a.ppm").read_bytes() == (tmp_path / "b.ppm").read_bytes()
    assert np.array_equal(bio.load_image(str(tmp_path / "a.ppm")), rgb)


# ---------------------------------------------------------------------------
# JSON sidecars
def test_config_sidecar_byte_identical(tmp_path, rio):
    cfg = bsm.BsmConfig(n=512, window=12, spread=3.25, seed=9, d_max=64, lambda_c=5.0, lambda_e=7.5,
                        lr_tolerance=0.0, vote_radius=6, gt_scale=4.0, threads=3)
    bio.save_config(cfg, str(tmp_path / "a.json"))
    rio.save_config(str(tmp_path / "b.json"), 512, 12, 9, 64, 6, 3, 3.25, 5.0, 7.5, 0.0, 4.0, cfg.generator)
    assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
    assert bio.load_config(str(tmp_path / "b.json")) == cfg
    got = rio.load_config(str(tmp_path / "a.json"))
    assert got["n"] == 512 and got["window"] == 12 and got["spread"] == 3.25 and got["gt_scale"] == 4.0


def test_config_partial_and_bad(tmp_path, rio):
    (tmp_path / "p.json").write_text('{"d_max": 30, "S": 16}')
    c = bio.load_config(str(tmp_path / "p.json"))
    r = rio.load_config(str(tmp_path / "p.json"))
    assert c.d_max == r["d_max"] == 30 and c.window == r["window"] == 16 and c.n == r["n"] == 4096
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(bio.FormatError, match="bad config file"):
        bio.load_config(str(tmp_path / "bad.json"))
    from oracle import RefIOError
    with pytest.raises(RefIOError, match="bad config file"):
        rio.load_config(str(tmp_path / "bad.json"))


def test_pattern_sidecar_byte_identical(tmp_path, rio):
    p = bsm.generate_pattern(70, 6, 2.0, 37)
    bio.save_pattern(p, str(tmp_path / "a.json"))
    rio.save_pattern(str(tmp_path / "b.json"), p.pairs, p.n, p.window, p.spread, p.seed)
    assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
    q = bio.load_pattern(str(tmp_path / "b.json"))
    assert q.n == 70 and q.window == 6 and np.array_equal(q.pairs, p.pairs)
    n, w, sp, sd, pairs = rio.load_pattern(str(tmp_path / "a.json"))
    assert (n, w, sp, sd) == (70, 6, 2.0, 37) and np.array_equal(pairs, p.pairs)


def test_pattern_sidecar_errors(tmp_path, rio):
    from oracle import RefIOError
    import json
    p = bsm.generate_pattern(8, 6, 2.0, 1)
    base = {"generator": bsm.GENERATOR_NAME, "n": 8, "S": 6, "spread": 2.0, "seed": 1,
            "pairs": p.pairs.tolist()}
    cases = {"gen": {**base, "generator": "other"}, "count": {**base, "n": 9},
             "outside": {**base, "pairs": [[9, 0, 0, 0]] + base["pairs"][1:]}}
    for name, obj in cases.items():
        f = tmp_path / f"{name}.json"
        f.write_text(json.dumps(obj))
        with pytest.raises(RefIOError) as want:
            rio.load_pattern(str(f))
        with pytest.raises(bio.FormatError) as got:
            bio.load_pattern(str(f))
        assert str(got.value) == want.value.msg


# ---------------------------------------------------------------------------
# PNG subset (libpng simplified API semantics for 8-bit gray / RGB / palette)
def _png(img, ctype, filters=(0,), palette=None):
    h, w = img.shape[:2]
    bpp = {0: 1, 2: 3, 3: 1}[ctype]
    rows = np.asarray(img, np.uint8).reshape(h, w * bpp).astype(np.int32)
    raw = bytearray()
    prev = np.zeros(w * bpp, np.int32)
    for y in range(h):
        ft = filters[y % len(filters)]
        cur = rows[y]
        left = np.concatenate([np.zeros(bpp, np.int32), cur[:-bpp]])
        upl = np.concatenate([np.zeros(bpp, np.int32), prev[:-bpp]])
        if ft == 0:
            out = cur
        elif ft == 1:
            out = cur - left
        elif ft == 2:
            out = cur - prev
        elif ft == 3:
            out = cur - ((left + prev) >> 1)
        else:
            pa, pb, pc = np.abs(prev - upl), np.abs(left - upl), np.abs(left + prev - 2 * upl)
            pred = np.where((pa <= pb) & (pa <= pc), left, np.where(pb <= pc, prev, upl))
            out = cur - pred
        raw += bytes([ft]) + (out & 255).astype(np.uint8).tobytes()
        prev = cur

    def chunk(t, b):
        return struct.pack(">I", len(b)) + t + b + struct.pack(">I", zlib.crc32(t + b) & 0xFFFFFFFF)

    s = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, ctype, 0, 0, 0))
    if palette is not None:
        s += chunk(b"PLTE", np.asarray(palette, np.uint8).tobytes())
    return s + chunk(b"IDAT", zlib.compress(bytes(raw))) + chunk(b"IEND", b"")


def test_png_decoding(tmp_path):
    rng = np.random.default_rng(11)
    # the reference's own fixtures (test_image_io.cpp): 2x2 RGB and 2x1 gray
    rgb = np.array([[[255, 0, 0], [0, 255, 0]], [[0, 0, 255], [10, 20, 30]]], np.uint8)
    (tmp_path / "a.png").write_bytes(_png(rgb, 2))
    assert np.array_equal(bio.load_image(str(tmp_path / "a.png")), rgb)
    g = np.array([[7, 200]], np.uint8)
    (tmp_path / "g.png").write_bytes(_png(g, 0))
    assert np.array_equal(bio.load_image(str(tmp_path / "g.png")), np.repeat(g[:, :, None], 3, 2))
    d = bio.load_gt_disparity(str(tmp_path / "g.png"), 1.0)
    assert d.disparity.tolist() == [[7.0, 200.0]] and d.valid.tolist() == [[1, 1]]
    for filters in ((0,), (1,), (2,), (3,), (4,), (0, 1, 2, 3, 4)):
        img = rng.integers(0, 256, size=(9, 13, 3), dtype=np.uint8)
        (tmp_path / "f.png").write_bytes(_png(img, 2, filters))
        assert np.array_equal(bio.load_image(str(tmp_path / "f.png")), img), filters
    pal = rng.integers(0, 256, size=(16, 3), dtype=np.uint8)
    idx = rng.integers(0, 16, size=(5, 6), dtype=np.uint8)
    (tmp_path / "p.png").write_bytes(_png(idx, 3, (4,), pal))
    assert np.array_equal(bio.load_image(str(tmp_path / "p.png")), pal[idx])
    (tmp_path / "bad.png").write_bytes(_png(rgb, 2)[:-20])
    with pytest.raises(bio.FormatError, match="bad PNG"):
        bio.load_image(str(tmp_path / "bad.png"))
    with pytest.raises(bio.FormatError, match="colour-to-gray"):
        bio.load_gt_disparity(str(tmp_path / "a.png"), 1.0)


# ---------------------------------------------------------------------------
# evaluation (eval.hpp)
def test_bad_pixel_rate_matches_reference(rio):
    rng = np.random.default_rng(5)
    for it in range(6):
        h, w = 13, 17
        d = (rng.random((h, w)) * 20).astype(np.float32)
        v = (rng.random((h, w)) < 0.8).astype(np.uint8)
        gd = (d + rng.normal(0, 1.2, size=(h, w))).astype(np.float32)
        gv = (rng.random((h, w)) < 0.9).astype(np.uint8)
        reg = None if it % 2 else (rng.random((h, w)) * 255).astype(np.float32)
        thr = [0.5, 1.0, 2.0][it % 3]
        want = rio.bad_pixel_rate(d, v, gd, gv, reg, thr)
        got = ev.bad_pixel_rate(bsm.DisparityMap(d, v), bsm.DisparityMap(gd, gv), reg, thr)
        assert (got.bad_pixel_rate, got.counted, got.bad) == want


def test_bad_pixel_rate_kats():
    # test_eval.cpp: perfect 0, one bad in a hundred, all invalid 100, exclusive threshold, errors
    gt = bsm.DisparityMap(np.full((10, 10), 5.0, np.float32), np.ones((10, 10), np.uint8))
    assert ev.bad_pixel_rate(gt, gt).bad_pixel_rate == 0.0
    r = bsm.DisparityMap(gt.disparity.copy(), gt.valid.copy())
    r.disparity[3, 4] = 9.0
    assert ev.bad_pixel_rate(r, gt).bad_pixel_rate == 1.0
    r2 = bsm.DisparityMap(gt.disparity.copy(), np.zeros((10, 10), np.uint8))
    assert ev.bad_pixel_rate(r2, gt).bad_pixel_rate == 100.0
    r3 = bsm.DisparityMap(gt.disparity + np.float32(1.0), gt.valid.copy())
    assert ev.bad_pixel_rate(r3, gt, None, 1.0).bad_pixel_rate == 0.0
    with pytest.raises(ev.EmptyRegion):
        ev.bad_pixel_rate(gt, gt, np.zeros((10, 10), np.float32))
    with pytest.raises(bsm.DimensionMismatch):
        ev.bad_pixel_rate(gt, bsm.DisparityMap(np.zeros((9, 10), np.float32), np.ones((9, 10), np.uint8)))
    with pytest.raises(bsm.InvalidArgument, match="threshold must be > 0"):
        ev.bad_pixel_rate(gt, gt, None, 0.0)


def test_linear_fit_and_csv_match_reference(tmp_path, rio):
    rng = np.random.default_rng(6)
    for xs, ys in (([1, 2, 3, 4], [2, 4, 6, 8]), (list(range(8)), list(rng.random(8))),
                   ([512, 1024, 2048, 4096], [0.31, 0.52, 1.01, 2.05]), ([1, 2], [3, 3])):
        assert ev.linear_fit_r2(xs, ys) == rio.linear_fit_r2(xs, ys)
    with pytest.raises(bsm.InvalidArgument):
        ev.linear_fit_r2([1, 1], [2, 3])
    pts = [ev.SweepPoint(512, 12.3456789, 0.123456), ev.SweepPoint(4096, 7.0, 1.99995)]
    ev.write_sweep_csv(str(tmp_path / "a.csv"), pts)
    rio.write_sweep_csv(str(tmp_path / "b.csv"), [512, 4096], [12.3456789, 7.0], [0.123456, 1.99995])
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()
    m = ev.RadiometricMatrix([[1.0, 2.5, 3.0], [4.0, 5.125, 6.0], [7.0, 8.0, 9.75]])
    ev.write_radiometric_csv(str(tmp_path / "r1.csv"), m)
    dg, od = rio.radiometric(str(tmp_path / "r2.csv"), np.array(m.rate))
    assert (tmp_path / "r1.csv").read_bytes() == (tmp_path / "r2.csv").read_bytes()
    assert (m.diagonal_mean(), m.off_diagonal_mean()) == (dg, od)


# ---------------------------------------------------------------------------
# CLI: host-side behaviour (no device needed)
def _cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_1402_2020_b200", *args], capture_output=True, text=True,
                          cwd=cwd or ROOT, env={**os.environ, "PYTHONPATH": ROOT})


def test_cli_errors(tmp_path):
    assert _cli().returncode != 0                                    # no subcommand
    r = _cli("match", str(tmp_path / "nope.pgm"), str(tmp_path / "nope.pgm"), str(tmp_path / "o.pgm"),
             "--d_max", "4")
    assert r.returncode == 1 and "error: cannot open" in r.stderr
    img = tmp_path / "i.pgm"
    img.write_bytes(b"P5\n4 3\n255\n" + bytes(range(12)))
    r = _cli("match", str(img), str(img), str(tmp_path / "o.pgm"))
    assert r.returncode == 1 and "d_max" in r.stderr                  # test_cli.cpp:177-183
    other = tmp_path / "j.pgm"
    other.write_bytes(b"P5\n5 3\n255\n" + bytes(range(15)))
    r = _cli("match", str(img), str(other), str(tmp_path / "o.pgm"), "--d_max", "2")
    assert r.returncode == 1 and "dimensions differ" in r.stderr


def test_cli_eval(tmp_path):
    gt = bsm.DisparityMap(np.full((4, 5), 3.0, np.float32), np.ones((4, 5), np.uint8))
    bio.save_disparity(gt, str(tmp_path / "gt.pgm"), 16.0)
    r = _cli("eval", str(tmp_path / "gt.pgm"), str(tmp_path / "gt.pgm"))
    assert r.returncode == 0 and r.stdout == "all        0.00  (0 of 20 pixels beyond 1.00)\n"
    bad = bsm.DisparityMap(gt.disparity.copy(), gt.valid.copy())
    bad.disparity[0, 0] = 9.0
    bio.save_disparity(bad, str(tmp_path / "r.pgm"), 16.0)
    mask = np.full((4, 5, 3), 255, np.uint8)
    bio.save_ppm(mask, str(tmp_path / "m.ppm"))
    r = _cli("eval", str(tmp_path / "r.pgm"), str(tmp_path / "gt.pgm"), "--nonocc", str(tmp_path / "m.ppm"),
             "--disc", str(tmp_path / "m.ppm"))
    assert r.stdout.splitlines() == ["nonocc     5.00  (1 of 20 pixels beyond 1.00)",
                                     "disc       5.00  (1 of 20 pixels beyond 1.00)"]
