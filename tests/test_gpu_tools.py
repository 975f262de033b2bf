"""The callers either side of the path on the GPU:
the CLI's output files, the length sweep and the radiometric protocol, against
the reference pipeline (oracle/_ref) and its own writers / scoring
(oracle/_ref/libbsm_ref_io.so)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1402_2020_b200 as bsm
from paper_1402_2020_b200 import evaluation as ev
from paper_1402_2020_b200 import io as bio
from paper_1402_2020_b200.synth import colour_pair, synth_pair

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rio():
    from oracle import RefIO
    return RefIO()


def _cli(*args, impl="python"):
    if impl == "cpp":  # the C++ tool (paper_1402_2020_b200/csrc/bsm_cli.cpp)
        return subprocess.run([os.path.join(ROOT, "paper_1402_2020_b200", "bsm"), *args], capture_output=True,
                              text=True, cwd=ROOT)
    return subprocess.run([sys.executable, "-m", "paper_1402_2020_b200", *args], capture_output=True, text=True,
                          cwd=ROOT, env={**os.environ, "PYTHONPATH": ROOT})


def _crop(h=40, w=160, seed=1):
    left, right = synth_pair(0, seed, 450, 375)
    return left[100:100 + h, 50:50 + w].copy(), right[100:100 + h, 50:50 + w].copy()


@pytest.mark.parametrize("impl", ["python", "cpp"])
@pytest.mark.parametrize("colour", [False, True])
def test_cli_match_files_byte_identical(tmp_path, ref, rio, default_pairs, colour, impl):
    if colour:
        L, R = colour_pair(36, 150, seed=3)
        bio.save_ppm(L, str(tmp_path / "l.ppm"))
        bio.save_ppm(R, str(tmp_path / "r.ppm"))
        lp, rp = str(tmp_path / "l.ppm"), str(tmp_path / "r.ppm")
    else:
        L, R = _crop()
        for nm, im in (("l.pgm", L), ("r.pgm", R)):
            (tmp_path / nm).write_bytes(b"P5\n%d %d\n255\n" % (im.shape[1], im.shape[0]) + im.tobytes())
        lp, rp = str(tmp_path / "l.pgm"), str(tmp_path / "r.pgm")
    out = str(tmp_path / "d.pgm")
    r = _cli("match", lp, rp, out, "--d_max", "60", "--stages", "--gt_scale", "4",
             "--emit-pattern", str(tmp_path / "pat.json"), impl=impl)
    assert r.returncode == 0, r.stderr
    want = ref.pipeline(L, R, default_pairs, 26, 60, threads=16, want_unmasked=True, channels=3 if colour else 1)
    ones = np.ones_like(want["refined_v"])
    for path, (d, v) in ((out, (want["refined_d"], want["refined_v"])),
                         (str(tmp_path / "d.refined.pgm"), (want["refined_d"], want["refined_v"])),
                         (str(tmp_path / "d.masked.pgm"), (want["left_d"], ones)),
                         (str(tmp_path / "d.unmasked.pgm"), (want["unmasked_d"], ones))):
        rio.save_disparity(str(tmp_path / "want.pgm"), d, v, 4.0)
        assert open(path, "rb").read() == (tmp_path / "want.pgm").read_bytes(), path
    rio.save_config(str(tmp_path / "want.json"), 4096, 26, 42, 60, 20, 1, 4.0, 9.0, 16.0, 1.0, 4.0,
                    bsm.GENERATOR_NAME)
    assert (tmp_path / "d.pgm.config.json").read_bytes() == (tmp_path / "want.json").read_bytes()
    rio.save_pattern(str(tmp_path / "want_pat.json"), default_pairs, 4096, 26, 4.0, 42)
    assert (tmp_path / "pat.json").read_bytes() == (tmp_path / "want_pat.json").read_bytes()
    # float output and a saved pattern fed back in
    r = _cli("match", lp, rp, str(tmp_path / "d.pfm"), "--d_max", "60", "--pattern", str(tmp_path / "pat.json"),
             impl=impl)
    assert r.returncode == 0, r.stderr
    rio.save_disparity(str(tmp_path / "want.pfm"), want["refined_d"], want["refined_v"], 1.0, pfm=True)
    assert (tmp_path / "d.pfm").read_bytes() == (tmp_path / "want.pfm").read_bytes()


@pytest.mark.parametrize("impl", ["python", "cpp"])
def test_cli_bench_line(tmp_path, impl):
    L, R = _crop(24, 96)
    for nm, im in (("l.pgm", L), ("r.pgm", R)):
        (tmp_path / nm).write_bytes(b"P5\n%d %d\n255\n" % (im.shape[1], im.shape[0]) + im.tobytes())
    r = _cli("bench", str(tmp_path / "l.pgm"), str(tmp_path / "r.pgm"), "--d_max", "32", "--runs", "2", impl=impl)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("median of 2 runs: ") and "(96x24, d_max=32, n=4096, threads=1)" in r.stdout


def _scene(seed, h=48, w=180):
    left, right, gt = synth_pair(0, seed, 450, 375, with_gt=True)
    sl = (slice(120, 120 + h), slice(60, 60 + w))
    g = gt[sl].astype(np.float32)
    return left[sl].copy(), right[sl].copy(), bsm.DisparityMap(g, (g > 0).astype(np.uint8))


def test_length_sweep_matches_reference(ref, rio):
    scenes = [_scene(11), _scene(12)]
    n_values = [64, 256, 1000]
    cfg = bsm.BsmConfig(d_max=60)
    pts = ev.length_sweep([ev.SweepScene(L, R, g, None, 60) for L, R, g in scenes], n_values, cfg)
    for p in pts:
        pairs = ref.generate_pattern(p.n, 26, 4.0, 42)
        rates = []
        for L, R, g in scenes:
            w = ref.pipeline(L, R, pairs, 26, 60, threads=16)
            rates.append(rio.bad_pixel_rate(w["refined_d"], w["refined_v"], g.disparity, g.valid, None, 1.0)[0])
        assert p.avg_error == sum(rates) / len(rates)
        assert p.wall_time > 0
    with pytest.raises(bsm.InvalidArgument, match="below 64"):
        ev.length_sweep([ev.SweepScene(*scenes[0], None, 60)], [32], cfg)


def test_radiometric_protocol_matches_reference(ref, rio, default_pairs):
    L, R, g = _scene(13)
    curves = [lambda x: x, lambda x: np.clip(x.astype(np.int32) * 3 // 4 + 40, 0, 255).astype(np.uint8),
              lambda x: (255.0 * (x / 255.0) ** 0.7).round().astype(np.uint8)]
    lefts = [c(L) for c in curves]
    rights = [c(R) for c in curves]
    region = np.full(L.shape, 255.0, np.float32)
    region[:, :20] = 0.0
    cfg = bsm.BsmConfig(d_max=60)
    pat = bsm.SamplingPattern(4096, 26, 4.0, 42, default_pairs)
    m = ev.radiometric_protocol(lefts, rights, g, region, pat, cfg)
    for i in range(3):
        for j in range(3):
            w = ref.pipeline(lefts[i], rights[j], default_pairs, 26, 60, threads=16)
            want = rio.bad_pixel_rate(w["refined_d"], w["refined_v"], g.disparity, g.valid, region, 1.0)[0]
            assert m.rate[i][j] == want
    dg, od = rio.radiometric(None, np.array(m.rate))
    assert (m.diagonal_mean(), m.off_diagonal_mean()) == (dg, od)


def _write_scene(root, L, R, gt, scale):
    os.makedirs(root, exist_ok=True)
    bio.save_ppm(np.repeat(L[:, :, None], 3, 2) if L.ndim == 2 else L, os.path.join(root, "im2.ppm"))
    bio.save_ppm(np.repeat(R[:, :, None], 3, 2) if R.ndim == 2 else R, os.path.join(root, "im6.ppm"))
    bio.save_disparity(gt, os.path.join(root, "disp2.pgm"), scale)
    mask = np.full(L.shape[:2] + (3,), 255, np.uint8)
    mask[:, :12] = 0
    bio.save_ppm(mask, os.path.join(root, "nonocc.ppm"))


@pytest.mark.parametrize("impl", ["python", "cpp"])
def test_cli_sweep_and_radiometric(tmp_path, impl):
    # a scene directory in the stock layout and a 3-condition radiometric set
    L, R, g = _scene(21)
    scene = str(tmp_path / "scene")
    _write_scene(scene, L, R, g, 4.0)
    os.rename(os.path.join(scene, "nonocc.ppm"), os.path.join(scene, "nonocc.pgm.tmp"))
    m = bio.load_image(os.path.join(scene, "nonocc.pgm.tmp"))
    (tmp_path / "scene" / "nonocc.pgm").write_bytes(b"P5\n%d %d\n255\n" % (m.shape[1], m.shape[0]) +
                                                    m[:, :, 0].tobytes())
    os.remove(os.path.join(scene, "nonocc.pgm.tmp"))
    out = str(tmp_path / "sweep.csv")
    r = _cli("sweep", scene, "--d_max", "60", "--gt_scale", "4", "--n_values", "256,1024", "--out", out, impl=impl)
    assert r.returncode == 0, r.stderr
    lines = open(out).read().splitlines()
    assert lines[0] == "n,avg_error,wall_time" and [ln.split(",")[0] for ln in lines[1:]] == ["256", "1024"]
    # the sweep's error column equals the evaluation layer on the same scene
    ds = bio.load_stereo_dataset(scene, "scene", 60, 4.0)
    pts = ev.length_sweep([ev.SweepScene(ds.left, ds.right, ds.gt, ds.mask_nonocc, 60)], [256, 1024],
                          bsm.BsmConfig(d_max=60, gt_scale=4.0))
    assert [ln.split(",")[1] for ln in lines[1:]] == ["%.6f" % p.avg_error for p in pts]
    assert "linear fit of time vs n" in r.stdout and os.path.exists(out + ".config.json")

    rset = str(tmp_path / "rad")
    os.makedirs(rset)
    curves = [lambda x: x, lambda x: np.clip(x.astype(np.int32) * 3 // 4 + 40, 0, 255).astype(np.uint8),
              lambda x: (255.0 * (x / 255.0) ** 0.7).round().astype(np.uint8)]
    for c, f in enumerate(curves):
        for side, img in (("left", L), ("right", R)):
            v = f(img)
            (tmp_path / "rad" / f"{side}_c{c}.pgm").write_bytes(b"P5\n%d %d\n255\n" % (v.shape[1], v.shape[0]) +
                                                                v.tobytes())
    bio.save_disparity(g, os.path.join(rset, "gt.pgm"), 4.0)
    out = str(tmp_path / "rad.csv")
    r = _cli("radiometric", rset, "--d_max", "60", "--gt_scale", "4", "--out", out, impl=impl)
    assert r.returncode == 0, r.stderr
    rs = bio.load_radiometric_set(rset, 60, 4.0)
    m = ev.radiometric_protocol(rs.lefts, rs.rights, rs.gt, None, bsm.generate_pattern(), bsm.BsmConfig(d_max=60))
    want = ["left_condition,right_condition,bad_pixel_rate"] + \
        ["%d,%d,%.6f" % (i, j, m.rate[i][j]) for i in range(3) for j in range(3)]
    assert open(out).read().splitlines() == want
    assert ("diagonal mean %.2f, off-diagonal mean %.2f" % (m.diagonal_mean(), m.off_diagonal_mean())) in r.stdout
