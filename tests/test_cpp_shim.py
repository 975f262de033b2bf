"""The C++ drop-in API (include/bsm/*.hpp over libbsm_cuda.so), compiled and
run as a client program would use it."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_1402_2020_b200")
BIN = os.path.join(ROOT, "build", "shim_test")


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(LIBDIR, "libbsm_cuda.so")),
            *[os.path.getmtime(os.path.join(ROOT, "include", "bsm", f))
              for f in os.listdir(os.path.join(ROOT, "include", "bsm"))]):
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
                        "-L", LIBDIR, "-lbsm_cuda", "-lz", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return BIN


def test_shim_compiles_and_host_checks(ref):
    out = subprocess.run([build(), "host"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    # the default pattern equals the reference's (FNV-1a over the pairs)
    pairs = ref.generate_pattern(4096, 26, 4.0, 42)
    h = 1469598103934665603
    for v in pairs.reshape(-1):
        h = ((h ^ (int(v) & 0xFFFF)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    assert f"pattern_fnv {h}" in out.stdout


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_shim_no_cpu_fallback():
    out = subprocess.run([build(), "nodevice"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("colour", [False, True])
def test_shim_pipeline_matches_reference(tmp_path, ref, default_pairs, colour):
    from paper_1402_2020_b200.synth import workload_pair, colour_pair
    if colour:
        L, R = colour_pair(40, 160, seed=5)
    else:
        left, right = workload_pair("c1")
        L, R = left[140:180, 60:220].copy(), right[140:180, 60:220].copy()
    H, W = L.shape[:2]
    (tmp_path / "l.raw").write_bytes(L.tobytes())
    (tmp_path / "r.raw").write_bytes(R.tobytes())
    out = subprocess.run([build(), "gpu", str(tmp_path / "l.raw"), str(tmp_path / "r.raw"), str(W), str(H), "60",
                          str(tmp_path / "o.bin")], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    raw = np.fromfile(tmp_path / "o.bin", np.uint8)
    maps = []
    off = 0
    for _ in range(5):
        d = raw[off:off + 4 * W * H].view(np.float32).reshape(H, W)
        off += 4 * W * H
        v = raw[off:off + W * H].reshape(H, W)
        off += W * H
        maps.append((d, v))
    want = ref.pipeline(L, R, default_pairs, 26, 60, threads=8, want_unmasked=True, channels=3 if colour else 1)
    assert np.array_equal(maps[0][0], want["refined_d"]) and np.array_equal(maps[0][1], want["refined_v"])
    assert np.array_equal(maps[1][0], want["left_d"])
    assert np.array_equal(maps[2][0], want["right_d"])
    assert np.array_equal(maps[3][0], want["checked_d"]) and np.array_equal(maps[3][1], want["checked_v"])
    assert np.array_equal(maps[4][0], want["unmasked_d"])


# ---------------------------------------------------------------------------
# The C++ file/eval layer (include/bsm/image_io.hpp, eval.hpp, config.hpp,
# pattern.hpp) against the reference's own code (oracle/_ref/libbsm_ref_io.so),
# through the product's C ABI (include/bsm_io.h, paper_1402_2020_b200/libbsm_io.so),
# whose entry points mirror the reference driver's one for one.
IO_LIB = os.path.join(LIBDIR, "libbsm_io.so")


@pytest.fixture(scope="module")
def pair_io():
    from oracle import RefIO
    if not os.path.exists(IO_LIB):
        pytest.skip("libbsm_io.so not built")
    try:
        ref = RefIO()
    except FileNotFoundError as e:
        pytest.skip(str(e))
    return RefIO(IO_LIB, "bsmio_"), ref


def _outcome(fn, *args):
    from oracle import RefIOError
    try:
        return ("ok", fn(*args))
    except RefIOError as e:
        return ("err", e.kind, e.msg)


def _same(a, b):
    if a[0] != b[0]:
        return False
    if a[0] == "err":
        return a == b
    x, y = a[1], b[1]
    if isinstance(x, tuple):
        return all(np.array_equal(np.asarray(p).view(np.uint8), np.asarray(q).view(np.uint8)) for p, q in zip(x, y))
    return np.array_equal(x, y)


def test_cpp_io_readers_match_reference(tmp_path, pair_io):
    from test_io import PNM_CASES, _pfm
    shim, ref = pair_io
    cases = list(PNM_CASES)
    pf = np.random.default_rng(2).normal(30, 10, size=(4, 5)).astype(np.float32)
    pf[1, 1] = np.inf
    cases += [("le.pfm", _pfm(pf)), ("be.pfm", _pfm(pf, big=True)),
              ("g16.pgm", b"P5\n3 2\n65535\n" + np.arange(6, dtype=">u2").tobytes())]
    for name, payload in cases:
        p = tmp_path / name
        p.write_bytes(payload)
        assert _same(_outcome(shim.load_image, str(p)), _outcome(ref.load_image, str(p))), name
        for scale in (1.0, 4.0, 3.0):
            assert _same(_outcome(shim.load_gt, str(p), scale), _outcome(ref.load_gt, str(p), scale)), (name, scale)


def test_cpp_io_writers_and_sidecars_byte_identical(tmp_path, pair_io):
    shim, ref = pair_io
    rng = np.random.default_rng(4)
    d = (rng.random((6, 9)) * 80).astype(np.float32)
    d[0, :3] = [0.5 / 16, 2.5 / 16, 1e6]
    v = (rng.random((6, 9)) < 0.8).astype(np.uint8)
    for scale, pfm in ((16.0, False), (1.5, False), (1.0, True)):
        shim.save_disparity(str(tmp_path / "a"), d, v, scale, pfm)
        ref.save_disparity(str(tmp_path / "b"), d, v, scale, pfm)
        assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()
    g = (rng.random((5, 7)) * 300 - 20).astype(np.float32)
    shim.save_gray_pgm(str(tmp_path / "a"), g)
    ref.save_gray_pgm(str(tmp_path / "b"), g)
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()
    for args in ((4096, 26, 42, 60, 20, 1, 4.0, 9.0, 16.0, 1.0, 16.0, "mt19937_64-boxmuller-v1"),
                 (512, 12, 9, 64, 6, 3, 3.25, 5.0, 7.5, 0.0, 4.0, "mt19937_64-boxmuller-v1"),
                 (64, 8, 123456789012, 1, 1, 1, 1e-05, 0.1, 1e+20, 2.5, 0.125, "x")):
        shim.save_config(str(tmp_path / "a"), *args)
        ref.save_config(str(tmp_path / "b"), *args)
        assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes(), args
        assert shim.load_config(str(tmp_path / "b")) == ref.load_config(str(tmp_path / "a"))
    import paper_1402_2020_b200 as bsm
    p = bsm.generate_pattern(70, 6, 2.0, 37)
    shim.save_pattern(str(tmp_path / "a"), p.pairs, 70, 6, 2.0, 37)
    ref.save_pattern(str(tmp_path / "b"), p.pairs, 70, 6, 2.0, 37)
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()
    got, want = shim.load_pattern(str(tmp_path / "b")), ref.load_pattern(str(tmp_path / "a"))
    assert got[:4] == want[:4] and np.array_equal(got[4], want[4])


def test_cpp_eval_matches_reference(tmp_path, pair_io):
    shim, ref = pair_io
    rng = np.random.default_rng(8)
    for it in range(4):
        d = (rng.random((9, 12)) * 20).astype(np.float32)
        v = (rng.random((9, 12)) < 0.8).astype(np.uint8)
        gd = (d + rng.normal(0, 1.3, size=d.shape)).astype(np.float32)
        gv = (rng.random(d.shape) < 0.9).astype(np.uint8)
        reg = None if it % 2 else (rng.random(d.shape) * 255).astype(np.float32)
        assert shim.bad_pixel_rate(d, v, gd, gv, reg, 1.0) == ref.bad_pixel_rate(d, v, gd, gv, reg, 1.0)
    assert _same(_outcome(shim.bad_pixel_rate, d, v, gd, gv, np.zeros(d.shape, np.float32), 1.0),
                 _outcome(ref.bad_pixel_rate, d, v, gd, gv, np.zeros(d.shape, np.float32), 1.0))
    xs, ys = [512, 1024, 2048, 4096], [0.31, 0.52, 1.01, 2.05]
    assert shim.linear_fit_r2(xs, ys) == ref.linear_fit_r2(xs, ys)
    shim.write_sweep_csv(str(tmp_path / "a"), [512, 4096], [12.3456789, 7.0], [0.123456, 1.99995])
    ref.write_sweep_csv(str(tmp_path / "b"), [512, 4096], [12.3456789, 7.0], [0.123456, 1.99995])
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()
    rate = np.arange(9, dtype=np.float64) * 1.25
    assert shim.radiometric(str(tmp_path / "a"), rate) == ref.radiometric(str(tmp_path / "b"), rate)
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()


def test_cpp_cli_host_behaviour(tmp_path):
    exe = os.path.join(LIBDIR, "bsm")
    if not os.path.exists(exe):
        pytest.skip("paper_1402_2020_b200/bsm not built")
    run = lambda *a: subprocess.run([exe, *a], capture_output=True, text=True)
    assert run().returncode != 0
    img = tmp_path / "i.pgm"
    img.write_bytes(b"P5\n4 3\n255\n" + bytes(range(12)))
    r = run("match", str(img), str(img), str(tmp_path / "o.pgm"))
    assert r.returncode == 1 and "d_max" in r.stderr
    r = run("match", str(tmp_path / "nope.pgm"), str(img), str(tmp_path / "o.pgm"), "--d_max", "2")
    assert r.returncode == 1 and "error: cannot open" in r.stderr
    import paper_1402_2020_b200 as bsm
    from paper_1402_2020_b200 import io as bio
    gt = bsm.DisparityMap(np.full((4, 5), 3.0, np.float32), np.ones((4, 5), np.uint8))
    bio.save_disparity(gt, str(tmp_path / "gt.pgm"), 16.0)
    r = run("eval", str(tmp_path / "gt.pgm"), str(tmp_path / "gt.pgm"))
    assert r.returncode == 0 and r.stdout == "all        0.00  (0 of 20 pixels beyond 1.00)\n"


# ---------------------------------------------------------------------------
# A plain C client (tests/cpp/capi_multi.c): the batch entry point and the
# NCCL partitions at world 1, with no C++ and no PyTorch in the process.
C_SRC = os.path.join(ROOT, "tests", "cpp", "capi_multi.c")
C_BIN = os.path.join(ROOT, "build", "capi_multi")


def test_c_client_compiles_against_the_header():
    os.makedirs(os.path.dirname(C_BIN), exist_ok=True)
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), C_SRC, "-o",
                    C_BIN, "-L", LIBDIR, "-lbsm_cuda", f"-Wl,-rpath,{LIBDIR}"], check=True)


@pytest.mark.gpu
def test_c_client_batch_and_nccl_match_reference(tmp_path, ref, default_pairs):
    from paper_1402_2020_b200.synth import synth_pair
    test_c_client_compiles_against_the_header()
    W, H, D = 170, 41, 48
    pairs = [synth_pair(0, 50 + i, W, H) for i in range(3)]
    (tmp_path / "p.raw").write_bytes(b"".join(l.tobytes() + r.tobytes() for l, r in pairs))
    out = subprocess.run([C_BIN, str(W), str(H), str(D), str(tmp_path / "p.raw"), str(tmp_path / "o.bin")],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    raw = np.fromfile(tmp_path / "o.bin", np.uint8)
    px = W * H
    maps = [(raw[k * 5 * px:k * 5 * px + 4 * px].view(np.float32).reshape(H, W),
             raw[k * 5 * px + 4 * px:(k + 1) * 5 * px].reshape(H, W)) for k in range(len(raw) // (5 * px))]
    assert len(maps) == 3 + 1 + 3 + 1
    want = [ref.pipeline(l, r, default_pairs, 26, D, threads=8) for l, r in pairs]
    got_order = [0, 1, 2, 0, 0, 1, 2, 1]  # batch, frame bands of pair 0, sharded pairs, p2p frame of pair 1
    for (d, v), i in zip(maps, got_order):
        assert np.array_equal(d, want[i]["refined_d"]) and np.array_equal(v, want[i]["refined_v"])
