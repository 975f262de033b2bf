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
                        "-L", LIBDIR, "-lbsm_cuda", f"-Wl,-rpath,{LIBDIR}"], check=True)
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
