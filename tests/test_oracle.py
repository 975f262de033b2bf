"""Pin the checkers (CPU, no GPU needed).

1. The C restatement (oracle/bsm_oracle.c) against the reference library
   compiled in place (oracle/_ref) on seeded inputs.
2. Both against the known-answer values of the reference's own GoogleTest
   suite (proj/tests/*.cpp), restated here.
3. The golden fixtures (tests/golden) against the reference on the small
   BASELINE workload c1 maps file.
"""
import json
import os

import numpy as np
import pytest

from conftest import random_u8

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(s: str) -> np.ndarray:
    """BitString::from_bits (bitstring.hpp:33-43) for <= 64 bits."""
    w = 0
    for i, ch in enumerate(s):
        if ch == "1":
            w |= 1 << i
    return np.array([w], np.uint64)


# --------------------------------------------------------------------------
# Known answers (test_matcher.cpp, test_descriptor.cpp, test_refine.cpp,
# test_image.cpp, test_pattern.cpp)
@pytest.mark.parametrize("lib", ["ref", "orc"])
def test_masked_hamming_known_answers(lib, request):
    L = request.getfixturevalue(lib)
    a, b = bits("1010"), bits("0110")
    assert L.masked_hamming_words(a, b, bits("1111")) == 2   # test_matcher.cpp:33-39
    assert L.masked_hamming_words(a, b, bits("1000")) == 1
    assert L.masked_hamming_words(a, b, bits("0000")) == 0


@pytest.mark.parametrize("lib", ["ref", "orc"])
def test_quarter_threshold_known_answers(lib, request):
    L = request.getfixturevalue(lib)
    assert L.quarter_threshold([1, 2, 3, 4, 5, 6, 7, 8]) == 2.0   # test_descriptor.cpp:64-72
    assert L.quarter_threshold([8, 7, 6, 5, 4, 3, 2, 1]) == 2.0
    assert L.quarter_threshold([5.0] * 8) == 5.0
    assert L.quarter_threshold([9, 3]) == 3.0


def test_quarter_threshold_matches_reference(ref, orc):
    rng = np.random.default_rng(11)  # test_descriptor.cpp:74-83
    for n in (8, 64, 4096):
        for _ in range(20):
            w = (rng.integers(0, 1000, size=n) / 8.0).astype(np.float32)
            s = np.sort(w)[max(1, n // 4) - 1]
            assert ref.quarter_threshold(w) == s == orc.quarter_threshold(w)


def test_masked_hamming_random_triples(ref, orc):
    rng = np.random.default_rng(2024)  # acceptance.cpp:247-263 (1000 triples of 4096 bits)
    for _ in range(200):
        a, b, m = (rng.integers(0, 2**63, size=64, dtype=np.uint64) for _ in range(3))
        want = sum(bin(int(x)).count("1") for x in (a ^ b) & m)
        assert ref.masked_hamming_words(a, b, m) == want == orc.masked_hamming_words(a, b, m)


@pytest.mark.parametrize("lib", ["ref", "orc"])
def test_gray_lab_lut(lib, request, ref):
    L = request.getfixturevalue(lib)
    g, lab = L.gray_lab_lut()
    g_ref, lab_ref = ref.gray_lab_lut()
    assert np.array_equal(g.view(np.uint32), g_ref.view(np.uint32))
    assert np.array_equal(lab.view(np.uint32), lab_ref.view(np.uint32))
    assert np.all(np.diff(g) > 0)  # strictly increasing: u8 compares == float compares
    assert lab[255][0] == pytest.approx(100.0, abs=1e-4) and abs(lab[255][1]) < 1e-3


@pytest.mark.parametrize("lib", ["ref", "orc"])
def test_lab_red_known_answer(lib, request, ref):
    # test_image.cpp:49-54: red -> (53.2408, 80.0925, 67.2032) +- 0.01
    L = request.getfixturevalue(lib)
    rgb = np.array([[[255, 0, 0], [0, 255, 0], [10, 200, 30]]], np.uint8)
    g, lab = L.to_gray_lab(rgb)
    assert lab[0, 0] == pytest.approx([53.2408, 80.0925, 67.2032], abs=0.01)
    g2, lab2 = ref.to_gray_lab(rgb)
    assert np.array_equal(g.view(np.uint32), g2.view(np.uint32))
    assert np.array_equal(lab.view(np.uint32), lab2.view(np.uint32))


def test_pattern_matches_reference(ref, orc):
    for n, S, sp, seed in [(4096, 26, 4.0, 42), (70, 6, 2.0, 37), (128, 8, 2.0, 5), (16, 4, 1.5, 9)]:
        a = ref.generate_pattern(n, S, sp, seed)
        b = orc.generate_pattern(n, S, sp, seed)
        assert np.array_equal(a, b)
        half = S // 2
        assert np.abs(a).max() <= half
        assert not np.any((a[:, 0] == a[:, 2]) & (a[:, 1] == a[:, 3]))  # no degenerate pairs


def test_vote_weight_known_answers(ref, orc):
    # test_refine.cpp:104-122: 0.9394 and 0.1194 to 1e-4
    x = np.array([50.0, 0.0, 0.0], np.float32)
    p2 = np.array([60.0, 4.0, -4.0], np.float32)
    for L in (ref, orc):
        assert L.vote_weight(x, x, 1, 0, 9.0, 16.0) == pytest.approx(0.9394, abs=1e-4)
        assert L.vote_weight(x, p2, 2, 0, 9.0, 16.0) == pytest.approx(0.1194, abs=1e-4)
    assert ref.vote_weight(x, p2, 2, 0, 9.0, 16.0) == orc.vote_weight(x, p2, 2, 0, 9.0, 16.0)


@pytest.mark.parametrize("lib", ["ref", "orc"])
def test_lr_check_known_answers(lib, request):
    L = request.getfixturevalue(lib)
    c = lambda v: np.full((1, 10), v, np.float32)
    assert L.lr_check(c(5), c(5), 1.0)[1][0, 7] == 1      # test_refine.cpp:58-86
    d, v = L.lr_check(c(5), c(2), 1.0)
    assert v[0, 7] == 0 and d[0, 7] == 5.0
    assert L.lr_check(c(5), c(5), 1.0)[1][0, 3] == 0
    assert L.lr_check(c(5), c(4), 1.0)[1][0, 7] == 1
    assert L.lr_check(c(5), c(4), 0.5)[1][0, 7] == 0


# --------------------------------------------------------------------------
# Restatement == reference on seeded inputs
@pytest.mark.parametrize("n,window,spread,seed,h,w", [
    (4096, 26, 4.0, 42, 9, 30), (70, 6, 2.0, 37, 6, 6), (96, 16, 4.0, 29, 7, 11), (64, 8, 2.0, 5, 1, 1)])
def test_field_restatement_matches_reference(ref, orc, n, window, spread, seed, h, w):
    pairs = ref.generate_pattern(n, window, spread, seed)
    img = random_u8(h, w, seed)
    d1, m1 = ref.compute_field_u8(img, pairs, window)
    d2, m2 = orc.compute_field_u8(img, pairs, window)
    assert np.array_equal(d1, d2) and np.array_equal(m1, m2)
    words = (n + 63) // 64
    if n % 64:
        assert np.all(d1[..., words - 1] >> np.uint64(n % 64) == 0)  # pad bits zero
        assert np.all(m1[..., words - 1] >> np.uint64(n % 64) == 0)


def test_wta_restatement_matches_reference(ref, orc):
    rng = np.random.default_rng(3)
    H, W, n = 4, 40, 128
    f = lambda: rng.integers(0, 2**63, size=(H, W, 2), dtype=np.uint64)
    a, m, b = f(), f(), f()
    for d_max in (1, 5, 8, 60):
        for rr in (0, 1):
            for um in (True, False):
                assert np.array_equal(ref.wta(a, m, b, n, d_max, rr, um), orc.wta(a, m, b, n, d_max, rr, um))


def test_vote_refine_restatement_matches_reference(ref, orc):
    rng = np.random.default_rng(13)
    _, lab256 = ref.gray_lab_lut()
    for trial in range(3):
        img = random_u8(16, 16, trial)
        d = rng.integers(0, 10, size=(16, 16)).astype(np.float32)
        v = (rng.integers(0, 5, size=(16, 16)) < 3).astype(np.uint8)
        for radius in (3, 20):
            r1 = ref.vote_refine(d, v, lab256[img], 9.0, 16.0, radius)
            r2 = orc.vote_refine(d, v, lab256[img], 9.0, 16.0, radius)
            assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])


def test_pipeline_restatement_matches_reference(ref, orc, default_pairs):
    from paper_1402_2020_b200.synth import workload_pair
    left, right = workload_pair("c1")
    L, R = left[200:230, 100:200].copy(), right[200:230, 100:200].copy()
    want = ref.pipeline(L, R, default_pairs, 26, 40, threads=4)
    got = orc.pipeline_u8(L, R, default_pairs, 26, 40)
    for k in got:
        assert np.array_equal(got[k], want[k]), k


def test_reference_thread_count_determinism(ref, default_pairs):
    # test_pipeline.cpp:42-63: output independent of the thread count
    from paper_1402_2020_b200.synth import workload_pair
    left, right = workload_pair("c3")
    L, R = left[100:140, 100:220].copy(), right[100:140, 100:220].copy()
    a = ref.pipeline(L, R, default_pairs, 26, 64, threads=1)
    b = ref.pipeline(L, R, default_pairs, 26, 64, threads=8)
    for k in ("refined_d", "refined_v", "checked_v"):
        assert np.array_equal(a[k], b[k])


# --------------------------------------------------------------------------
# Golden fixtures
def test_golden_c1_maps_consistent_with_hashes():
    import hashlib
    g = json.load(open(os.path.join(GOLDEN, "c1.json")))
    z = np.load(os.path.join(GOLDEN, "c1_maps.npz"))
    for k, h in g["maps"].items():
        a = z[k].astype(np.float32) if k.endswith("_d") else z[k]
        assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == h, k


def test_golden_inputs_reproducible():
    import hashlib
    from paper_1402_2020_b200.synth import workload_pair
    for key in ("c1", "c3", "c2"):
        g = json.load(open(os.path.join(GOLDEN, f"{key}.json")))
        left, right = workload_pair(key)
        assert hashlib.sha256(left.tobytes()).hexdigest() == g["inputs"]["left"]
        assert hashlib.sha256(right.tobytes()).hexdigest() == g["inputs"]["right"]


def test_golden_c1_matches_restatement_sample(orc, default_pairs):
    """The golden c1 maps (reference) reproduced by the restatement on a band."""
    from paper_1402_2020_b200.synth import workload_pair
    z = np.load(os.path.join(GOLDEN, "c1_maps.npz"))
    left, right = workload_pair("c1")
    # the left/right WTA of interior rows depend only on rows within the window
    y0, y1 = 180, 186
    L, R = left[y0 - 13:y1 + 13], right[y0 - 13:y1 + 13]
    got = orc.pipeline_u8(L, R, default_pairs, 26, 60)
    assert np.array_equal(got["left_d"][13:-13], z["left_d"][y0:y1].astype(np.float32))
    assert np.array_equal(got["right_d"][13:-13], z["right_d"][y0:y1].astype(np.float32))
