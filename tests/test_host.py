"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/bsm_cuda.h declares, its host pieces (pattern, colour
tables) match the reference bit for bit, and argument validation raises the
reference's exception types and messages."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1402_2020_b200 as bsm
from paper_1402_2020_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "bsm_cuda.h")).read()
    return sorted(set(re.findall(r"\b(bsm_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # the Python binding binds exactly the declared surface
    assert set(_lib.exported_symbols()) == set(names)


def test_io_library_exports_every_declared_symbol():
    """libbsm_io.so (include/bsm_io.h): the file / evaluation layer's C ABI,
    bound by io.py and evaluation.py."""
    from paper_1402_2020_b200 import io as bio
    txt = open(os.path.join(ROOT, "include", "bsm_io.h")).read()
    names = sorted(set(re.findall(r"\b(bsmio_[a-z0-9_]+)\s*\(", txt)))
    assert len(names) >= 14
    L = C.CDLL(bio.IO_PATH)
    assert not [n for n in names if not hasattr(L, n)]
    assert set(bio._SIGS) | {"bsmio_last_error"} == set(names)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pattern_matches_reference(ref):
    for n, S, sp, seed in [(4096, 26, 4.0, 42), (70, 6, 2.0, 37), (512, 12, 3.0, 9)]:
        p = bsm.generate_pattern(n, S, sp, seed)
        assert np.array_equal(p.pairs, ref.generate_pattern(n, S, sp, seed))


def test_lut_matches_reference(ref):
    g, l = bsm.gray_lab_lut()
    g2, l2 = ref.gray_lab_lut()
    assert np.array_equal(g.view(np.uint32), g2.view(np.uint32))
    assert np.array_equal(l.view(np.uint32), l2.view(np.uint32))


def test_rgb_conversion_matches_reference(ref):
    rgb = np.random.default_rng(4).integers(0, 256, size=(17, 23, 3), dtype=np.uint8)
    g, l = bsm.to_gray_lab(rgb)
    g2, l2 = ref.to_gray_lab(rgb)
    assert np.array_equal(g.view(np.uint32), g2.view(np.uint32))
    assert np.array_equal(l.view(np.uint32), l2.view(np.uint32))


def test_rgb24_tables_match_reference_exhaustively(ref):
    # every 24-bit colour, in 16 slices of 2^20 (index (r << 16) | (g << 8) | b)
    g, l = bsm.rgb24_tables()
    k = np.arange(1 << 20, dtype=np.uint32)
    for s in range(16):
        idx = k + (s << 20)
        rgb = np.stack([(idx >> 16) & 255, (idx >> 8) & 255, idx & 255], axis=-1).astype(np.uint8)
        g2, l2 = ref.to_gray_lab(rgb.reshape(1024, 1024, 3))
        assert np.array_equal(g[idx].view(np.uint32), g2.reshape(-1).view(np.uint32)), s
        assert np.array_equal(l[idx].view(np.uint32), l2.reshape(-1, 3).view(np.uint32)), s


def test_pattern_errors():
    with pytest.raises(bsm.InvalidArgument, match="n must be >= 1"):
        bsm.generate_pattern(0)
    with pytest.raises(bsm.InvalidArgument, match="window must be >= 2"):
        bsm.generate_pattern(16, 1)
    with pytest.raises(bsm.InvalidArgument, match="spread must be > 0"):
        bsm.generate_pattern(16, 4, 0.0)


def test_config_validate_messages():
    # config.hpp:30-44
    cases = [
        (dict(n=0, d_max=4), "n must be >= 1"),
        (dict(window=1, d_max=4), "S must be >= 2"),
        (dict(spread=0.0, d_max=4), "spread must be > 0"),
        (dict(), "d_max must be set"),
        (dict(d_max=4, lambda_c=0.0), "lambda_c must be > 0"),
        (dict(d_max=4, lambda_e=-1.0), "lambda_e must be > 0"),
        (dict(d_max=4, lr_tolerance=-1.0), "lr_tolerance must be >= 0"),
        (dict(d_max=4, vote_radius=0), "vote_radius must be >= 1"),
        (dict(d_max=4, gt_scale=0.0), "gt_scale must be > 0"),
        (dict(d_max=4, threads=0), "threads must be >= 1"),
        (dict(d_max=4, generator="x"), "unknown generator"),
    ]
    for kw, msg in cases:
        with pytest.raises(bsm.InvalidArgument, match=msg):
            bsm.BsmConfig(**kw).validate()
    bsm.BsmConfig(d_max=4).validate()


def test_api_validation_before_device():
    a = np.zeros((4, 5), np.uint8)
    with pytest.raises(bsm.DimensionMismatch, match="left/right dimensions differ"):
        bsm.run_pipeline(a, np.zeros((4, 6), np.uint8), bsm.BsmConfig(d_max=3))
    with pytest.raises(bsm.InvalidArgument, match="d_max"):
        bsm.run_pipeline(a, a, bsm.BsmConfig())
    with pytest.raises(bsm.InvalidArgument, match="uint8"):
        bsm.run_pipeline(a.astype(np.float32), a, bsm.BsmConfig(d_max=3))
    m = bsm.DisparityMap(np.zeros((4, 4), np.float32), np.ones((4, 4), np.uint8))
    m2 = bsm.DisparityMap(np.zeros((4, 5), np.float32), np.ones((4, 5), np.uint8))
    with pytest.raises(bsm.DimensionMismatch, match="map dimensions differ"):
        bsm.lr_check(m, m2, 1.0)
    with pytest.raises(bsm.DimensionMismatch, match="map/image dimensions differ"):
        bsm.vote_refine(m, a)
    with pytest.raises(bsm.InvalidArgument, match="lambda_c"):
        bsm.vote_refine(m, np.zeros((4, 4), np.uint8), lambda_c=0)
    f = np.zeros((4, 4, 1), np.uint64)
    with pytest.raises(bsm.DimensionMismatch, match="do not agree in size"):
        bsm.wta(f, f, np.zeros((4, 5, 1), np.uint64), 3)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    with pytest.raises(bsm.CudaError, match="no CPU fallback"):
        bsm.Context(0)


def test_c_abi_null_and_range_checks():
    L = _lib.lib()
    assert L.bsm_ctx_create(0, None) == _lib.BSM_INVALID_ARGUMENT
    assert L.bsm_generate_pattern(4, 4, 1.0, 1, None) == _lib.BSM_INVALID_ARGUMENT
    assert L.bsm_set_pattern(None, None, 4, 4) == _lib.BSM_INVALID_ARGUMENT
    assert L.bsm_pipeline_u8(None, None, None, 4, 4, None, 0, None) == _lib.BSM_INVALID_ARGUMENT
    assert b"null" in L.bsm_last_error()
    names = L.bsm_timing_names().decode().split(",")
    assert names[:3] == ["h2d", "descriptor", "mask"]
