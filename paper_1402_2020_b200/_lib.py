"""ctypes binding of libbsm_cuda.so (include/bsm_cuda.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no CPU
fallback: if the shared library is missing or no CUDA device is usable, every
compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbsm_cuda.so")
SYNTH_PATH = os.path.join(_HERE, "libbsm_synth.so")

BSM_OK = 0
BSM_INVALID_ARGUMENT = 1
BSM_DIMENSION_MISMATCH = 2
BSM_CUDA_ERROR = 3
BSM_UNSUPPORTED = 4
BSM_NCCL_ERROR = 5


class BsmError(RuntimeError):
    """bsm::Error (errors.hpp:8-10)."""


class InvalidArgument(BsmError):
    """bsm::InvalidArgument (errors.hpp:20-22)."""


class DimensionMismatch(BsmError):
    """bsm::DimensionMismatch (errors.hpp:25-27)."""


class CudaError(BsmError):
    """Device failure or no usable device (this build has no CPU fallback)."""


class Unsupported(BsmError):
    """Valid input outside this build's envelope (e.g. n > 8192)."""


_EXC = {
    BSM_INVALID_ARGUMENT: InvalidArgument,
    BSM_DIMENSION_MISMATCH: DimensionMismatch,
    BSM_CUDA_ERROR: CudaError,
    BSM_UNSUPPORTED: Unsupported,
    BSM_NCCL_ERROR: BsmError,
}


class bsm_params(C.Structure):
    _fields_ = [
        ("d_max", C.c_int),
        ("lambda_c", C.c_double),
        ("lambda_e", C.c_double),
        ("lr_tolerance", C.c_double),
        ("vote_radius", C.c_int),
    ]


class bsm_maps(C.Structure):
    _fields_ = [
        ("refined_d", C.c_void_p),
        ("refined_v", C.c_void_p),
        ("left_d", C.c_void_p),
        ("right_d", C.c_void_p),
        ("checked_d", C.c_void_p),
        ("checked_v", C.c_void_p),
        ("unmasked_d", C.c_void_p),
    ]


_P = C.c_void_p
_I = C.c_int
_D = C.c_double

# name -> argtypes (all return int status unless listed in _RET)
_SIGS = {
    "bsm_ctx_create": [_I, C.POINTER(C.c_void_p)],
    "bsm_ctx_destroy": [_P],
    "bsm_generate_pattern": [_I, _I, _D, C.c_uint64, _P],
    "bsm_set_pattern": [_P, _P, _I, _I],
    "bsm_gray_lab_lut": [_P, _P],
    "bsm_to_gray_lab": [_P, _I, _I, _P, _P],
    "bsm_compute_field_u8": [_P, _P, _I, _I, _P, _P],
    "bsm_wta": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P],
    "bsm_lr_check": [_P, _P, _P, _I, _I, _D, _P, _P],
    "bsm_vote_refine_u8": [_P, _P, _P, _P, _I, _I, _D, _D, _I, _P, _P],
    "bsm_vote_refine_lab": [_P, _P, _P, _P, _I, _I, _D, _D, _I, _P, _P],
    "bsm_device_exp": [_P, _P, _I, _P],
    "bsm_set_refine_mode": [_P, _I],
    "bsm_pipeline_u8": [_P, _P, _P, _I, _I, C.POINTER(bsm_params), _I, C.POINTER(bsm_maps)],
    "bsm_pipeline_rgb": [_P, _P, _P, _I, _I, C.POINTER(bsm_params), _I, C.POINTER(bsm_maps)],
    "bsm_pipeline_rgb_device": [_P, _P, _P, _I, _I, C.POINTER(bsm_params), _I],
    "bsm_compute_field_f32": [_P, _P, _P, _I, _I, _P, _P],
    "bsm_rgb24_tables": [_P, _P],
    "bsm_pipeline_u8_device": [_P, _P, _P, _I, _I, C.POINTER(bsm_params), _I],
    "bsm_fetch_maps": [_P, C.POINTER(bsm_maps)],
    "bsm_pipeline_band_u8": [_P, _P, _P, _I, _I, _I, _I, C.POINTER(bsm_params), _P, _P],
    "bsm_pipeline_band_u8_device": [_P, _P, _P, _I, _I, _I, _I, C.POINTER(bsm_params)],
    "bsm_result_device": [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "bsm_copy_result_device": [_P, _P, _P],
    "bsm_pipeline_batch_u8": [_P, _I, _P, _P, _I, _I, C.POINTER(bsm_params), _P, _P],
    "bsm_pipeline_batch_u8_device": [_P, _I, _P, _P, _I, _I, C.POINTER(bsm_params), _P, _P],
    "bsm_comm_unique_id": [_P],
    "bsm_comm_create": [_P, _P, _I, _I, C.POINTER(C.c_void_p)],
    "bsm_comm_destroy": [_P],
    "bsm_pipeline_frame_bands_u8": [_P, _P, _P, _P, _I, _I, C.POINTER(bsm_params), _P, _P],
    "bsm_pipeline_pairs_sharded_u8": [_P, _P, _I, _P, _P, _I, _I, C.POINTER(bsm_params), _I, _P, _P],
    "bsm_frame_create": [_P, _I, _I, _I, _I, C.POINTER(C.c_void_p), _P],
    "bsm_frame_attach": [_P, _P],
    "bsm_pipeline_frame_bands_p2p_u8": [_P, _P, _P, _P, C.POINTER(bsm_params)],
    "bsm_frame_fetch": [_P, _P, _P],
    "bsm_frame_destroy": [_P],
    "bsm_stream": [_P, C.POINTER(C.c_void_p)],
    "bsm_stream_wait": [_P, _P],
    "bsm_debug_check_guards": [_P, C.POINTER(C.c_longlong), C.POINTER(C.c_int)],
    "bsm_set_profiling": [_P, _I],
    "bsm_last_timings": [_P, _P, _I, C.POINTER(C.c_int)],
    "bsm_last_launch_count": [_P, C.POINTER(C.c_int)],
    "bsm_measure_popc_peak": [_P, C.POINTER(C.c_double)],
    "bsm_measure_word_peaks": [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "bsm_measure_mma_peak": [_P, C.POINTER(C.c_double)],
}
_RET = {"bsm_last_error": C.c_char_p, "bsm_version": C.c_char_p, "bsm_timing_names": C.c_char_p}

_lib = None


def lib() -> C.CDLL:
    """Load libbsm_cuda.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(
                f"{LIB_PATH} is missing: run __graft_entry__.build(); there is no CPU fallback"
            )
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        for name, rt in _RET.items():
            f = getattr(L, name)
            f.argtypes = []
            f.restype = rt
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != BSM_OK:
        msg = lib().bsm_last_error().decode(errors="replace")
        raise _EXC.get(rc, BsmError)(msg)


def exported_symbols() -> list[str]:
    return sorted(list(_SIGS) + list(_RET))
