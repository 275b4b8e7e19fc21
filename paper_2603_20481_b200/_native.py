"""ctypes binding of the C ABI (include/specsense_b200.h).

Loads the in-tree ``_lib/libspecsense_b200.so`` and fails loudly when it is
missing -- there is no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("SSB_LIB_PATH") or Path(__file__).resolve().parent / "_lib" / "libspecsense_b200.so")

SS_OK, SS_EVALIDATION, SS_EFORMAT, SS_ECUDA, SS_ENOMEM, SS_EUNSUPPORTED, SS_ECAPACITY = range(7)
SS_FMT_F32, SS_FMT_I16 = 0, 1


class DetectorCfg(C.Structure):
    _fields_ = [("savgol_window", C.c_int), ("savgol_order", C.c_int), ("psd_margin_db", C.c_double),
                ("min_component_area", C.c_int), ("one_d_opening_along_time", C.c_int)]


class Box(C.Structure):
    _fields_ = [("f0_hz", C.c_double), ("f1_hz", C.c_double), ("t0_s", C.c_double), ("t1_s", C.c_double)]


class BinBox(C.Structure):
    _fields_ = [("t0", C.c_int32), ("t1", C.c_int32), ("f0", C.c_int32), ("f1", C.c_int32)]


class Extent(C.Structure):
    _fields_ = [("min_t", C.c_int64), ("max_t", C.c_int64), ("min_f", C.c_int64), ("max_f", C.c_int64),
                ("area", C.c_int64)]


class BatchOut(C.Structure):
    _fields_ = [("psd_raw", C.c_void_p), ("psd_smoothed", C.c_void_p), ("floor_thr", C.c_void_p),
                ("active", C.c_void_p), ("n_active", C.c_void_p), ("boxes", C.c_void_p),
                ("bin_boxes", C.c_void_p), ("n_boxes", C.c_void_p), ("box_capacity", C.c_int32)]


class BaselineCfg(C.Structure):
    _fields_ = [("conv_threshold", C.c_double), ("rate_change_threshold", C.c_double), ("noise_offset_db", C.c_double),
                ("max_kernel_rows", C.c_int), ("max_kernel_cols", C.c_int)]


class EngineCfg(C.Structure):
    _fields_ = [("n_fft", C.c_int), ("plot_rows", C.c_int), ("fmt", C.c_int), ("sample_rate_hz", C.c_double),
                ("n_banks", C.c_int), ("paced", C.c_int), ("deadline_s", C.c_double), ("box_capacity", C.c_int),
                ("hop", C.c_int), ("window", C.c_int), ("shard_count", C.c_int), ("shard_index", C.c_int),
                ("stage_timing", C.c_int)]


class PlotRecord(C.Structure):
    _fields_ = [("plot_index", C.c_uint64), ("start_seq", C.c_uint64), ("latency_s", C.c_double),
                ("deadline_s", C.c_double), ("met", C.c_int32), ("n_boxes", C.c_int32), ("n_active", C.c_int32),
                ("noise_floor", C.c_float), ("threshold", C.c_float), ("complete_s", C.c_double),
                ("done_s", C.c_double), ("gpu_s", C.c_double), ("stage_s", C.c_double * 8)]


# name -> (restype, argtypes); every symbol include/specsense_b200.h declares
_P = C.c_void_p
_I = C.c_int
SIGNATURES = {
    "ss_open": (_I, [_I, C.POINTER(_P)]),
    "ss_close": (None, [_P]),
    "ss_last_error": (C.c_char_p, [_P]),
    "ss_abi_version": (_I, []),
    "ss_default_detector_cfg": (None, [C.POINTER(DetectorCfg)]),
    "ss_set_stream": (_I, [_P, _P]),
    "ss_synchronize": (_I, [_P]),
    "ss_set_async": (_I, [_P, _I]),
    "ss_wait": (_I, [_P]),
    "ss_launch_count": (C.c_int64, [_P]),
    "ss_enable_stage_timing": (_I, [_P, _I]),
    "ss_stage_times": (_I, [_P, C.POINTER(C.c_double)]),
    "ss_tf_plots": (_I, [_P, _P, _I, _I, _I, _I, _P]),
    "ss_stft_plots": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "ss_stft_sense_batch": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, C.c_uint64, C.c_double, C.POINTER(DetectorCfg), _P,
                                 C.POINTER(BatchOut)]),
    "ss_psd_cols": (_I, [_P, _P, _I, _I, _I, _I, _P]),
    "ss_savgol_smooth": (_I, [_P, _P, _I, _I, _I, _P]),
    "ss_floor": (_I, [_P, _P, _I, C.POINTER(DetectorCfg), _P, _P, _P, C.POINTER(C.c_int32)]),
    "ss_prune": (_I, [_P, _P, _I, C.c_float, _P, C.POINTER(C.c_int32)]),
    "ss_otsu": (_I, [_P, _P, _I, C.POINTER(C.c_int32), C.POINTER(C.c_float)]),
    "ss_binarize_cols": (_I, [_P, _P, _I, _I, _P, _I, _I, _I, _P]),
    "ss_morph_cols": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "ss_consolidate": (_I, [_P, _P, _I, _I, _I, _P]),
    "ss_components": (_I, [_P, _P, _I, _I, _I, _P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "ss_detect_batch": (_I, [_P, _P, _I, _I, _I, _P, C.c_double, C.POINTER(DetectorCfg), C.POINTER(BatchOut)]),
    "ss_sense_batch": (_I, [_P, _P, _I, _I, _I, _I, C.c_uint64, C.c_double, C.POINTER(DetectorCfg), _P,
                            C.POINTER(BatchOut)]),
    "ss_test_libm": (_I, [_P, _P, C.c_int64, _I, _I, _P]),
    "ss_fft_twiddle_count": (C.c_int64, [_I]),
    "ss_fft_twiddles": (_I, [_I, _P]),
    "ss_default_baseline_cfg": (None, [C.POINTER(BaselineCfg)]),
    "ss_baseline_kernel_sizes": (_I, [_I, _I, C.POINTER(BaselineCfg), _P, _I]),
    "ss_baseline_detect": (_I, [_P, _P, _I, _I, C.c_uint64, C.c_double, C.POINTER(BaselineCfg), _P, _P, _I,
                                C.POINTER(_I)]),
    "ss_engine_open": (_I, [_I, C.POINTER(EngineCfg), C.POINTER(DetectorCfg), C.POINTER(_P)]),
    "ss_engine_close": (None, [_P]),
    "ss_engine_last_error": (C.c_char_p, [_P]),
    "ss_engine_push": (_I, [_P, _P, C.c_int64, C.c_uint64]),
    "ss_engine_push_async": (_I, [_P, _P, C.c_int64, C.c_uint64]),
    "ss_engine_push_fence": (_I, [_P]),
    "ss_engine_mark_lost": (_I, [_P, C.c_uint64, C.c_uint64]),
    "ss_engine_finish": (_I, [_P]),
    "ss_engine_poll": (_I, [_P, _I, C.POINTER(PlotRecord), _P, _P, _I, C.POINTER(_I)]),
    "ss_engine_stats": (_I, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                             C.POINTER(C.c_uint64)]),
}

_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load() -> C.CDLL:
    """Load the native library (RuntimeError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise RuntimeError(f"specsense-b200 native library missing at {_LIB_PATH}; "
                           "run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_LOCAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
