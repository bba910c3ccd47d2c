"""Loader for libfic_b200.so — the CUDA library behind the C-ABI (include/fic_b200.h).

There is no fallback: if the library is missing or fails to load, every entry point
raises.  `build()` (or `python -m paper_1404_0774_b200.build`) produces the library
in-tree.
"""
import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FIC_LIB") or os.path.join(HERE, "libfic_b200.so")

_lock = threading.Lock()
_lib = None


class ExtensionMissing(RuntimeError):
    pass


def _declare(L):
    vp, i32, u64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
    L.fic_last_error.restype = ctypes.c_char_p
    L.fic_errc_name.argtypes = [i32]
    L.fic_errc_name.restype = ctypes.c_char_p
    L.fic_version.restype = ctypes.c_char_p
    L.fic_normalize_params.argtypes = [vp, vp]
    L.fic_validate_geometry.argtypes = [i32, i32, vp]
    L.fic_encode.argtypes = [vp, i32, i32, vp, vp, vp]
    L.fic_encode_parallel.argtypes = [vp, i32, i32, vp, i32, i32, i32, vp, vp]
    L.fic_encode_range.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp]
    L.fic_encode_rows.argtypes = [vp, i32, i32, vp, i32, i32, vp, vp]
    L.fic_encode_batch.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    L.fic_encode_device.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.fic_encode_batch_device.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp]
    L.fic_encode_rows_device.argtypes = [vp, i32, i32, vp, i32, i32, vp, vp, vp]
    i64 = ctypes.c_int64
    L.fic_record_layout.argtypes = [i32, i32, vp, vp, vp]
    L.fic_serialize.argtypes = [vp, i32, i32, vp, vp, i64, vp]
    L.fic_serialize_device.argtypes = [vp, i32, i32, vp, vp, i64, vp, vp]
    L.fic_deserialize.argtypes = [vp, i64, vp, vp, vp, vp, i64, vp]
    L.fic_decode_step.argtypes = [vp, i32, i32, vp, i32, i32, vp, i32, vp]
    L.fic_decode.argtypes = [vp, i32, i32, vp, i32, i32, i32, vp, i32, i32, i32, f64, vp, vp, vp]
    L.fic_collage_error.argtypes = [vp, i32, i32, vp, i32, i32, vp, vp]
    L.fic_decoded_error_bound.argtypes = [f64, f64, vp]
    L.fic_kernel_launch_count.restype = u64
    L.fic_matcher_timing.argtypes = [vp, vp, i32]
    L.fic_set_matcher_timing.argtypes = [i32]
    L.fic_scan_timing.argtypes = [vp, vp, i32]
    L.fic_scan_expand_timing.argtypes = [vp, vp, i32]
    L.fic_last_survivors.argtypes = [vp, i32]
    L.fic_debug_trace.argtypes = [vp, i32]
    L.fic_decode_timing.argtypes = [vp, vp, vp, i32]
    L.fic_pool_timing.argtypes = [vp, vp, vp, i32]
    L.fic_is_shadow.argtypes = [vp, i32, f64, vp]
    L.fic_least_squares_fit.argtypes = [vp, i32, vp, i32, f64, vp]
    L.fic_least_squares_clamped.argtypes = [vp, i32, vp, i32, vp, vp]
    L.fic_least_squares.argtypes = [vp, i32, vp, i32, vp, vp]
    L.fic_debug_pool.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp]
    L.fic_set_device.argtypes = [i32]
    L.fic_device_count.argtypes = [vp]
    for name in ["fic_normalize_params", "fic_validate_geometry", "fic_encode", "fic_encode_parallel",
                 "fic_encode_range", "fic_encode_rows", "fic_encode_batch", "fic_encode_device",
                 "fic_decode_step", "fic_decode", "fic_collage_error", "fic_decoded_error_bound",
                 "fic_matcher_timing", "fic_set_device", "fic_device_count", "fic_scan_timing",
                 "fic_scan_expand_timing", "fic_last_survivors", "fic_decode_timing", "fic_encode_batch_device", "fic_debug_trace",
                 "fic_is_shadow", "fic_least_squares_fit", "fic_least_squares_clamped", "fic_least_squares",
                 "fic_debug_pool", "fic_pool_timing", "fic_encode_rows_device", "fic_record_layout",
                 "fic_serialize", "fic_serialize_device", "fic_deserialize"]:
        getattr(L, name).restype = i32
    return L


def lib():
    """The loaded library (loaded once, on first use)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ExtensionMissing(
                        f"{LIB_PATH} is not built; run `python -m paper_1404_0774_b200.build` "
                        "(there is no CPU fallback)")
                _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


# Every symbol include/fic_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "fic_last_error", "fic_errc_name", "fic_version", "fic_normalize_params", "fic_validate_geometry",
    "fic_encode", "fic_encode_parallel", "fic_encode_range", "fic_encode_rows", "fic_encode_batch",
    "fic_encode_device", "fic_decode_step", "fic_decode", "fic_collage_error", "fic_decoded_error_bound",
    "fic_kernel_launch_count", "fic_matcher_timing", "fic_set_matcher_timing", "fic_set_device",
    "fic_device_count", "fic_scan_timing", "fic_scan_expand_timing", "fic_last_survivors", "fic_decode_timing", "fic_encode_batch_device",
    "fic_debug_trace", "fic_is_shadow", "fic_least_squares_fit", "fic_least_squares_clamped", "fic_least_squares",
    "fic_debug_pool", "fic_pool_timing", "fic_encode_rows_device", "fic_record_layout", "fic_serialize",
    "fic_serialize_device", "fic_deserialize",
]
