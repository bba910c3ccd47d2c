"""ctypes mirror of include/fic_b200.h (the C-ABI boundary).

The record layouts here are the single Python-side definition of `fic_params`,
`fic_mapping` and `fic_stats`; `MAPPING_DTYPE` is the matching numpy structured
dtype so code arrays cross the boundary without per-record conversion.
"""
import ctypes

import numpy as np

# Errc names in ordinal order (proj/include/fic/error.hpp:10-29); C code = ordinal + 1.
ERRC_NAMES = [
    "MalformedHeader", "UnsupportedMaxval", "TruncatedData", "NotSquare", "NotPowerOfTwo",
    "IndivisibleByRange", "TooSmallForDomain", "OddSide", "SideMismatch", "OutOfBounds",
    "NoValidPositions", "OutOfRange", "GeometryError", "ScaleMismatch", "DimensionMismatch",
    "NonContractive", "BadParams", "IoError",
]
FIC_OK = 0
FIC_ERR_CUDA = 100
FIC_ERR_INTERNAL = 101

INITIAL_KINDS = {"mid-gray": 0, "black": 1}
INITIAL_SUPPLIED = 2


def errc_name(code: int) -> str:
    if code == 0:
        return "Ok"
    if 1 <= code <= len(ERRC_NAMES):
        return ERRC_NAMES[code - 1]
    if code == FIC_ERR_CUDA:
        return "CudaError"
    return "InternalError"


class FicParams(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("step", ctypes.c_int32),
        ("s_bits", ctypes.c_int32),
        ("o_bits", ctypes.c_int32),
        ("s_max", ctypes.c_double),
        ("shadow_eps", ctypes.c_double),
    ]


class FicMapping(ctypes.Structure):
    _fields_ = [
        ("x", ctypes.c_int32),
        ("y", ctypes.c_int32),
        ("sym", ctypes.c_int32),
        ("qs", ctypes.c_uint32),
        ("qo", ctypes.c_uint32),
        ("reserved", ctypes.c_int32),
        ("residual", ctypes.c_double),
    ]


class FicStats(ctypes.Structure):
    _fields_ = [
        ("candidates_tested", ctypes.c_uint64),
        ("shadow_ranges", ctypes.c_uint64),
        ("shadow_codeblocks", ctypes.c_uint64),
    ]

    def as_dict(self):
        return {
            "candidates_tested": int(self.candidates_tested),
            "shadow_ranges": int(self.shadow_ranges),
            "shadow_codeblocks": int(self.shadow_codeblocks),
        }


class FicLinearFit(ctypes.Structure):  # LinearFit (proj/include/fic/encoder.hpp:15-19)
    _fields_ = [("s", ctypes.c_double), ("o", ctypes.c_double), ("residual", ctypes.c_double)]


class FicQuantizedFit(ctypes.Structure):  # QuantizedFit (proj/include/fic/encoder.hpp:24-30)
    _fields_ = [("qs", ctypes.c_uint32), ("qo", ctypes.c_uint32), ("s", ctypes.c_double), ("o", ctypes.c_double),
                ("residual", ctypes.c_double)]


MAPPING_DTYPE = np.dtype(
    [("x", "<i4"), ("y", "<i4"), ("sym", "<i4"), ("qs", "<u4"), ("qo", "<u4"),
     ("reserved", "<i4"), ("residual", "<f8")]
)
assert MAPPING_DTYPE.itemsize == ctypes.sizeof(FicMapping) == 32
assert ctypes.sizeof(FicParams) == 32


def make_params(n=4, step=0, s_bits=5, o_bits=7, s_max=1.0, shadow_eps=0.0) -> FicParams:
    return FicParams(int(n), int(step), int(s_bits), int(o_bits), float(s_max), float(shadow_eps))


def ptr(arr: np.ndarray, ctype=ctypes.c_void_p):
    """Raw pointer of a C-contiguous numpy array (or None for None)."""
    if arr is None:
        return None
    assert arr.flags["C_CONTIGUOUS"]
    return ctypes.cast(arr.ctypes.data, ctype)
