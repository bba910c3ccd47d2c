"""FIC1 container (proj/src/format.cpp:105-185): 20-byte little-endian header plus one
byte-aligned, MSB-first record per range.  The records are packed and
unpacked on the device behind the C-ABI (csrc/fic1.cu: fic_serialize / fic_deserialize /
fic_serialize_device); this module is the Python surface over it.
"""
import ctypes

import numpy as np

from . import abi
from ._lib import lib
from .abi import MAPPING_DTYPE, FicParams, ptr

MAGIC = b"FIC1"
HEADER_BYTES = 20


def _check(rc):
    from .codec import _check as check
    check(rc)


def record_layout(width, height, p):
    """record_layout (format.cpp:78-89): (positions x, positions y, field widths, record bytes)."""
    f = (ctypes.c_int32 * 7)()
    nbytes = ctypes.c_int32()
    _check(lib().fic_record_layout(int(width), int(height), ctypes.byref(p.struct), f, ctypes.byref(nbytes)))
    return int(f[5]), int(f[6]), [int(f[i]) for i in range(5)], int(nbytes.value)


def serialize(enc):
    """serialize (format.cpp:105-141) -> bytes; the records are packed on the device."""
    from .codec import CodecError
    p = enc.params
    m = np.ascontiguousarray(enc.mappings, MAPPING_DTYPE)
    count = (enc.width // p.n) * (enc.height // p.n)
    if len(m) != count:
        raise CodecError(abi.ERRC_NAMES.index("BadParams") + 1, f"mapping count {len(m)} != range count {count}")
    size = ctypes.c_int64()
    L = lib()
    _check(L.fic_serialize(ptr(m), int(enc.width), int(enc.height), ctypes.byref(p.struct), None, 0,
                           ctypes.byref(size)))
    out = np.empty(size.value, np.uint8)
    _check(L.fic_serialize(ptr(m), int(enc.width), int(enc.height), ctypes.byref(p.struct), ptr(out),
                           int(size.value), ctypes.byref(size)))
    return out.tobytes()


def serialize_device(d_maps_ptr, width, height, params, d_out_ptr=None, cap=0, stream=0):
    """(extension) FIC1 bytes of device-resident records packed into device memory on `stream`
    (e.g. rank 0's gathered codes).  Without `d_out_ptr`, returns only the byte count."""
    size = ctypes.c_int64()
    _check(lib().fic_serialize_device(ctypes.c_void_p(d_maps_ptr), int(width), int(height),
                                      ctypes.byref(params.struct), ctypes.c_void_p(d_out_ptr or 0), int(cap),
                                      ctypes.byref(size), ctypes.c_void_p(stream)))
    return int(size.value)


def deserialize(data):
    """deserialize (format.cpp:143-185) -> EncodedImage; the records are unpacked on the device."""
    from .codec import CodecParams, EncodedImage
    b = np.frombuffer(bytes(data), np.uint8)
    w, h = ctypes.c_int32(), ctypes.c_int32()
    fp = FicParams()
    count = ctypes.c_int64()
    L = lib()
    _check(L.fic_deserialize(ptr(b) if len(b) else None, len(b), ctypes.byref(w), ctypes.byref(h), ctypes.byref(fp),
                             None, 0, ctypes.byref(count)))
    m = np.zeros(max(count.value, 1), MAPPING_DTYPE)
    _check(L.fic_deserialize(ptr(b), len(b), ctypes.byref(w), ctypes.byref(h), ctypes.byref(fp), ptr(m),
                             int(count.value), ctypes.byref(count)))
    return EncodedImage(w.value, h.value, CodecParams._from_struct(fp), m[: count.value])
