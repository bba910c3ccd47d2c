"""Python surface of the codec — the `fic` module API (proj/python/bindings/module.cpp:42-189,
proj/python/fic/__init__.py) re-hosted on the C-ABI of libfic_b200.so.

Same names, argument meanings and error behaviour as the reference bindings:
`CodecError` carries the reference's "Name: detail" text, `CodecParams(...)` normalises
on construction (module.cpp:49-62), `encode` validates workers/chunk only when
workers > 1 (module.cpp:101-102), `decode` accepts 'mid-gray' | 'black' | uint8 array
(module.cpp:109-140).  Extensions beyond the reference surface (stats, ranges, row
shards, batches, traced decode) are marked as such.
"""
import ctypes

import numpy as np

from . import abi
from ._lib import lib
from .abi import MAPPING_DTYPE, FicParams, FicStats, ptr


class CodecError(RuntimeError):
    """fic.CodecError (module.cpp:45): message is "<Errc name>: <detail>"."""

    def __init__(self, code, detail=""):
        self.code = int(code)
        self.name = abi.errc_name(self.code)
        msg = self.name if not detail else f"{self.name}: {detail}"
        super().__init__(msg)


def _check(rc):
    if rc != 0:
        raise CodecError(rc, lib().fic_last_error().decode(errors="replace"))


class CodecParams:
    """CodecParams (proj/include/fic/params.hpp:8-24), normalised at construction."""

    __slots__ = ("_p",)

    def __init__(self, n=4, step=0, s_bits=5, o_bits=7, s_max=1.0, shadow_eps=0.0):
        raw = abi.make_params(n, step, s_bits, o_bits, s_max, shadow_eps)
        out = FicParams()
        _check(lib().fic_normalize_params(ctypes.byref(raw), ctypes.byref(out)))
        self._p = out

    @classmethod
    def _from_struct(cls, p):
        obj = cls.__new__(cls)
        obj._p = p
        return obj

    n = property(lambda self: self._p.n)
    step = property(lambda self: self._p.step)
    s_bits = property(lambda self: self._p.s_bits)
    o_bits = property(lambda self: self._p.o_bits)
    s_max = property(lambda self: self._p.s_max)
    shadow_eps = property(lambda self: self._p.shadow_eps)

    @property
    def struct(self):
        return self._p

    def __eq__(self, other):
        return isinstance(other, CodecParams) and all(
            getattr(self, f) == getattr(other, f) for f in ("n", "step", "s_bits", "o_bits", "s_max", "shadow_eps"))

    def __repr__(self):  # module.cpp:69-73 (std::to_string -> 6 decimals)
        return (f"CodecParams(n={self.n}, step={self.step}, s_bits={self.s_bits}, o_bits={self.o_bits}, "
                f"s_max={self.s_max:.6f})")


class EncodedImage:
    """EncodedImage (proj/include/fic/encoded_image.hpp:30-41): header + row-major mappings.

    `mappings` is a numpy array of MAPPING_DTYPE records (x, y, sym, qs, qo, reserved,
    residual); `stats` (extension) holds EncodeStats of the encode that produced it."""

    def __init__(self, width, height, params, mappings, stats=None):
        self.width = int(width)
        self.height = int(height)
        self.params = params
        self.mappings = mappings
        self.stats = stats

    @property
    def mapping_count(self):
        return int(len(self.mappings))

    def serialize(self):
        from .fic1 import serialize
        return serialize(self)

    @staticmethod
    def deserialize(data):
        from .fic1 import deserialize
        return deserialize(data)

    def __eq__(self, other):  # RangeMapping equality ignores the residual (encoded_image.hpp:23-25)
        if not isinstance(other, EncodedImage):
            return NotImplemented
        keys = ["x", "y", "sym", "qs", "qo"]
        return (self.width == other.width and self.height == other.height and self.params == other.params
                and len(self.mappings) == len(other.mappings)
                and all(np.array_equal(self.mappings[k], other.mappings[k]) for k in keys))

    def __repr__(self):
        return f"EncodedImage({self.width}x{self.height}, {self.mapping_count} mappings)"


def _u8_2d(image):
    arr = np.ascontiguousarray(np.asarray(image), dtype=np.uint8)
    if arr.ndim != 2:
        raise ValueError("expected a 2D uint8 array (height x width)")
    return arr


def _range_count(h, w, p):
    return (w // p.n) * (h // p.n) if p.n > 0 else 0


def encode(image, params=None, workers=1, chunk=(16, 16), out=None):
    """Full-search PIFS encode (module.cpp:94-107 -> encode_sequential / encode_parallel).
    (extension) `out`: a caller-owned MAPPING_DTYPE array of at least (w/n)*(h/n) records to
    encode into (page-locked memory, e.g. a pinned torch tensor's numpy view, is filled by DMA
    directly, as a page-locked `image` is read); the result's mappings are a view of it."""
    params = CodecParams() if params is None else params
    img = _u8_2d(image)
    h, w = img.shape
    count = _range_count(h, w, params)
    if out is None:
        out = np.zeros(max(count, 1), MAPPING_DTYPE)
    elif out.dtype != MAPPING_DTYPE or out.ndim != 1 or len(out) < count or not out.flags.c_contiguous:
        raise ValueError(f"out must be a contiguous MAPPING_DTYPE array of at least {count} records")
    st = FicStats()
    L = lib()
    if workers > 1:
        rc = L.fic_encode_parallel(ptr(img), w, h, ctypes.byref(params.struct), int(workers), int(chunk[0]),
                                   int(chunk[1]), ptr(out), ctypes.byref(st))
    else:
        rc = L.fic_encode(ptr(img), w, h, ctypes.byref(params.struct), ptr(out), ctypes.byref(st))
    _check(rc)
    return EncodedImage(w, h, params, out[:count], st.as_dict())


def encode_with_stats(image, params=None):
    """(extension) encode plus EncodeStats (proj/include/fic/encoder.hpp:49-53) as a dict."""
    enc = encode(image, params)
    return enc, enc.stats


def encode_range(image, x, y, params=None):
    """(extension) encode_range (proj/src/encoder.cpp:332-342): (record, stats)."""
    params = CodecParams() if params is None else params
    img = _u8_2d(image)
    h, w = img.shape
    out = np.zeros(1, MAPPING_DTYPE)
    st = FicStats()
    _check(lib().fic_encode_range(ptr(img), w, h, int(x), int(y), ctypes.byref(params.struct), ptr(out),
                                  ctypes.byref(st)))
    return out[0], st.as_dict()


def encode_rows(image, row_begin, row_end, params=None):
    """(extension) encode range rows [row_begin, row_end) only — the per-rank shard of the
    multi-GPU encoder.  Returns (records, stats)."""
    params = CodecParams() if params is None else params
    img = _u8_2d(image)
    h, w = img.shape
    count = max(0, row_end - row_begin) * (w // params.n)
    out = np.zeros(max(count, 1), MAPPING_DTYPE)
    st = FicStats()
    _check(lib().fic_encode_rows(ptr(img), w, h, ctypes.byref(params.struct), int(row_begin), int(row_end),
                                 ptr(out), ctypes.byref(st)))
    return out[:count], st.as_dict()


def encode_batch(images, params=None, out=None):
    """(extension) encode a (count, side, side) uint8 volume (up to 64 slices per encode pass,
    pipelined: the next pass uploads while the current one encodes; each slice's codes equal its
    own fic_encode); returns a list of EncodedImage (views of one record array) and the summed
    stats.  `out`: a caller-owned MAPPING_DTYPE array of at least count*(w/n)*(h/n) records (a
    page-locked one, like a page-locked volume, is filled by DMA directly)."""
    params = CodecParams() if params is None else params
    vol = np.ascontiguousarray(np.asarray(images), dtype=np.uint8)
    if vol.ndim != 3:
        raise ValueError("expected a 3D uint8 array (count x height x width)")
    c, h, w = vol.shape
    per = _range_count(h, w, params)
    if out is None:
        out = np.empty(max(c * per, 1), MAPPING_DTYPE)
    elif out.dtype != MAPPING_DTYPE or out.ndim != 1 or len(out) < c * per or not out.flags.c_contiguous:
        raise ValueError(f"out must be a contiguous MAPPING_DTYPE array of at least {c * per} records")
    st = FicStats()
    _check(lib().fic_encode_batch(ptr(vol), c, w, h, ctypes.byref(params.struct), ptr(out), ctypes.byref(st)))
    return [EncodedImage(w, h, params, out[i * per:(i + 1) * per]) for i in range(c)], st.as_dict()


def _maps(enc):
    m = np.ascontiguousarray(enc.mappings, MAPPING_DTYPE)
    if len(m) != _range_count(enc.height, enc.width, enc.params):
        raise CodecError(abi.ERRC_NAMES.index("BadParams") + 1, "mapping count does not cover the range grid")
    return m


def decode_traced(enc, scale=1, iterations=16, initial="mid-gray", convergence_eps=None):
    """(extension) decode_traced (proj/src/decoder.cpp:113-128): (image, step_rmse, iterations_run)."""
    maps = _maps(enc)
    sup = None
    sw = sh = 0
    if isinstance(initial, str):
        if initial not in abi.INITIAL_KINDS:
            raise ValueError("initial must be 'mid-gray', 'black', or an array")
        kind = abi.INITIAL_KINDS[initial]
    else:
        sup = _u8_2d(initial)
        sh, sw = sup.shape
        kind = abi.INITIAL_SUPPLIED
    kw, kh = enc.width * max(scale, 0), enc.height * max(scale, 0)
    out = np.empty((max(kh, 1), max(kw, 1)), np.uint8)
    rm = np.zeros(max(iterations, 1), np.float64)
    runs = ctypes.c_int32(0)
    _check(lib().fic_decode(ptr(maps), enc.width, enc.height, ctypes.byref(enc.params.struct), int(scale),
                            int(iterations), kind, ptr(sup), sw, sh, int(convergence_eps is not None),
                            float(convergence_eps or 0.0), ptr(out), ptr(rm), ctypes.byref(runs)))
    return out, rm[: runs.value].copy(), runs.value


def decode(enc, scale=1, iterations=16, initial="mid-gray", convergence_eps=None):
    """Iterative decode at an integer magnification (module.cpp:109-140)."""
    return decode_traced(enc, scale, iterations, initial, convergence_eps)[0]


def decode_step(raster, enc, scale=1):
    """(extension) one application of the stored transform to an fp64 raster (decoder.cpp:39-79)."""
    cur = np.ascontiguousarray(raster, np.float64)
    if cur.ndim != 2:
        raise ValueError("expected a 2D float64 raster")
    nxt = np.empty_like(cur)
    maps = _maps(enc)
    _check(lib().fic_decode_step(ptr(cur), cur.shape[1], cur.shape[0], ptr(maps), enc.width, enc.height,
                                 ctypes.byref(enc.params.struct), int(scale), ptr(nxt)))
    return nxt


def collage_error(image, enc):
    """RMSE between the image and one application of the stored transform (decoder.cpp:134-140)."""
    img = _u8_2d(image)
    maps = _maps(enc)
    out = ctypes.c_double()
    _check(lib().fic_collage_error(ptr(img), img.shape[1], img.shape[0], ptr(maps), enc.width, enc.height,
                                   ctypes.byref(enc.params.struct), ctypes.byref(out)))
    return out.value


def decoded_error_bound(collage_rmse, s_max):
    """collage_rmse / (1 - s_max); NonContractive when s_max >= 1 (decoder.cpp:142-146)."""
    out = ctypes.c_double()
    _check(lib().fic_decoded_error_bound(float(collage_rmse), float(s_max), ctypes.byref(out)))
    return out.value


def validate_geometry(image, params=None):
    """validate_geometry (proj/src/image.cpp:138-149)."""
    params = CodecParams() if params is None else params
    img = _u8_2d(image)
    _check(lib().fic_validate_geometry(img.shape[1], img.shape[0], ctypes.byref(params.struct)))


def rmse(a, b):
    """Integer-exact SSE -> RMSE (proj/src/metrics.cpp:8-17).  Host utility."""
    a, b = _u8_2d(a), _u8_2d(b)
    if a.shape != b.shape:
        raise CodecError(abi.ERRC_NAMES.index("DimensionMismatch") + 1, "image geometry differs")
    d = a.astype(np.int64) - b.astype(np.int64)
    return float(np.sqrt(float(np.sum(d * d)) / float(a.size)))


def psnr(a, b):
    """20*log10(255/rmse); inf for identical images (proj/src/metrics.cpp:19-23)."""
    e = rmse(a, b)
    if e == 0.0:
        return float("inf")
    return float(20.0 * np.log10(255.0 / e))


# ---------------------------------------------------------------- per-candidate fit pipeline
class LinearFit:
    """LinearFit (proj/include/fic/encoder.hpp:15-19)."""

    __slots__ = ("s", "o", "residual")

    def __init__(self, s=0.0, o=0.0, residual=0.0):
        self.s, self.o, self.residual = float(s), float(o), float(residual)

    def __repr__(self):
        return f"LinearFit(s={self.s!r}, o={self.o!r}, residual={self.residual!r})"


class QuantizedFit:
    """QuantizedFit (proj/include/fic/encoder.hpp:24-30)."""

    __slots__ = ("qs", "qo", "s", "o", "residual")

    def __init__(self, qs=0, qo=0, s=0.0, o=0.0, residual=0.0):
        self.qs, self.qo = int(qs), int(qo)
        self.s, self.o, self.residual = float(s), float(o), float(residual)

    def __repr__(self):
        return f"QuantizedFit(qs={self.qs}, qo={self.qo}, s={self.s!r}, o={self.o!r}, residual={self.residual!r})"


def _block(samples):
    """A fic::Block (proj/include/fic/transforms.hpp:13-25): a square 2-D array of samples."""
    b = np.ascontiguousarray(np.asarray(samples, dtype=np.float64))
    if b.ndim != 2 or b.shape[0] != b.shape[1]:
        raise ValueError("expected a square 2D block of samples (side x side)")
    return b, int(b.shape[0])


def is_shadow(block, eps=0.0):
    """is_shadow (proj/src/encoder.cpp:60-67): N*sum(b^2) - sum(b)^2 <= eps."""
    b, side = _block(block)
    out = ctypes.c_int32()
    _check(lib().fic_is_shadow(ptr(b), side, float(eps), ctypes.byref(out)))
    return bool(out.value)


def least_squares_fit(a, b, shadow_eps=0.0):
    """least_squares_fit (proj/src/encoder.cpp:69-76): unconstrained fit of b ~ s*a + o."""
    (a, sa), (b, sb) = _block(a), _block(b)
    f = abi.FicLinearFit()
    _check(lib().fic_least_squares_fit(ptr(a), sa, ptr(b), sb, float(shadow_eps), ctypes.byref(f)))
    return LinearFit(f.s, f.o, f.residual)


def least_squares_clamped(a, b, params=None):
    """least_squares_clamped (proj/src/encoder.cpp:78-88): s clamped, o re-fitted and clamped."""
    params = CodecParams() if params is None else params
    (a, sa), (b, sb) = _block(a), _block(b)
    f = abi.FicLinearFit()
    _check(lib().fic_least_squares_clamped(ptr(a), sa, ptr(b), sb, ctypes.byref(params.struct), ctypes.byref(f)))
    return LinearFit(f.s, f.o, f.residual)


def least_squares(a, b, params=None):
    """least_squares (proj/src/encoder.cpp:90-102): clamped fit through the quantisers."""
    params = CodecParams() if params is None else params
    (a, sa), (b, sb) = _block(a), _block(b)
    f = abi.FicQuantizedFit()
    _check(lib().fic_least_squares(ptr(a), sa, ptr(b), sb, ctypes.byref(params.struct), ctypes.byref(f)))
    return QuantizedFit(f.qs, f.qo, f.s, f.o, f.residual)


def debug_pool(image, params=None, probes=None, want_q8=True):
    """(test support) K1 read-back (C-ABI fic_debug_pool): the device pool's exact moments
    {sq, den (-1 = flat)}, its u16 cells per isometry q8[d, s, i] = q[perm_s(i)], the flat
    count and, for `probes` = (ranges, domains, syms) index arrays, the survivor evaluation's
    exact correlations sum_i q8[d, s, i] * b_i."""
    params = CodecParams() if params is None else params
    img = _u8_2d(image)
    h, w = img.shape
    p = params
    D = (((w - 2 * p.n) // p.step + 1) ** 2) if w >= 2 * p.n else 0
    sq = np.zeros(max(D, 1), np.int64)
    den = np.zeros(max(D, 1), np.int64)
    q8 = np.zeros((max(D, 1), 8, p.n * p.n), np.uint16) if want_q8 else None
    flat = ctypes.c_uint64()
    if probes is not None:
        rr, dd, ss = (np.ascontiguousarray(x, np.int32) for x in probes)
        corr = np.zeros(len(rr), np.int64)
        args = (len(rr), ptr(rr), ptr(dd), ptr(ss), ptr(corr))
    else:
        corr = None
        args = (0, None, None, None, None)
    _check(lib().fic_debug_pool(ptr(img), w, h, ctypes.byref(p.struct), ptr(sq), ptr(den), ptr(q8),
                                ctypes.byref(flat), *args))
    return {"sq": sq[:D], "den": den[:D], "q8": q8[:D] if want_q8 else None, "flat_count": int(flat.value),
            "corr": corr}


def set_device(device):
    """(extension) select the CUDA device for this thread's codec calls."""
    _check(lib().fic_set_device(int(device)))


def encode_device(d_image_ptr, width, height, d_out_ptr, params=None, stream=0, stats=False):
    """(extension) device-resident encode: raw device pointers (e.g. torch tensor data_ptr())
    of a uint8 image and a (width/n)^2 x 32-byte record buffer, enqueued on `stream`
    (a cudaStream_t handle as int).  Returns stats when `stats` (synchronises)."""
    params = CodecParams() if params is None else params
    st = FicStats()
    _check(lib().fic_encode_device(ctypes.c_void_p(d_image_ptr), int(width), int(height),
                                   ctypes.byref(params.struct), ctypes.c_void_p(d_out_ptr),
                                   ctypes.byref(st) if stats else None, ctypes.c_void_p(stream)))
    return st.as_dict() if stats else None


def encode_rows_device(d_image_ptr, width, height, row_begin, row_end, d_out_ptr, params=None, stream=0):
    """(extension) device-resident range-row shard: rows [row_begin, row_end) of the range grid
    of a device image into (row_end - row_begin) * (width/n) device records (the multi-GPU
    split of one image).  Synchronises `stream`; returns the shard's stats."""
    params = CodecParams() if params is None else params
    st = FicStats()
    _check(lib().fic_encode_rows_device(ctypes.c_void_p(d_image_ptr), int(width), int(height),
                                        ctypes.byref(params.struct), int(row_begin), int(row_end),
                                        ctypes.c_void_p(d_out_ptr), ctypes.byref(st), ctypes.c_void_p(stream)))
    return st.as_dict()


def encode_batch_device(d_images_ptr, count, width, height, d_out_ptr, params=None, stream=0):
    """(extension) device-resident volume encode: `count` uint8 slices back to back at
    `d_images_ptr`, count x (width/n)^2 records at `d_out_ptr`; up to 64 slices per encode
    pass.  Synchronises `stream`; returns the summed stats."""
    params = CodecParams() if params is None else params
    st = FicStats()
    _check(lib().fic_encode_batch_device(ctypes.c_void_p(d_images_ptr), int(count), int(width), int(height),
                                         ctypes.byref(params.struct), ctypes.c_void_p(d_out_ptr),
                                         ctypes.byref(st), ctypes.c_void_p(stream)))
    return st.as_dict()


def kernel_launch_count():
    """(extension) number of this library's kernels launched so far."""
    return int(lib().fic_kernel_launch_count())


def matcher_timing(reset=False):
    """(extension) (average matcher ms, timed launches) since the last reset."""
    ms = ctypes.c_double()
    n = ctypes.c_uint64()
    lib().fic_matcher_timing(ctypes.byref(ms), ctypes.byref(n), int(reset))
    return ms.value, n.value


def set_matcher_timing(enabled):
    lib().fic_set_matcher_timing(int(bool(enabled)))


def scan_timing(reset=False):
    """(extension) (average ms of the full-level tcgen05 scan kernel, timed launches)."""
    ms = ctypes.c_double()
    n = ctypes.c_uint64()
    lib().fic_scan_timing(ctypes.byref(ms), ctypes.byref(n), int(reset))
    return ms.value, n.value


def scan_expand_timing(reset=False):
    """(extension) (average ms of the full-level scan kernel + its expand_kernel, timed launches)."""
    ms = ctypes.c_double()
    n = ctypes.c_uint64()
    lib().fic_scan_expand_timing(ctypes.byref(ms), ctypes.byref(n), int(reset))
    return ms.value, n.value


def decode_timing(reset=False):
    """(extension) (average ms, average algorithmic bytes, timed calls) of the decode iterations."""
    ms = ctypes.c_double()
    by = ctypes.c_double()
    n = ctypes.c_uint64()
    lib().fic_decode_timing(ctypes.byref(ms), ctypes.byref(by), ctypes.byref(n), int(reset))
    return ms.value, by.value, n.value


def pool_timing(reset=False):
    """(extension) (average ms, average algorithmic bytes, timed launches) of the K1 pool builder."""
    ms = ctypes.c_double()
    by = ctypes.c_double()
    n = ctypes.c_uint64()
    lib().fic_pool_timing(ctypes.byref(ms), ctypes.byref(by), ctypes.byref(n), int(reset))
    return ms.value, by.value, n.value


def last_survivors():
    """(extension) survivors per scan level of this process's last tcgen05-path encode."""
    buf = (ctypes.c_uint64 * 8)()
    n = lib().fic_last_survivors(buf, 8)
    return [int(buf[i]) for i in range(min(n, 8))]
