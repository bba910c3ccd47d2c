"""TEST INFRASTRUCTURE ONLY — ctypes access to the parity checkers.

* `Oracle`    : the C restatement in oracle/fic_oracle.c (oracle/_build/libfic_oracle.so)
* `Reference` : the unmodified reference library compiled from /root/reference/proj
                (oracle/_ref/libfic_ref.so, recipe in oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may
import this package; the product package never does.
"""
import ctypes
import os
import subprocess

import numpy as np

from paper_1404_0774_b200.abi import (
    MAPPING_DTYPE, FicParams, FicStats, errc_name, make_params, ptr,
)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libfic_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfic_ref.so")
REF_SRC = "/root/reference/proj"


def build(force=False):
    """Compile the C restatement, and the reference library when its sources exist here."""
    targets = ["oracle"]
    if os.path.isdir(REF_SRC):
        targets.append("ref")
    if force:
        subprocess.check_call(["make", "-C", HERE, "clean"])
    subprocess.check_call(["make", "-C", HERE, "-j8"] + targets)


class OracleError(RuntimeError):
    pass


def _check(rc, lib_err=None):
    if rc != 0:
        detail = lib_err() if lib_err else ""
        raise OracleError(f"{errc_name(rc)}: {detail}")


def _params(p):
    if isinstance(p, FicParams):
        return p
    if isinstance(p, dict):
        return make_params(**p)
    return make_params(p.n, p.step, p.s_bits, p.o_bits, p.s_max, p.shadow_eps)


class Oracle:
    """The C restatement (oracle/fic_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        self.L = L
        vp, i32, u32, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double
        L.oracle_mt19937.argtypes = [u32, ctypes.c_int64, vp]
        L.oracle_noise_image.argtypes = [i32, u32, vp]
        L.oracle_smooth_image.argtypes = [i32, u32, vp]
        L.oracle_normalize_params.argtypes = [vp, vp]
        L.oracle_validate_geometry.argtypes = [i32, i32, vp]
        L.oracle_quantize.argtypes = [f64, f64, i32]
        L.oracle_quantize.restype = u32
        L.oracle_dequantize.argtypes = [u32, f64, i32]
        L.oracle_dequantize.restype = f64
        L.oracle_domain_count.argtypes = [i32, vp]
        L.oracle_domain_count.restype = ctypes.c_int64
        L.oracle_domain_pool.argtypes = [vp, i32, vp, vp, vp, vp, vp]
        L.oracle_encode.argtypes = [vp, i32, i32, vp, i32, vp, vp]
        L.oracle_encode_ranges.argtypes = [vp, i32, i32, vp, i32, vp, vp, vp, vp]
        L.oracle_decode_step.argtypes = [vp, vp, i32, vp, i32, vp]
        L.oracle_decode.argtypes = [vp, i32, vp, i32, i32, i32, vp, i32, f64, vp, vp, vp]
        L.oracle_collage_error.argtypes = [vp, vp, i32, vp, vp]
        L.oracle_rmse.argtypes = [vp, vp, ctypes.c_int64]
        L.oracle_rmse.restype = f64
        L.oracle_psnr.argtypes = [vp, vp, ctypes.c_int64]
        L.oracle_psnr.restype = f64
        L.oracle_raster_rmse.argtypes = [vp, vp, ctypes.c_int64]
        L.oracle_raster_rmse.restype = f64

    # fixtures
    def mt19937(self, seed, count):
        out = np.empty(count, np.uint32)
        self.L.oracle_mt19937(seed, count, ptr(out))
        return out

    def noise_image(self, side, seed):
        out = np.empty((side, side), np.uint8)
        self.L.oracle_noise_image(side, seed, ptr(out))
        return out

    def smooth_image(self, side, seed):
        out = np.empty((side, side), np.uint8)
        self.L.oracle_smooth_image(side, seed, ptr(out))
        return out

    # params / quantiser
    def normalize(self, params):
        p, out = _params(params), FicParams()
        _check(self.L.oracle_normalize_params(ctypes.byref(p), ctypes.byref(out)))
        return out

    def validate_geometry(self, w, h, params):
        p = self.normalize(params)
        return self.L.oracle_validate_geometry(w, h, ctypes.byref(p))

    def quantize(self, v, maxv, bits):
        return int(self.L.oracle_quantize(v, maxv, bits))

    def dequantize(self, code, maxv, bits):
        return float(self.L.oracle_dequantize(code, maxv, bits))

    # domain pool (integer moments)
    def domain_pool(self, img, params):
        p = self.normalize(params)
        img = np.ascontiguousarray(img, np.uint8)
        w = img.shape[1]
        D = int(self.L.oracle_domain_count(w, ctypes.byref(p)))
        N = p.n * p.n
        q = np.empty((D, N), np.int16)
        sq = np.empty(D, np.int64)
        sqq = np.empty(D, np.int64)
        flat = np.empty(D, np.uint8)
        self.L.oracle_domain_pool(ptr(img), w, ctypes.byref(p), ptr(q), ptr(sq), ptr(sqq), ptr(flat))
        return q, sq, sqq, flat.astype(bool)

    # encoder
    def encode(self, img, params, brute=False):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        p = _params(params)
        pn = self.normalize(p) if w == h and w > 0 else p
        n = pn.n if pn.n > 0 else 1
        out = np.zeros(max((w // n) * (h // n), 1), MAPPING_DTYPE)
        st = FicStats()
        _check(self.L.oracle_encode(ptr(img), w, h, ctypes.byref(p), int(brute), ptr(out), ctypes.byref(st)))
        return out[: (w // n) * (h // n)], st.as_dict()

    def encode_ranges(self, img, params, xs, ys):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        xs = np.ascontiguousarray(xs, np.int32)
        ys = np.ascontiguousarray(ys, np.int32)
        out = np.zeros(len(xs), MAPPING_DTYPE)
        st = FicStats()
        _check(self.L.oracle_encode_ranges(ptr(img), w, h, ctypes.byref(_params(params)), len(xs), ptr(xs),
                                           ptr(ys), ptr(out), ctypes.byref(st)))
        return out, st.as_dict()

    def encode_threaded(self, img, params, threads=None, rows=None):
        """Same records as encode() (one range at a time, reference order within each range),
        spread over host threads by range rows; `rows` restricts to a subset of range rows."""
        from concurrent.futures import ThreadPoolExecutor
        img = np.ascontiguousarray(img, np.uint8)
        p = self.normalize(params)
        R = img.shape[1] // p.n
        rows = list(range(R)) if rows is None else list(rows)
        threads = threads or os.cpu_count() or 1

        def work(row):
            xs = np.arange(R, dtype=np.int32) * p.n
            ys = np.full(R, row * p.n, np.int32)
            return self.encode_ranges(img, p, xs, ys)

        with ThreadPoolExecutor(threads) as ex:
            parts = list(ex.map(work, rows))
        out = np.concatenate([m for m, _ in parts]) if parts else np.zeros(0, MAPPING_DTYPE)
        st = {k: sum(s[k] for _, s in parts) for k in ("candidates_tested", "shadow_ranges", "shadow_codeblocks")}
        return out, st

    # decoder
    def decode_step(self, cur, maps, width, params, scale=1):
        cur = np.ascontiguousarray(cur, np.float64)
        nxt = np.empty_like(cur)
        maps = np.ascontiguousarray(maps, MAPPING_DTYPE)
        _check(self.L.oracle_decode_step(ptr(cur), ptr(maps), width, ctypes.byref(_params(params)), scale,
                                         ptr(nxt)))
        return nxt

    def decode(self, maps, width, params, scale=1, iterations=16, initial="mid-gray", convergence_eps=None):
        maps = np.ascontiguousarray(maps, MAPPING_DTYPE)
        kw = width * scale
        out = np.empty((kw, kw), np.uint8)
        rm = np.zeros(max(iterations, 1), np.float64)
        runs = ctypes.c_int32(0)
        sup = None
        if isinstance(initial, str):
            kind = {"mid-gray": 0, "black": 1}[initial]
        else:
            kind = 2
            sup = np.ascontiguousarray(initial, np.uint8)
        _check(self.L.oracle_decode(ptr(maps), width, ctypes.byref(_params(params)), scale, iterations, kind,
                                    ptr(sup), int(convergence_eps is not None),
                                    float(convergence_eps or 0.0), ptr(out), ptr(rm), ctypes.byref(runs)))
        return out, rm[: runs.value].copy(), runs.value

    def collage_error(self, img, maps, params):
        img = np.ascontiguousarray(img, np.uint8)
        maps = np.ascontiguousarray(maps, MAPPING_DTYPE)
        out = ctypes.c_double()
        _check(self.L.oracle_collage_error(ptr(img), ptr(maps), img.shape[1], ctypes.byref(_params(params)),
                                           ctypes.byref(out)))
        return out.value

    def rmse(self, a, b):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        return float(self.L.oracle_rmse(ptr(a), ptr(b), a.size))

    def psnr(self, a, b):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        return float(self.L.oracle_psnr(ptr(a), ptr(b), a.size))


class Reference:
    """The unmodified reference library (oracle/_ref/libfic_ref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise OracleError(f"reference library not built: {path}")
        L = ctypes.CDLL(path)
        self.L = L
        vp, i32, u32, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_hardware_concurrency.restype = i32
        L.ref_encode.argtypes = [vp, i32, i32, vp, i32, i32, i32, vp, vp]
        L.ref_encode_range.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp]
        L.ref_oracle_encode.argtypes = [vp, i32, i32, vp, vp]
        L.ref_decode_step.argtypes = [vp, vp, i32, i32, vp, i32, vp]
        L.ref_decode.argtypes = [vp, i32, i32, vp, i32, i32, i32, vp, i32, f64, vp, vp, vp]
        L.ref_collage_error.argtypes = [vp, vp, i32, i32, vp, vp]
        L.ref_serialize.argtypes = [vp, i32, i32, vp, vp, ctypes.c_int64]
        L.ref_serialize.restype = ctypes.c_int64
        L.ref_noise_image.argtypes = [i32, u32, vp]
        L.ref_smooth_image.argtypes = [i32, u32, vp]
        L.ref_psnr.argtypes = [vp, vp, i32, i32]
        L.ref_psnr.restype = f64
        L.ref_least_squares.argtypes = [i32, vp, i32, vp, i32, vp, f64, vp]
        L.ref_is_shadow.argtypes = [vp, i32, f64]

    def _err(self):
        return self.L.ref_last_error().decode()

    @property
    def hardware_concurrency(self):
        return int(self.L.ref_hardware_concurrency())

    def noise_image(self, side, seed):
        out = np.empty((side, side), np.uint8)
        self.L.ref_noise_image(side, seed, ptr(out))
        return out

    def smooth_image(self, side, seed):
        out = np.empty((side, side), np.uint8)
        self.L.ref_smooth_image(side, seed, ptr(out))
        return out

    def encode(self, img, params, workers=1, chunk=(16, 16)):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        p = _params(params)
        n = p.n if p.n > 0 else 1
        out = np.zeros(max((w // n) * (h // n), 1), MAPPING_DTYPE)
        st = FicStats()
        _check(self.L.ref_encode(ptr(img), w, h, ctypes.byref(p), workers, chunk[0], chunk[1], ptr(out),
                                 ctypes.byref(st)), self._err)
        return out[: (w // n) * (h // n)], st.as_dict()

    def encode_range(self, img, x, y, params):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.zeros(1, MAPPING_DTYPE)
        st = FicStats()
        _check(self.L.ref_encode_range(ptr(img), img.shape[1], img.shape[0], x, y, ctypes.byref(_params(params)),
                                       ptr(out), ctypes.byref(st)), self._err)
        return out[0], st.as_dict()

    def oracle_encode(self, img, params):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        p = _params(params)
        out = np.zeros((w // p.n) * (h // p.n), MAPPING_DTYPE)
        _check(self.L.ref_oracle_encode(ptr(img), w, h, ctypes.byref(p), ptr(out)), self._err)
        return out

    def decode_step(self, cur, maps, width, params, scale=1, height=None):
        cur = np.ascontiguousarray(cur, np.float64)
        nxt = np.empty_like(cur)
        maps = np.ascontiguousarray(maps, MAPPING_DTYPE)
        height = width if height is None else height
        _check(self.L.ref_decode_step(ptr(cur), ptr(maps), width, height, ctypes.byref(_params(params)), scale,
                                      ptr(nxt)), self._err)
        return nxt

    def decode(self, maps, width, params, scale=1, iterations=16, initial="mid-gray", convergence_eps=None,
               height=None):
        maps = np.ascontiguousarray(maps, MAPPING_DTYPE)
        height = width if height is None else height
        out = np.empty((height * scale, width * scale), np.uint8)
        rm = np.zeros(max(iterations, 1), np.float64)
        runs = ctypes.c_int32(0)
        sup = None
        if isinstance(initial, str):
            kind = {"mid-gray": 0, "black": 1}[initial]
        else:
            kind = 2
            sup = np.ascontiguousarray(initial, np.uint8)
        _check(self.L.ref_decode(ptr(maps), width, height, ctypes.byref(_params(params)), scale, iterations, kind,
                                 ptr(sup), int(convergence_eps is not None), float(convergence_eps or 0.0),
                                 ptr(out), ptr(rm), ctypes.byref(runs)), self._err)
        return out, rm[: runs.value].copy(), runs.value

    def collage_error(self, img, maps, params):
        img = np.ascontiguousarray(img, np.uint8)
        maps = np.ascontiguousarray(maps, MAPPING_DTYPE)
        out = ctypes.c_double()
        _check(self.L.ref_collage_error(ptr(img), ptr(maps), img.shape[1], img.shape[0],
                                        ctypes.byref(_params(params)), ctypes.byref(out)), self._err)
        return out.value

    def serialize(self, maps, width, params):
        maps = np.ascontiguousarray(maps, MAPPING_DTYPE)
        p = _params(params)
        n = self.L.ref_serialize(ptr(maps), width, width, ctypes.byref(p), None, 0)
        if n < 0:
            _check(int(-n), self._err)
        buf = np.empty(n, np.uint8)
        self.L.ref_serialize(ptr(maps), width, width, ctypes.byref(p), ptr(buf), n)
        return buf.tobytes()

    def psnr(self, a, b):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        return float(self.L.ref_psnr(ptr(a), ptr(b), a.shape[1], a.shape[0]))

    def least_squares(self, kind, a, b, params=None, shadow_eps=0.0):
        """kind: 'fit' | 'clamped' | 'quantized' -> (s, o, residual, qs, qo)."""
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros(5, np.float64)
        k = {"fit": 0, "clamped": 1, "quantized": 2}[kind]
        p = _params(params if params is not None else {})
        _check(self.L.ref_least_squares(k, ptr(a), a.shape[0], ptr(b), b.shape[0], ctypes.byref(p),
                                        float(shadow_eps), ptr(out)), self._err)
        return float(out[0]), float(out[1]), float(out[2]), int(out[3]), int(out[4])

    def is_shadow(self, b, eps=0.0):
        b = np.ascontiguousarray(b, np.float64)
        return bool(self.L.ref_is_shadow(ptr(b), b.shape[0], float(eps)))
