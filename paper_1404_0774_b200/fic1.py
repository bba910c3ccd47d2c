"""FIC1 container (proj/src/format.cpp:105-185): 20-byte little-endian header plus one
byte-aligned, MSB-first record per range.  Host-side packing of the gathered codes,
vectorised over records with numpy.
"""
import numpy as np

from . import abi
from .abi import MAPPING_DTYPE

MAGIC = b"FIC1"
HEADER_BYTES = 20


def _ceil_log2(count):  # format.cpp:35-37
    return 0 if count <= 1 else int(count - 1).bit_length()


def _per_axis(width, n, step):  # positions_per_axis (codebook.cpp:7-11)
    from .codec import CodecError
    if step < 1:
        raise CodecError(abi.ERRC_NAMES.index("BadParams") + 1, "step must be >= 1")
    if width < 2 * n:
        raise CodecError(abi.ERRC_NAMES.index("NoValidPositions") + 1, f"width {width} < 2n")
    return (width - 2 * n) // step + 1


def record_layout(width, height, p):
    px, py = _per_axis(width, p.n, p.step), _per_axis(height, p.n, p.step)
    fields = [_ceil_log2(px), _ceil_log2(py), 3, p.s_bits, p.o_bits]
    return px, py, fields, (sum(fields) + 7) // 8


def _pack_fields(values, widths):
    """MSB-first concatenation of fixed-width fields per record -> (count, bytes) uint8."""
    count = len(values[0])
    cols = []
    for v, w in zip(values, widths):
        if w == 0:
            continue
        shifts = np.arange(w - 1, -1, -1, dtype=np.uint64)
        cols.append(((v.astype(np.uint64)[:, None] >> shifts[None, :]) & np.uint64(1)).astype(np.uint8))
    bits = np.concatenate(cols, axis=1) if cols else np.zeros((count, 0), np.uint8)
    pad = (-bits.shape[1]) % 8
    if pad:
        bits = np.concatenate([bits, np.zeros((count, pad), np.uint8)], axis=1)
    return np.packbits(bits, axis=1)


def _unpack_fields(records, widths):
    bits = np.unpackbits(records, axis=1)
    out, pos = [], 0
    for w in widths:
        v = np.zeros(len(records), np.uint64)
        for i in range(w):
            v = (v << np.uint64(1)) | bits[:, pos + i].astype(np.uint64)
        out.append(v)
        pos += w
    return out


def serialize(enc):
    from .codec import CodecError
    p = enc.params
    px, py, widths, rec_bytes = record_layout(enc.width, enc.height, p)
    m = np.asarray(enc.mappings)
    if len(m) != (enc.width // p.n) * (enc.height // p.n):
        raise CodecError(abi.ERRC_NAMES.index("BadParams") + 1,
                         f"mapping count {len(m)} != range count {(enc.width // p.n) * (enc.height // p.n)}")
    x, y = m["x"].astype(np.int64), m["y"].astype(np.int64)
    if np.any(x % p.step) or np.any(y % p.step):
        raise CodecError(abi.ERRC_NAMES.index("OutOfRange") + 1, "domain position off the step grid")
    xi, yi = x // p.step, y // p.step
    if np.any(xi >= px) or np.any(yi >= py):
        raise CodecError(abi.ERRC_NAMES.index("OutOfRange") + 1, "domain index outside the grid")
    header = bytearray(MAGIC)
    header += int(enc.width).to_bytes(4, "little") + int(enc.height).to_bytes(4, "little")
    header += int(p.n).to_bytes(2, "little") + int(p.step).to_bytes(2, "little")
    header += bytes([p.s_bits & 0xFF, p.o_bits & 0xFF])
    header += int(round(p.s_max * 1000.0)).to_bytes(2, "little")
    if len(m) == 0:
        return bytes(header)
    recs = _pack_fields([xi, yi, m["sym"].astype(np.int64), m["qs"].astype(np.int64), m["qo"].astype(np.int64)],
                        widths)
    assert recs.shape[1] == rec_bytes
    return bytes(header) + recs.tobytes()


def deserialize(data):
    from .codec import CodecError, CodecParams, EncodedImage
    b = bytes(data)
    if len(b) < HEADER_BYTES:
        raise CodecError(abi.ERRC_NAMES.index("TruncatedData") + 1, "short header")
    if b[:4] != MAGIC:
        raise CodecError(abi.ERRC_NAMES.index("MalformedHeader") + 1, "bad magic")
    width = int.from_bytes(b[4:8], "little")
    height = int.from_bytes(b[8:12], "little")
    n = int.from_bytes(b[12:14], "little")
    step = int.from_bytes(b[14:16], "little")
    s_bits, o_bits = b[16], b[17]
    s_max = int.from_bytes(b[18:20], "little") / 1000.0
    p = CodecParams(n=n, step=step, s_bits=s_bits, o_bits=o_bits, s_max=s_max)
    if width <= 0 or height <= 0 or width % p.n or height % p.n:
        raise CodecError(abi.ERRC_NAMES.index("MalformedHeader") + 1, "dimensions incompatible with range size")
    px, py, widths, rec_bytes = record_layout(width, height, p)
    count = (width // p.n) * (height // p.n)
    body = count * rec_bytes
    if len(b) - HEADER_BYTES < body:
        raise CodecError(abi.ERRC_NAMES.index("TruncatedData") + 1,
                         f"{len(b) - HEADER_BYTES} body bytes, need {body}")
    recs = np.frombuffer(b, np.uint8, count=body, offset=HEADER_BYTES).reshape(count, rec_bytes)
    xi, yi, sym, qs, qo = _unpack_fields(recs, widths)
    bad = np.nonzero((xi >= px) | (yi >= py))[0]
    if len(bad):
        raise CodecError(abi.ERRC_NAMES.index("OutOfRange") + 1,
                         f"domain index outside the grid in record {int(bad[0])}")
    m = np.zeros(count, MAPPING_DTYPE)
    m["x"] = (xi * p.step).astype(np.int32)
    m["y"] = (yi * p.step).astype(np.int32)
    m["sym"] = sym.astype(np.int32)
    m["qs"] = qs.astype(np.uint32)
    m["qo"] = qo.astype(np.uint32)
    return EncodedImage(width, height, p, m)
