"""PGM I/O (proj/src/image.cpp:21-121): P5/P2, maxval 255, '#' comments.  Host utility,
outside the accelerated path; kept so callers of fic.load_pgm / fic.write_pgm switch over.
"""
import numpy as np

from . import abi

_WS = b" \t\n\r\x0b\x0c"


def _err(name, detail):
    from .codec import CodecError
    return CodecError(abi.ERRC_NAMES.index(name) + 1, detail)


class _Scanner:
    def __init__(self, data):
        self.b = data
        self.pos = 0

    def _skip(self):
        b = self.b
        while self.pos < len(b):
            c = b[self.pos:self.pos + 1]
            if c in _WS and c != b"":
                self.pos += 1
            elif c == b"#":
                while self.pos < len(b) and b[self.pos:self.pos + 1] != b"\n":
                    self.pos += 1
            else:
                break

    def token(self):
        self._skip()
        start = self.pos
        while self.pos < len(self.b) and self.b[self.pos:self.pos + 1] not in _WS:
            self.pos += 1
        return self.b[start:self.pos].decode("latin-1")


def _int(tok, what):
    if not tok:
        raise _err("MalformedHeader", f"missing {what}")
    if not tok.isdigit() or not tok.isascii():
        raise _err("MalformedHeader", f"non-numeric {what} '{tok}'")
    v = int(tok)
    if v > 2**31 - 1:
        raise _err("MalformedHeader", f"{what} out of range")
    return v


def load_pgm(data):
    b = bytes(data)
    s = _Scanner(b)
    magic = s.token()
    binary = magic == "P5"
    if not binary and magic != "P2":
        raise _err("MalformedHeader", f"magic '{magic}' is not P5/P2")
    w = _int(s.token(), "width")
    h = _int(s.token(), "height")
    if w <= 0 or h <= 0:
        raise _err("MalformedHeader", "zero-sized image")
    maxval = _int(s.token(), "maxval")
    if maxval != 255:
        raise _err("UnsupportedMaxval", f"maxval {maxval} != 255")
    count = w * h
    if binary:
        if s.pos >= len(b) or b[s.pos:s.pos + 1] not in _WS:
            raise _err("MalformedHeader", "missing separator before raster")
        s.pos += 1
        if len(b) - s.pos < count:
            raise _err("TruncatedData", f"{len(b) - s.pos} raster bytes, need {count}")
        return np.frombuffer(b, np.uint8, count=count, offset=s.pos).reshape(h, w).copy()
    out = np.empty(count, np.uint8)
    for i in range(count):
        tok = s.token()
        if not tok:
            raise _err("TruncatedData", f"{i} samples, need {count}")
        v = _int(tok, "sample")
        if v > maxval:
            raise _err("MalformedHeader", f"sample {v} exceeds maxval")
        out[i] = v
    return out.reshape(h, w)


def write_pgm(image):
    img = np.ascontiguousarray(np.asarray(image), np.uint8)
    if img.ndim != 2:
        raise ValueError("expected a 2D uint8 array (height x width)")
    h, w = img.shape
    return f"P5\n{w} {h}\n255\n".encode() + img.tobytes()
