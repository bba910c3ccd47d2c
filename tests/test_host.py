"""CPU: host-side pieces around the accelerated path — the FIC1 record layout (SURVEY §8 row F1,
proj/src/format.cpp:78-89; the packing itself runs on the device, tests/test_gpu_fic1.py), PGM I/O,
EncodedImage semantics, synthetic inputs."""
import numpy as np
import pytest

import paper_1404_0774_b200 as fic
from paper_1404_0774_b200 import images
from paper_1404_0774_b200.abi import MAPPING_DTYPE
from paper_1404_0774_b200.fic1 import record_layout


def gradient_image(side):
    y, x = np.mgrid[0:side, 0:side]
    return ((x * 3 + y * 2) // 4 % 256).astype(np.uint8)


def test_pgm_round_trip_and_errors():
    # test_smoke.py:14-21
    img = gradient_image(32)
    assert np.array_equal(fic.load_pgm(fic.write_pgm(img)), img)
    with pytest.raises(fic.CodecError, match="MalformedHeader"):
        fic.load_pgm(b"P6 1 1 255 x")
    with pytest.raises(fic.CodecError, match="UnsupportedMaxval"):
        fic.load_pgm(b"P5 1 1 65535\nxx")
    with pytest.raises(fic.CodecError, match="TruncatedData"):
        fic.load_pgm(b"P5 4 4 255\nabc")
    assert np.array_equal(fic.load_pgm(b"P2\n# c\n2 2\n255\n1 2\n3 4\n"), np.array([[1, 2], [3, 4]], np.uint8))


def test_fic1_record_width():
    # test_format.cpp:76-96: 27-bit records pad to 4 bytes (e.g. 256^2, n=4, step=4: 6+6+3+5+7)
    _, _, widths, nbytes = record_layout(256, 256, fic.CodecParams(n=4, step=4))
    assert sum(widths) == 27 and nbytes == 4
    px, py, widths, nbytes = record_layout(512, 512, fic.CodecParams(n=8, step=4))
    assert (px, py, widths, nbytes) == (125, 125, [7, 7, 3, 5, 7], 4)
    with pytest.raises(fic.CodecError, match="NoValidPositions"):
        record_layout(8, 8, fic.CodecParams(n=8))


def test_encoded_image_equality_ignores_residual():
    m = np.zeros(16, MAPPING_DTYPE)
    m["qo"] = np.arange(16)
    enc = fic.EncodedImage(16, 16, fic.CodecParams(), m)
    other = fic.EncodedImage(enc.width, enc.height, enc.params, enc.mappings.copy())
    other.mappings["residual"] += 1.0
    assert enc == other
    other.mappings["qo"][0] ^= 1
    assert enc != other


def test_synthetic_images_deterministic():
    for gen in (lambda: images.phantom(64, 1), lambda: images.ct_slice(64, 2), lambda: images.xray(64, 3)):
        a, b = gen(), gen()
        assert a.dtype == np.uint8 and a.shape == (64, 64)
        assert np.array_equal(a, b)
    vol = images.volume(3, 32, 1404005)
    assert vol.shape == (3, 32, 32) and not np.array_equal(vol[0], vol[1])


def test_metrics():
    # test_smoke.py:77-82
    a = np.full((16, 16), 100, dtype=np.uint8)
    b = np.full((16, 16), 101, dtype=np.uint8)
    assert fic.rmse(a, b) == 1.0
    assert fic.psnr(a, a) == float("inf")
