"""GPU parity of the iterated decoder (K3) against the oracle.

Every fp64 raster value is computed in the reference's operation order, so rasters
and the final uint8 image are bit-exact; step RMSE uses a fixed-order tree reduction
instead of the reference's sequential sum, so it is checked to 1e-12 relative.
"""
import numpy as np
import pytest

import paper_1404_0774_b200 as fic
from paper_1404_0774_b200 import images

pytestmark = pytest.mark.gpu


def _enc(oracle, img, **pv):
    maps, _ = oracle.encode(img, pv)
    return fic.EncodedImage(img.shape[1], img.shape[0], fic.CodecParams(**pv), maps)


@pytest.mark.parametrize("scale", [1, 2, 3])
def test_decode_step_bit_exact(oracle, scale):
    img = oracle.smooth_image(32, 61)
    enc = _enc(oracle, img, s_max=0.9)
    rng = np.random.default_rng(5)
    cur = rng.uniform(-20, 300, size=(32 * scale, 32 * scale))
    got = fic.decode_step(cur, enc, scale)
    want = oracle.decode_step(cur, enc.mappings, 32, dict(s_max=0.9), scale)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("initial", ["mid-gray", "black", "supplied"])
@pytest.mark.parametrize("scale", [1, 2])
def test_decode_bit_exact(oracle, initial, scale):
    img = oracle.smooth_image(64, 64)
    enc = _enc(oracle, img, n=4, step=2)
    init = initial
    if initial == "supplied":
        init = oracle.noise_image(64 * scale, 9)
    out, rm, runs = fic.decode_traced(enc, scale=scale, iterations=10, initial=init)
    wout, wrm, wruns = oracle.decode(enc.mappings, 64, dict(n=4, step=2), scale, 10, init)
    assert np.array_equal(out, wout)
    assert runs == wruns == 10
    np.testing.assert_allclose(rm, wrm, rtol=1e-12, atol=1e-300)


def test_cfg1_decode_psnr(oracle):
    img = images.phantom(256, 1404001)
    pv = dict(n=8, step=8)
    enc = fic.encode(img, fic.CodecParams(**pv))
    out = fic.decode(enc, iterations=10)
    wmaps, _ = oracle.encode_threaded(img, pv)
    wout, _, _ = oracle.decode(wmaps, 256, pv, 1, 10)
    assert np.array_equal(out, wout)
    assert abs(fic.psnr(img, out) - oracle.psnr(img, wout)) < 0.01


def test_early_stop_and_constants(oracle):
    # test_decoder.cpp:90-98: one step reaches the fixed point, the second proves it
    img = np.full((16, 16), 200, np.uint8)
    enc = fic.encode(img)
    _, rm, runs = fic.decode_traced(enc, convergence_eps=1e-12)
    assert runs == 2
    # representable constants decode exactly in one iteration (test_decoder.cpp:27-35)
    for v in (0, 255):
        img = np.full((16, 16), v, np.uint8)
        assert np.array_equal(fic.decode(fic.encode(img), iterations=1), img)


def test_collage_error(oracle):
    img = oracle.noise_image(16, 65)
    enc = fic.encode(img)
    expected = np.sqrt(np.sum(enc.mappings["residual"]) / img.size)
    ce = fic.collage_error(img, enc)
    assert ce == pytest.approx(expected, rel=1e-6)
    assert ce == pytest.approx(oracle.collage_error(img, enc.mappings, {}), rel=1e-12)


def test_monotone_step_rmse(oracle):
    img = oracle.smooth_image(32, 64)
    enc = fic.encode(img, fic.CodecParams(s_max=0.9))
    _, rm, runs = fic.decode_traced(enc)
    assert runs == 16
    assert all(rm[t + 1] <= rm[t] + 1e-9 for t in range(1, len(rm) - 1))


def test_decode_errors():
    img = np.zeros((16, 16), np.uint8)
    img[::2] = 255
    enc = fic.encode(img)
    with pytest.raises(fic.CodecError, match="BadParams"):
        fic.decode(enc, scale=0)
    with pytest.raises(fic.CodecError, match="BadParams"):
        fic.decode(enc, iterations=0)
    with pytest.raises(fic.CodecError, match="ScaleMismatch"):
        fic.decode(enc, initial=np.zeros((8, 8), np.uint8))
    with pytest.raises(fic.CodecError, match="DimensionMismatch"):
        fic.collage_error(np.zeros((32, 32), np.uint8), enc)
    with pytest.raises(fic.CodecError, match="NonContractive"):
        fic.decoded_error_bound(1.0, 1.0)


def _random_maps(W, n, step, seed):
    """Random but valid code records (every isometry, codes across their range)."""
    from paper_1404_0774_b200.abi import MAPPING_DTYPE
    rng = np.random.default_rng(seed)
    R = (W // n) ** 2
    P = (W - 2 * n) // step + 1
    m = np.zeros(R, MAPPING_DTYPE)
    m["x"] = rng.integers(0, P, R) * step
    m["y"] = rng.integers(0, P, R) * step
    m["sym"] = np.arange(R) % 8
    m["qs"] = rng.integers(0, 32, R)
    m["qo"] = rng.integers(0, 128, R)
    return m


# (image side, n, step, scale): kn = n * scale covers the tiled decoder (kn a multiple of 32,
# or a divisor of 32) and the per-pixel kernel (kn = 40, 24)
@pytest.mark.parametrize("W,n,step,scale", [(32, 8, 4, 4), (32, 8, 2, 8), (64, 4, 2, 16), (32, 2, 1, 1),
                                            (64, 8, 8, 1), (32, 8, 4, 5), (32, 8, 4, 3), (16, 4, 1, 8),
                                            (64, 4, 3, 1), (32, 4, 1, 2)])
def test_decode_step_tiled_geometries(oracle, W, n, step, scale):
    maps = _random_maps(W, n, step, W * 1000 + n * 10 + scale)
    pv = dict(n=n, step=step)
    enc = fic.EncodedImage(W, W, fic.CodecParams(**pv), maps)
    rng = np.random.default_rng(scale)
    cur = rng.uniform(-20, 300, size=(W * scale, W * scale))
    got = fic.decode_step(cur, enc, scale)
    want = oracle.decode_step(cur, maps, W, pv, scale)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    out, rm, runs = fic.decode_traced(enc, scale=scale, iterations=3, initial="mid-gray")
    wout, wrm, _ = oracle.decode(maps, W, pv, scale, 3)
    assert np.array_equal(out, wout)
    np.testing.assert_allclose(rm, wrm, rtol=1e-12, atol=1e-300)


def _random_maps_wh(rng, w, h, n, count, s_bits=5, o_bits=7, step=1):
    """Valid random mappings (every 2n-wide window inside the w x h image)."""
    from paper_1404_0774_b200.abi import MAPPING_DTYPE
    m = np.zeros(count, MAPPING_DTYPE)
    m["x"] = rng.integers(0, (w - 2 * n) // step + 1, count) * step
    m["y"] = rng.integers(0, (h - 2 * n) // step + 1, count) * step
    m["sym"] = rng.integers(0, 8, count)
    m["qs"] = rng.integers(0, 1 << s_bits, count)
    m["qo"] = rng.integers(0, 1 << o_bits, count)
    return m


@pytest.mark.parametrize("scale", [1, 2, 3])
def test_decode_off_grid_origins(oracle, scale):
    """Mappings edited off the encoder's step grid (odd x / y with an even step): the
    mean-raster decoder must not be used at odd magnifications (its 2x2 means sit on the
    even grid); every raster value stays bit-exact with the reference decoder."""
    img = oracle.smooth_image(64, 64)
    pv = dict(n=4, step=2)
    maps, _ = oracle.encode(img, pv)
    maps = maps.copy()
    rng = np.random.default_rng(77)
    idx = rng.choice(len(maps), 40, replace=False)
    maps["x"][idx] = np.minimum(maps["x"][idx] + 1, 64 - 8)
    maps["y"][idx[::2]] = np.minimum(maps["y"][idx[::2]] + 1, 64 - 8)
    assert np.any(maps["x"] % 2 == 1)
    enc = fic.EncodedImage(64, 64, fic.CodecParams(**pv), maps)
    out, rm, runs = fic.decode_traced(enc, scale=scale, iterations=6)
    wout, wrm, wruns = oracle.decode(maps, 64, pv, scale, 6)
    assert np.array_equal(out, wout)
    np.testing.assert_allclose(rm, wrm, rtol=1e-12, atol=1e-300)
    assert abs(fic.collage_error(img, enc) - oracle.collage_error(img, maps, pv)) <= 1e-12 * oracle.collage_error(
        img, maps, pv)


@pytest.mark.parametrize("w,h,n,scale", [(64, 32, 4, 1), (32, 64, 8, 2), (36, 20, 8, 1), (96, 64, 4, 3),
                                         (256, 128, 8, 1)])
def test_decode_non_square(w, h, n, scale):
    """decode / decode_step on non-square geometries (a deserialised FIC1 header may be
    non-square, format.cpp:145-185) and sides that are not multiples of n (pixels outside the
    range grid stay 0, decoder.cpp:56) against the compiled reference decoder."""
    import os
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    ref = Reference()
    rng = np.random.default_rng(w * 1000 + h)
    count = (w // n) * (h // n)
    maps = _random_maps_wh(rng, w, h, n, count)
    pv = dict(n=n, s_max=0.8)
    enc = fic.EncodedImage(w, h, fic.CodecParams(**pv), maps)
    out, rm, runs = fic.decode_traced(enc, scale=scale, iterations=5)
    wout, wrm, wruns = ref.decode(maps, w, pv, scale, 5, height=h)
    assert out.shape == (h * scale, w * scale)
    assert np.array_equal(out, wout)
    np.testing.assert_allclose(rm, wrm, rtol=1e-12, atol=1e-300)
    cur = rng.uniform(-10, 270, (h * scale, w * scale))
    got = fic.decode_step(cur, enc, scale)
    want = ref.decode_step(cur, maps, w, pv, scale, height=h)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
