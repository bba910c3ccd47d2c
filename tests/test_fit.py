"""The public per-candidate fit pipeline through the C-ABI:
fic_is_shadow / fic_least_squares_fit / fic_least_squares_clamped / fic_least_squares
(proj/src/encoder.cpp:60-102).  Host fp64, so these run without a GPU.

* the reference's own worked examples (proj/tests/test_encoder.cpp:15-60),
* bit-exact agreement with the compiled reference (oracle/_ref) on random blocks,
* the encoder-vs-pipeline agreement check (test_encoder.cpp:169-202) is in
  tests/test_gpu_fit.py (it needs a device encode).
"""
import os

import numpy as np
import pytest

import paper_1404_0774_b200 as fic

REF_SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                      "libfic_ref.so")


def blk(side, vals):
    return np.asarray(vals, np.float64).reshape(side, side)


def test_is_shadow_known_answers():
    # test_encoder.cpp:15-21
    assert fic.is_shadow(np.full((4, 4), 128.0), 0.0)
    assert not fic.is_shadow(blk(2, [0, 255, 0, 255]), 0.0)
    assert not fic.is_shadow(blk(2, [1, 1, 1, 2]), 0.0)  # 4*7 - 5^2 = 3 > 0
    assert fic.is_shadow(blk(2, [1, 1, 1, 2]), 3.0)


def test_least_squares_known_answers():
    # perfect self-match survives the default quantiser (test_encoder.cpp:23-29)
    a = blk(2, [10, 30, 70, 110])
    q = fic.least_squares(a, a, fic.CodecParams())
    assert (q.s, q.o, q.residual) == (1.0, 0.0, 0.0)
    # zero-variance code block forces s = 0, o = mean (:31-38)
    f = fic.least_squares_fit(blk(2, [5, 5, 5, 5]), blk(2, [1, 3, 5, 7]))
    assert (f.s, f.o, f.residual) == (0.0, 4.0, 20.0)
    # exact regression line (:40-46)
    f = fic.least_squares_clamped(blk(2, [0, 2, 4, 6]), blk(2, [1, 2, 3, 4]), fic.CodecParams())
    assert (f.s, f.o, f.residual) == (0.5, 1.0, 0.0)
    # clamped scale re-fits the offset (:48-58)
    raw = fic.least_squares_fit(blk(2, [0, 1, 2, 3]), blk(2, [1, 3, 5, 7]))
    assert (raw.s, raw.residual) == (2.0, 0.0)
    f = fic.least_squares_clamped(blk(2, [0, 1, 2, 3]), blk(2, [1, 3, 5, 7]), fic.CodecParams())
    assert (f.s, f.o, f.residual) == (1.0, 2.5, 5.0)


def test_least_squares_errors():
    # mismatched blocks (test_encoder.cpp:60-63)
    with pytest.raises(fic.CodecError, match="SideMismatch"):
        fic.least_squares_fit(np.zeros((2, 2)), np.zeros((4, 4)))
    with pytest.raises(fic.CodecError, match="SideMismatch"):
        fic.least_squares(np.zeros((2, 2)), np.zeros((4, 4)))
    # params are normalised first (least_squares_clamped, encoder.cpp:79)
    with pytest.raises(fic.CodecError, match="BadParams"):
        p = fic.CodecParams()
        p._p.n = 3
        fic.least_squares_clamped(np.zeros((2, 2)), np.zeros((2, 2)), p)
    with pytest.raises(ValueError):
        fic.least_squares_fit(np.zeros((2, 3)), np.zeros((2, 3)))


def test_raw_fit_minimises():
    # test_encoder.cpp:65-86: the unconstrained fit is the minimum of the quadratic
    rng = np.random.default_rng(41)
    for _ in range(20):
        a = rng.integers(0, 256, (4, 4)).astype(np.float64)
        b = rng.integers(0, 256, (4, 4)).astype(np.float64)
        f = fic.least_squares_fit(a, b)
        for ds, do in [(1e-3, 0), (-1e-3, 0), (0, 1e-2), (0, -1e-2)]:
            r = float(np.sum(((f.s + ds) * a + (f.o + do) - b) ** 2))
            assert r >= f.residual - 1e-9


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (needs /root/reference)")
def test_against_compiled_reference():
    """Bit-exact against the unmodified reference functions on random and degenerate blocks,
    under several parameter sets (s_max clamp both ways, coarse quantisers, shadow_eps)."""
    from oracle import Reference
    ref = Reference()
    rng = np.random.default_rng(1404)
    params = [dict(), dict(s_max=0.5, s_bits=3, o_bits=4), dict(s_max=2.0, shadow_eps=50.0), dict(n=8, s_bits=16)]
    for trial in range(600):
        side = [1, 2, 4, 8][trial % 4]
        kind = trial % 5
        if kind == 0:
            a = rng.integers(0, 256, (side, side)) * 1.0
        elif kind == 1:
            a = rng.integers(0, 1021, (side, side)) / 4.0  # contracted cells (2x2 means)
        elif kind == 2:
            a = np.full((side, side), float(rng.integers(0, 256)))  # flat code block
        elif kind == 3:
            a = rng.normal(100, 40, (side, side))
        else:
            a = np.zeros((side, side))
            a.flat[rng.integers(0, side * side)] = 1.0
        b = rng.integers(0, 256, (side, side)) * 1.0
        if trial % 7 == 0:
            b = 3.0 * a - 17.0  # exact line, |s| > s_max
        pv = params[trial % len(params)]
        p = fic.CodecParams(**pv)
        eps = pv.get("shadow_eps", 0.0)
        got = fic.least_squares_fit(a, b, eps)
        want = ref.least_squares("fit", a, b, pv, eps)
        assert np.array([got.s, got.o, got.residual]).tobytes() == np.array(want[:3]).tobytes(), (trial, pv)
        got = fic.least_squares_clamped(a, b, p)
        want = ref.least_squares("clamped", a, b, pv)
        assert np.array([got.s, got.o, got.residual]).tobytes() == np.array(want[:3]).tobytes(), (trial, pv)
        got = fic.least_squares(a, b, p)
        want = ref.least_squares("quantized", a, b, pv)
        assert (got.qs, got.qo) == want[3:], (trial, pv)
        assert np.array([got.s, got.o, got.residual]).tobytes() == np.array(want[:3]).tobytes(), (trial, pv)
        for e in (0.0, 3.0, 1e3):
            assert fic.is_shadow(b, e) == ref.is_shadow(b, e)
            assert fic.is_shadow(a, e) == ref.is_shadow(a, e)
