"""GPU-side checks of the integer core and the per-candidate pipeline.

* K1 read-back (C-ABI fic_debug_pool): the pool builder's exact moments {Sq, den}, flat
  flags/count and its per-isometry u16 cells equal the oracle's domain pool bit for bit
  (north_star: "integer moments and Sigma rd must be bit-exact"; encoder.cpp:205-223), and the
  survivor evaluation's DP2A correlations equal sum_i q[perm_s(i)] b_i (encoder.cpp:236-241),
  on the benched configurations (cfg2, cfg3, cfg4 moments) and the small geometries.
* The encoder agrees with the public per-candidate pipeline (proj/tests/test_encoder.cpp:169-202):
  the GPU encode of smooth_image(16, 51) equals the strict-minimum search over least_squares
  of every (domain, isometry) code block.
"""
import numpy as np
import pytest

import paper_1404_0774_b200 as fic
from paper_1404_0774_b200 import images

pytestmark = pytest.mark.gpu


def sym_perm(n):
    """perm[s, i] = the contracted cell isometry s reads for range pixel i (transforms.cpp:13-26)."""
    m = n - 1
    src = [lambda r, c: (r, c), lambda r, c: (m - c, r), lambda r, c: (m - r, m - c), lambda r, c: (c, m - r),
           lambda r, c: (r, m - c), lambda r, c: (m - r, c), lambda r, c: (c, r), lambda r, c: (m - c, m - r)]
    perm = np.zeros((8, n * n), np.int64)
    for s in range(8):
        for i in range(n * n):
            sr, sc = src[s](i // n, i % n)
            perm[s, i] = sr * n + sc
    return perm


CASES = {
    "cfg2": (lambda o: images.ct_slice(512, 1404002), dict(n=8, step=4), True),
    "cfg3": (lambda o: images.ct_slice(512, 1404002), dict(n=4, step=2), True),
    "cfg4": (lambda o: images.xray(2048, 1404004), dict(n=8, step=2), False),  # moments only (q8: 1 GB)
    "n2s1": (lambda o: o.noise_image(64, 7), dict(n=2, step=1), True),
    "flat": (lambda o: np.pad(o.smooth_image(64, 5)[:, 24:], ((0, 0), (24, 0)), constant_values=77),
             dict(n=4, step=2, shadow_eps=40.0), True),
}


@pytest.mark.parametrize("case", list(CASES))
def test_pool_moments_and_correlations_bit_exact(oracle, case):
    gen, pv, full_q8 = CASES[case]
    img = gen(oracle)
    p = fic.CodecParams(**pv)
    n, N = p.n, p.n * p.n
    q, sq, sqq, flat = oracle.domain_pool(img, pv)
    D = len(sq)
    rng = np.random.default_rng(sum(map(ord, case)))
    R = (img.shape[0] // n) ** 2
    k = 4096
    rr = rng.integers(0, R, k)
    dd = rng.integers(0, D, k)
    ss = rng.integers(0, 8, k)
    rr[:4] = [0, R - 1, 0, R - 1]  # first and last range and domain
    dd[:4] = [0, D - 1, D - 1, 0]
    got = fic.debug_pool(img, p, probes=(rr, dd, ss), want_q8=full_q8)
    assert np.array_equal(got["sq"], sq)
    want_den = np.where(flat, -1, N * sqq - sq * sq)
    assert np.array_equal(got["den"], want_den)
    assert got["flat_count"] == int(flat.sum())
    perm = sym_perm(n)
    if full_q8:
        assert np.array_equal(got["q8"].astype(np.int64), q.astype(np.int64)[:, perm])
    # exact correlations sum_i q[d, perm_s(i)] * b_i of the sampled candidates
    side = img.shape[0]
    RX = side // n
    b = img.astype(np.int64).reshape(RX, n, RX, n).transpose(0, 2, 1, 3).reshape(R, N)
    want = np.einsum("ki,ki->k", q.astype(np.int64)[dd[:, None], perm[ss]], b[rr])
    assert np.array_equal(got["corr"], want)


def contract(block):
    h = block.shape[0] // 2
    return (block[0::2, 0::2] + block[0::2, 1::2] + block[1::2, 0::2] + block[1::2, 1::2]) / 4.0


def apply_symmetry(b, s):
    n = b.shape[0]
    perm = sym_perm(n)[s]
    return b.reshape(-1)[perm].reshape(n, n)


def test_encoder_agrees_with_public_pipeline(oracle):
    # proj/tests/test_encoder.cpp:169-202
    img = oracle.smooth_image(16, 51)
    p = fic.CodecParams()
    enc = fic.encode(img, p)
    n = 4
    f = img.astype(np.float64)
    for ry in range(4):
        for rx in range(4):
            rng_blk = f[ry * 4:ry * 4 + 4, rx * 4:rx * 4 + 4]
            got = enc.mappings[ry * 4 + rx]
            if fic.is_shadow(rng_blk, p.shadow_eps):
                assert got["qs"] == 0 and (got["x"], got["y"]) == (0, 0)
                continue
            best, best_r = None, np.inf
            for x in range(0, 16 - 2 * n + 1, p.step):  # domain_positions: x outer, y inner
                for y in range(0, 16 - 2 * n + 1, p.step):
                    for s in range(8):
                        cb = apply_symmetry(contract(f[y:y + 2 * n, x:x + 2 * n]), s)
                        if fic.is_shadow(cb, p.shadow_eps):
                            continue
                        q = fic.least_squares(cb, rng_blk, p)
                        if q.residual < best_r:
                            best_r = q.residual
                            best = (x, y, s, q.qs, q.qo, q.residual)
            assert best is not None
            assert (int(got["x"]), int(got["y"]), int(got["sym"]), int(got["qs"]), int(got["qo"])) == best[:5]
            assert np.float64(got["residual"]).tobytes() == np.float64(best[5]).tobytes()
