"""CPU: pins the oracle (oracle/fic_oracle.c, a restatement of the reference's encode /
decode path) against the reference's own known answers and against golden vectors
produced by the unmodified reference library (tests/golden/make_golden.py)."""
import hashlib

import numpy as np
import pytest

from paper_1404_0774_b200 import images


KEYS = ["x", "y", "sym", "qs", "qo"]


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["residual"].view(np.uint64), b["residual"].view(np.uint64)), "residual bits"


def st(g):
    return {"candidates_tested": int(g[0]), "shadow_ranges": int(g[1]), "shadow_codeblocks": int(g[2])}


# ---- known answers of the reference's unit tests ----

def test_mt19937_and_fixtures(oracle, golden):
    assert oracle.mt19937(5489, 1)[0] == 3499211612  # std::mt19937 default-seed first draw
    assert np.array_equal(oracle.noise_image(32, 50), golden["noise32_v0_img"])
    assert np.array_equal(images.noise_image(32, 51), golden["noise32_v1_img"])
    for n, step in [(2, 1), (4, 3), (8, 3), (16, 4)]:
        side = max(64, 4 * n)
        assert np.array_equal(oracle.smooth_image(side, 52 + n), golden[f"geo_smooth_n{n}_s{step}_img"])
        assert np.array_equal(images.smooth_image(side, 52 + n), golden[f"geo_smooth_n{n}_s{step}_img"])


def test_quantizer_reference_points(oracle):
    # test_format.cpp:11-42, 147-161
    assert oracle.quantize(0.0, 1.0, 5) == 0 and oracle.dequantize(0, 1.0, 5) == 0.0
    assert oracle.quantize(1.0, 1.0, 5) == 31 and oracle.dequantize(31, 1.0, 5) == 1.0
    step = 2 * 0.9 / 31
    for i in range(-1000, 1001):
        s = 0.9 * i / 1000.0
        assert abs(s - oracle.dequantize(oracle.quantize(s, 0.9, 5), 0.9, 5)) <= step + 1e-12
    assert oracle.dequantize(oracle.quantize(255.0, 255.0, 7), 255.0, 7) == 255.0
    for sb in (2, 5, 9):
        for ob in (3, 7, 12):
            assert oracle.dequantize(oracle.quantize(1.0, 1.0, sb), 1.0, sb) == 1.0
            assert oracle.dequantize(oracle.quantize(255.0, 255.0, ob), 255.0, ob) == 255.0


def test_isometry_table_on_2x2():
    # test_transforms.cpp:22-31, via the decoder's symmetry_source on a 1x1-range grid:
    # apply_symmetry([[1,2],[3,4]], s) expected sample orders
    import ctypes
    from oracle import Oracle
    L = Oracle().L
    L.oracle_symmetry_source.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
    block = [1, 2, 3, 4]
    expect = {0: [1, 2, 3, 4], 1: [3, 1, 4, 2], 2: [4, 3, 2, 1], 3: [2, 4, 1, 3], 4: [2, 1, 4, 3], 5: [3, 4, 1, 2],
              6: [1, 3, 2, 4], 7: [4, 2, 3, 1]}
    for s, want in expect.items():
        got = []
        for r in range(2):
            for c in range(2):
                sr, sc = ctypes.c_int(), ctypes.c_int()
                L.oracle_symmetry_source(s, r, c, 2, ctypes.byref(sr), ctypes.byref(sc))
                got.append(block[sr.value * 2 + sc.value])
        assert got == want, s


def test_domain_counts(oracle):
    # test_codebook.cpp:10-48
    img = np.zeros((256, 256), np.uint8)
    q, sq, sqq, flat = oracle.domain_pool(img, dict(n=4, step=2))
    assert len(sq) == 15625
    assert len(oracle.domain_pool(img, dict(n=4, step=4))[1]) == 3969
    assert len(oracle.domain_pool(np.zeros((8, 8), np.uint8), dict(n=4, step=4))[1]) == 1
    assert (256 // 4) ** 2 * 15625 == 64000000


def test_shadow_known_answers(oracle):
    # test_encoder.cpp:102-121: constant images are all-shadow with exact mappings
    for v in (0, 128, 255):
        img = np.full((16, 16), v, np.uint8)
        m, s = oracle.encode(img, {})
        assert s == {"candidates_tested": 0, "shadow_ranges": 16, "shadow_codeblocks": 0}
        assert (m["qs"] == 0).all() and (m["x"] == 0).all() and (m["sym"] == 0).all()
        assert (m["qo"] == oracle.quantize(float(v), 255.0, 7)).all()
        if v in (0, 255):
            assert (m["residual"] == 0.0).all()


def test_single_domain_argmin(oracle):
    # test_encoder.cpp:123-129: noise_image(8, 42), one domain position, 8 candidates
    img = oracle.noise_image(8, 42)
    m, s = oracle.encode_ranges(img, {}, [0], [0])
    assert s["candidates_tested"] == 8
    b, _ = oracle.encode(img, {}, brute=True)
    same(m, b[:1])


# ---- golden vectors from the reference library ----

@pytest.mark.parametrize("i,pv", [(0, dict()), (1, dict(step=2, s_max=0.75)), (2, dict(o_bits=6, s_bits=4))])
def test_noise32_variants(oracle, golden, i, pv):
    img = golden[f"noise32_v{i}_img"]
    m, s = oracle.encode(img, pv)
    same(m, golden[f"noise32_v{i}_maps"])
    assert s == st(golden[f"noise32_v{i}_stats"])
    b, _ = oracle.encode(img, pv, brute=True)  # pruning never changes the answer
    same(b, m)  # (the device FIC1 packing of these records: tests/test_gpu_fic1.py)


@pytest.mark.parametrize("seed", range(201, 206))
def test_acceptance_brute_force(oracle, golden, seed):
    img = oracle.noise_image(32, seed)
    m, _ = oracle.encode(img, {})
    same(m, golden[f"accept_{seed}_maps"])


@pytest.mark.parametrize("n,step", [(2, 1), (4, 3), (8, 3), (16, 4)])
def test_geometry_sweep(oracle, golden, n, step):
    for kind in ("smooth", "noise"):
        key = f"geo_{kind}_n{n}_s{step}"
        m, s = oracle.encode(golden[key + "_img"], dict(n=n, step=step))
        same(m, golden[key + "_maps"])
        assert s == st(golden[key + "_stats"])


def test_flat_and_shadow_eps(oracle, golden):
    img = golden["flat_img"]
    for i, pv in enumerate([dict(), dict(shadow_eps=40.0), dict(n=8, step=2, shadow_eps=500.0)]):
        m, s = oracle.encode(img, pv)
        same(m, golden[f"flat{i}_maps"])
        assert s == st(golden[f"flat{i}_stats"])


def test_decoder_golden(oracle, golden):
    m = golden["dec_maps"]
    for scale in (1, 2):
        for init in ("mid-gray", "black"):
            key = f"dec_s{scale}_{init.replace('-', '')}"
            out, rm, runs = oracle.decode(m, 32, dict(s_max=0.9), scale, 12, init)
            assert np.array_equal(out, golden[key + "_out"])
            assert np.array_equal(rm.view(np.uint64), golden[key + "_rmse"].view(np.uint64))
    assert oracle.collage_error(golden["dec_img"], m, dict(s_max=0.9)) == golden["dec_collage"][0]


def test_cfg1_golden(oracle, golden):
    img = images.phantom(256, 1404001)
    assert hashlib.sha256(img.tobytes()).digest() == golden["cfg1_sha256"].tobytes()
    m, s = oracle.encode_threaded(img, dict(n=8, step=8))
    same(m, golden["cfg1_maps"])
    assert s == st(golden["cfg1_stats"])
    out, _, _ = oracle.decode(m, 256, dict(n=8, step=8), 1, 10)
    assert np.array_equal(out, golden["cfg1_dec10"])
    assert oracle.psnr(img, out) == golden["cfg1_psnr"][0]


@pytest.mark.parametrize("cfg,n,step", [("cfg2", 8, 4), ("cfg3", 4, 2), ("cfg4", 8, 2)])
def test_config_samples_golden(oracle, golden, cfg, n, step):
    gen = {"cfg2": lambda: images.ct_slice(512, 1404002), "cfg3": lambda: images.ct_slice(512, 1404002),
           "cfg4": lambda: images.xray(2048, 1404004)}[cfg]
    img = gen()
    assert hashlib.sha256(img.tobytes()).digest() == golden[f"{cfg}_sha256"].tobytes()
    idx = golden[f"{cfg}_sample_idx"]
    RX = img.shape[1] // n
    xs = (idx % RX) * n
    ys = (idx // RX) * n
    m, _ = oracle.encode_ranges(img, dict(n=n, step=step), xs, ys)
    same(m, golden[f"{cfg}_sample_maps"])
