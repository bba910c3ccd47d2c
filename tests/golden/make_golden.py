"""Generates tests/golden/golden.npz from the UNMODIFIED reference library.

    make -C oracle ref && python tests/golden/make_golden.py

The reference (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
oracle/_ref/libfic_ref.so) is run on the reference's own fixtures (noise_image /
smooth_image from proj/tests/testimg.hpp with the seeds its tests use) and on this
repo's synthetic configuration images (sampled ranges for the large ones).  The fixture
stores inputs (or their SHA-256 when large), code records, EncodeStats, decoded images,
step RMSE and FIC1 bytes.  It exists so the C restatement in oracle/ (and through it the
GPU path) is pinned to the reference even where /root/reference is absent.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402


def stats_arr(st):
    return np.array([st["candidates_tested"], st["shadow_ranges"], st["shadow_codeblocks"]], np.uint64)


def main():
    R = Reference()
    out = {}

    # test_encoder.cpp:152-167 — noise_image(32, 50..52) x three parameter variants
    variants = [dict(), dict(step=2, s_max=0.75), dict(o_bits=6, s_bits=4)]
    for i, pv in enumerate(variants):
        img = R.noise_image(32, 50 + i)
        m, st = R.encode(img, pv)
        out[f"noise32_v{i}_img"] = img
        out[f"noise32_v{i}_maps"] = m
        out[f"noise32_v{i}_stats"] = stats_arr(st)
        out[f"noise32_v{i}_fic1"] = np.frombuffer(R.serialize(m, 32, pv), np.uint8)

    # acceptance.cpp:73-91 — noise_image(32, 201..205), defaults; the reference brute force
    for seed in range(201, 206):
        img = R.noise_image(32, seed)
        out[f"accept_{seed}_maps"] = R.oracle_encode(img, {})

    # geometry sweep on the reference fixtures
    for n, step in [(2, 1), (4, 3), (8, 3), (16, 4)]:
        side = max(64, 4 * n)
        for kind, img in (("smooth", R.smooth_image(side, 52 + n)), ("noise", R.noise_image(side, 7 + step))):
            pv = dict(n=n, step=step)
            m, st = R.encode(img, pv)
            key = f"geo_{kind}_n{n}_s{step}"
            out[key + "_img"] = img
            out[key + "_maps"] = m
            out[key + "_stats"] = stats_arr(st)

    # shadow_eps and flat-codebook cases
    img = R.smooth_image(64, 5)
    img[:, :24] = 77
    for i, pv in enumerate([dict(), dict(shadow_eps=40.0), dict(n=8, step=2, shadow_eps=500.0)]):
        m, st = R.encode(img, pv)
        out[f"flat{i}_maps"] = m
        out[f"flat{i}_stats"] = stats_arr(st)
    out["flat_img"] = img

    # decoder: smooth_image(32, 61), s_max 0.9 at scales 1 and 2, from mid-gray and black
    img = R.smooth_image(32, 61)
    pv = dict(s_max=0.9)
    m, _ = R.encode(img, pv)
    out["dec_img"] = img
    out["dec_maps"] = m
    for scale in (1, 2):
        for init in ("mid-gray", "black"):
            o, rm, runs = R.decode(m, 32, pv, scale, 12, init)
            key = f"dec_s{scale}_{init.replace('-', '')}"
            out[key + "_out"] = o
            out[key + "_rmse"] = rm
    out["dec_collage"] = np.array([R.collage_error(img, m, pv)])

    # synthetic configuration images (this repo's generators; hashes pin them)
    cfg1 = images.phantom(256, 1404001)
    m, st = R.encode(cfg1, dict(n=8, step=8), workers=os.cpu_count() or 1)
    out["cfg1_sha256"] = np.frombuffer(hashlib.sha256(cfg1.tobytes()).digest(), np.uint8)
    out["cfg1_maps"] = m
    out["cfg1_stats"] = stats_arr(st)
    o, rm, _ = R.decode(m, 256, dict(n=8, step=8), 1, 10, "mid-gray")
    out["cfg1_dec10"] = o
    out["cfg1_psnr"] = np.array([R.psnr(cfg1, o)])

    rng = np.random.default_rng(1404)
    for cfg, gen, n, step, count in [("cfg2", lambda: images.ct_slice(512, 1404002), 8, 4, 48),
                                      ("cfg3", lambda: images.ct_slice(512, 1404002), 4, 2, 24),
                                      ("cfg4", lambda: images.xray(2048, 1404004), 8, 2, 6)]:
        img = gen()
        RX = img.shape[1] // n
        idx = np.sort(rng.choice(RX * RX, size=count, replace=False))
        maps = []
        for r in idx:
            rec, _ = R.encode_range(img, int(r % RX) * n, int(r // RX) * n, dict(n=n, step=step))
            maps.append(rec)
        out[f"{cfg}_sha256"] = np.frombuffer(hashlib.sha256(img.tobytes()).digest(), np.uint8)
        out[f"{cfg}_sample_idx"] = idx.astype(np.int64)
        out[f"{cfg}_sample_maps"] = np.array(maps)
        print(cfg, "sampled", count, flush=True)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), sum(v.nbytes for v in out.values()), "bytes")


if __name__ == "__main__":
    main()
