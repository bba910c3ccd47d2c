"""Generates tests/golden/cfg4_rows.npz: the UNMODIFIED reference's records for 16 full range
rows of cfg4 (2048x2048 X-ray-shaped synthetic image, 8x8 ranges, domain stride 2).

    make -C oracle ref && python tests/golden/make_cfg4_rows.py

A cfg4 row costs ~37 s of reference search on 16 host threads (256 ranges x 1,034,289
domains x 8 isometries), so the GPU test compares against these stored records instead of
re-running the reference (proj/src/encoder.cpp:332-342, encode_range per range, spread over
host threads) on the GPU box.  Rows: the first, the last, and 14 seeded random ones; every
row includes the first and last range columns.  The image is stored as its SHA-256.
"""
import hashlib
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402
from paper_1404_0774_b200.abi import MAPPING_DTYPE  # noqa: E402


def rows():
    rng = np.random.default_rng(14040004)
    mid = sorted(rng.choice(np.arange(1, 255), 14, replace=False).tolist())
    return [0] + mid + [255]


def main():
    ref = Reference()
    img = images.xray(2048, 1404004)
    pv = dict(n=8, step=2)
    rs = rows()
    jobs = [(r, c) for r in rs for c in range(256)]
    t0 = time.time()

    def one(job):
        r, c = job
        m, _ = ref.encode_range(img, c * 8, r * 8, pv)
        return m

    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        recs = list(ex.map(one, jobs))
    maps = np.array(recs, MAPPING_DTYPE)
    np.savez_compressed(os.path.join(HERE, "cfg4_rows.npz"), rows=np.array(rs, np.int32), maps=maps,
                        image_sha256=np.frombuffer(hashlib.sha256(img.tobytes()).digest(), np.uint8))
    print(f"{len(jobs)} ranges in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
